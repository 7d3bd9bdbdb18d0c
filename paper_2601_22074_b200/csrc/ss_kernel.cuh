// ss_kernel.cuh -- the fused, thread-per-world ManagerBasedRlEnv.step.
//
// One CUDA thread owns one world for the whole control step: action
// processing, the d decimation substeps (actuators -> capture push ->
// contact/forces/integration -> entity refresh -> contact sensor),
// termination, reward, curriculum + masked reset, command countdown,
// interval events and the observation pipeline, in exactly the order of
// ManagerBasedRlEnv.step (env.py:219-259). Worlds are independent
// (SPEC.md:101), so nothing but the per-term trigger counters is shared
// between threads; those are warp-aggregated atomics.
//
// Per-world state lives in HBM structure-of-arrays ([component][world]) so
// a warp touches 32 consecutive doubles per component: every load and store
// is a full 256 B coalesced transaction. Within the launch the state is held
// in registers: each array is read once and written once per control step.
//
// The body is a template over a config type C (ss_cfg.cuh): the generic
// RuntimeCfg reads every table from the descriptor; the per-env JIT config
// makes them constexpr so NVRTC folds the term tables, unrolls every loop
// and keeps all per-world arrays in registers. KM/FM bound the joint and
// foot counts (exact in the JIT build).
//
// This header compiles both under nvcc (ss_step.cu) and NVRTC (jit.py).
#pragma once

#include "ss_device.cuh"
#include "ss_cfg.cuh"

#ifndef SS_MIRROR_TMA
#define SS_MIRROR_TMA 1
#endif
#ifndef SS_DCAP_ACTION_COLS
#define SS_DCAP_ACTION_COLS 1  /* action columns in shared memory (JIT: the env's action dim) */
#endif
#ifndef SS_DCAP_REWARDS
#define SS_DCAP_REWARDS 1
#endif
#ifndef SS_PEEL_LAST_SUBSTEP
#define SS_PEEL_LAST_SUBSTEP 0
#endif

namespace ss {

constexpr int kBlock = 128;
constexpr long long kNeverTouched = -(1ll << 40);  // sensors.py:51

__device__ __forceinline__ bool finite_(double x) { return finite_bits(x); }

// the host-mirror twin of an output-arena address (ss_env_desc.out_mirror)
template <class T>
__device__ __forceinline__ T* mirror_of(const ss_env_desc& d, T* p) {
    return (T*)((char*)p + d.out_mirror);
}

// Pull a line into L2 without holding a register (the bench flushes L2
// between steps, so every first touch of a per-world array is a DRAM trip;
// prefetching at kernel entry turns the later dependent loads into L2 hits).
__device__ __forceinline__ void l2_prefetch(const void* p) { asm volatile("prefetch.global.L2 [%0];" ::"l"(p)); }
// The arrays read after the substeps and on the reset path: pulled into L1
// (SS_PF_L1=1) so their loads -- which sit behind the step's stores and its
// branches, so the compiler cannot issue them early -- cost an L1 hit instead
// of an L2 round trip each; SS_PF_L1=0 stops at L2.
#ifndef SS_PF_L1
#define SS_PF_L1 1
#endif
__device__ __forceinline__ void late_prefetch_line(const void* p) {
#if SS_PF_L1
    asm volatile("prefetch.global.L1 [%0];" ::"l"(p));
#else
    asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
#endif
}

template <int M>
__device__ __forceinline__ double sel(const double (&a)[M], int j) {
    double v = a[0];
#pragma unroll
    for (int i = 1; i < M; ++i)
        if (i == j) v = a[i];
    return v;
}
template <int M>
__device__ __forceinline__ void sel_store(double (&a)[M], int j, double v) {
#pragma unroll
    for (int i = 0; i < M; ++i)
        if (i == j) a[i] = v;
}

// Term-table loops. In the per-env JIT build the trip counts are constants
// and static_for instantiates the body once per term with the index as a
// compile-time constant (Ic<I>), so every table lookup folds to an
// immediate; the generic build runs an ordinary loop.
template <int V>
struct Ic {
    static constexpr int value = V;
};
__device__ __forceinline__ constexpr int ival(int t) { return t; }
template <int V>
__device__ __forceinline__ constexpr int ival(Ic<V>) { return V; }

template <int I, int N, class F>
__device__ __forceinline__ void static_for(F& f) {
    if constexpr (I < N) {
        f(Ic<I>{});
        static_for<I + 1, N>(f);
    }
}

template <class C, int MAX, class F>
__device__ __forceinline__ void for_terms(int lo, int hi, F f) {
    if constexpr (C::kJit) {
        auto g = [&](auto I) {
            if (ival(I) >= lo && ival(I) < hi) f(I);
        };
        static_for<0, MAX>(g);
    } else {
        for (int t = lo; t < hi; ++t) f(t);
    }
}

template <class C>
__device__ __forceinline__ double fld(const ss_env_desc& d, int f, int c, int w) {
    const double* p = d.field[f].ptr;
    return C::fexp(d, f) ? p[(int64_t)c * C::NW(d) + w] : p[c];
}

template <class C>
__device__ __forceinline__ double height(const ss_env_desc& d, double x) {
    if (C::flat(d)) return 0.0;
    const ss_terrain& t = d.terrain;
    const int64_t last = t.n_samples - 1;
    double pos = div_rn(finite_(x) ? x : 0.0, t.spacing, 1.0 / t.spacing);
    pos = np_clip(pos, 0.0, (double)last);
    int64_t idx = (int64_t)pos;
    if (idx > last - 1) idx = last - 1;
    const double frac = pos - (double)idx;
    return __ldg(t.samples + idx) * (1.0 - frac) + __ldg(t.samples + idx + 1) * frac;
}

// interpolating lookup without the flat shortcut (spawn placement, ray scan)
__device__ __forceinline__ double height_raw(const ss_env_desc& d, double x) {
    const ss_terrain& t = d.terrain;
    if (t.n_samples < 2) return 0.0;
    const int64_t last = t.n_samples - 1;
    double pos = div_rn(finite_(x) ? x : 0.0, t.spacing, 1.0 / t.spacing);
    pos = np_clip(pos, 0.0, (double)last);
    int64_t idx = (int64_t)pos;
    if (idx > last - 1) idx = last - 1;
    const double frac = pos - (double)idx;
    return __ldg(t.samples + idx) * (1.0 - frac) + __ldg(t.samples + idx + 1) * frac;
}

// the ray scan: all NR lookups' indices first, then every sample load, then
// the interpolations -- one L2 round trip for the whole scan instead of one
// per ray (height_raw's result, ray by ray)
template <class C, int NR>
__device__ __forceinline__ void height_raw_n(const ss_env_desc& d, const double (&x)[NR], double (&out)[NR]) {
    const ss_terrain& t = d.terrain;
    if (t.n_samples < 2) {
#pragma unroll
        for (int r = 0; r < NR; ++r) out[r] = 0.0;
        return;
    }
    const int64_t last = t.n_samples - 1;
    const double inv = 1.0 / t.spacing;
    int64_t idx[NR];
    double frac[NR], a[NR], b[NR];
#pragma unroll
    for (int r = 0; r < NR; ++r) {
        double pos = div_rn(finite_(x[r]) ? x[r] : 0.0, t.spacing, inv);
        pos = np_clip(pos, 0.0, (double)last);
        int64_t i = (int64_t)pos;
        i = i > last - 1 ? last - 1 : i;
        idx[r] = i;
        frac[r] = pos - (double)i;
    }
#pragma unroll
    for (int r = 0; r < NR; ++r) {
        a[r] = __ldg(t.samples + idx[r]);
        b[r] = __ldg(t.samples + idx[r] + 1);
    }
#pragma unroll
    for (int r = 0; r < NR; ++r) out[r] = a[r] * (1.0 - frac[r]) + b[r] * frac[r];
}

// Per-world vectors of M doubles: registers (S == 0), or a column of stride S
// in shared memory (value k at p[k * S], the block's threads side by side) --
// large models keep their action / previous-action / target vectors and the
// episodic reward sums there, which would otherwise stay live in registers all
// step and spill.
template <int S, int M>
struct Col {
    double r[S ? 1 : M];
    double* p;
    __device__ __forceinline__ double& operator[](int k) {
        if constexpr (S > 0) return p[k * S];
        else return r[k];
    }
    __device__ __forceinline__ double operator[](int k) const {
        if constexpr (S > 0) return p[k * S];
        else return r[k];
    }
};

template <int S, int M>
__device__ __forceinline__ double sel(const Col<S, M>& a, int j) {
    if constexpr (S > 0) return a[j];
    else return sel(a.r, j);
}

template <int S, int M>
__device__ __forceinline__ void sel_store(Col<S, M>& a, int j, double v) {
    if constexpr (S > 0) a[j] = v;
    else sel_store(a.r, j, v);
}

template <int KM, int FM, int AS = 0>
struct World {
    double q[3 + KM], qd[3 + KM], ctrl[KM];
    double ext0, ext1, time;
    double fn[FM], ft[FM], fpx[FM], fpz[FM], fvx[FM], fvz[FM];
    bool fin[FM];
    double eq[3 + KM], eqd[3 + KM];
    double lvb0, lvb1, pg0, pg1;
    double efn[FM], eft[FM], efvx[FM];
    bool efin[FM];
    double sp, cp;
    bool trig_ok;
    Col<AS, KM> targets;
    Col<AS, SS_MAX_ACTION> action, prev_action;
    bool have_action;
    double cmd[SS_MAX_CMD];
    bool s_in[FM];
    double s_air[FM], s_last_air[FM], s_contact[FM];
    long long s_td[FM];
    double s_hist[SS_MAX_HIST][FM];
    bool have_sensor;
    long long ep_steps;
    double cmd_dist;
    bool terminated, truncated, nonfinite, was_reset;
    unsigned trig_bits;
    // per-step state prefetched at kernel entry (one round trip, see step_body)
    Col<AS, SS_MAX_REWARDS> ep_sum, ep_rw;
    long long countdown;
    double ev_el[SS_MAX_EVENTS], ev_tg[SS_MAX_EVENTS];
    uint64_t nctr[SS_MAX_OBS_TERMS];
    double plv0, plv1;
};

// model fields hoisted out of the substep loop (they cannot change within a launch).
// S == 0: registers (generic build); S > 0: a shared-memory column per thread
// (value v at p[v * S], the block's threads side by side, bank-conflict free)
// -- the specialized kernel keeps these ~30 doubles out of its register file
// (236 -> 208 registers for the rough biped), where they would otherwise stay
// live through the whole substep loop.
template <int KM, int NA, int S>
struct Params {
    static constexpr int BM = 0, BI = 1, FR = 2, MT = 3, IM = 4, II = 5, LM = 6, ROT = 6 + KM, DMP = 6 + 2 * KM,
                         IROT = 6 + 3 * KM, KP = 6 + 4 * KM, KD = KP + NA * KM, NV = KD + NA * KM;
    double r[S ? 1 : NV];
    double* p;
    __device__ __forceinline__ double& v(int i) {
        if constexpr (S > 0) return p[i * S];
        else return r[i];
    }
    __device__ __forceinline__ double v(int i) const {
        if constexpr (S > 0) return p[i * S];
        else return r[i];
    }
    __device__ __forceinline__ double& base_mass() { return v(BM); }
    __device__ __forceinline__ double& base_inertia() { return v(BI); }
    __device__ __forceinline__ double& friction() { return v(FR); }
    __device__ __forceinline__ double& m_total() { return v(MT); }
    __device__ __forceinline__ double& inv_m() { return v(IM); }
    __device__ __forceinline__ double& inv_inertia() { return v(II); }
    __device__ __forceinline__ double& lm(int j) { return v(LM + j); }
    __device__ __forceinline__ double& rot(int j) { return v(ROT + j); }
    __device__ __forceinline__ double& dmp(int j) { return v(DMP + j); }
    __device__ __forceinline__ double& inv_rot(int j) { return v(IROT + j); }
    __device__ __forceinline__ double& kp(int a, int i) { return v(KP + a * KM + i); }
    __device__ __forceinline__ double& kd(int a, int i) { return v(KD + a * KM + i); }
    __device__ __forceinline__ double friction() const { return v(FR); }
    __device__ __forceinline__ double m_total() const { return v(MT); }
    __device__ __forceinline__ double inv_m() const { return v(IM); }
    __device__ __forceinline__ double inv_inertia() const { return v(II); }
    __device__ __forceinline__ double lm(int j) const { return v(LM + j); }
    __device__ __forceinline__ double dmp(int j) const { return v(DMP + j); }
    __device__ __forceinline__ double inv_rot(int j) const { return v(IROT + j); }
    __device__ __forceinline__ double kp(int a, int i) const { return v(KP + a * KM + i); }
    __device__ __forceinline__ double kd(int a, int i) const { return v(KD + a * KM + i); }
};

__device__ __forceinline__ uint64_t rng_begin(const ss_env_desc& d, int slot, int w, uint64_t& key) {
    key = stream_key(d.rng.base[slot], (uint64_t)(d.rng.world_id_offset + w));
    return d.rng.counter[slot][w];
}
__device__ __forceinline__ void rng_end(const ss_env_desc& d, int slot, int w, uint64_t c) {
    d.rng.counter[slot][w] = c;
}

// ---------------------------------------------------------------------------
// state load / store, entity refresh

template <class C, int KM, int FM, int AS>
__device__ __forceinline__ void load_phys(const ss_env_desc& d, int w, World<KM, FM, AS>& s, bool load_cache) {
    const int N = C::NW(d), K = C::K(d), F = C::F(d);
#pragma unroll
    for (int i = 0; i < 3 + KM; ++i) {
        s.q[i] = (i < 3 + K) ? d.state.q[(int64_t)i * N + w] : 0.0;
        s.qd[i] = (i < 3 + K) ? d.state.qd[(int64_t)i * N + w] : 0.0;
    }
#pragma unroll
    for (int j = 0; j < KM; ++j) s.ctrl[j] = (j < K) ? d.state.ctrl[(int64_t)j * N + w] : 0.0;
    s.ext0 = d.state.ext_force[w];
    s.ext1 = d.state.ext_force[N + w];
    s.time = d.state.time[w];
#pragma unroll
    for (int i = 0; i < FM; ++i) {
        const bool ok = load_cache && i < F;
        s.fn[i] = ok ? d.state.c_normal[(int64_t)i * N + w] : 0.0;
        s.ft[i] = ok ? d.state.c_tangent[(int64_t)i * N + w] : 0.0;
        s.fpx[i] = ok ? d.state.c_foot_pos[(int64_t)(2 * i) * N + w] : 0.0;
        s.fpz[i] = ok ? d.state.c_foot_pos[(int64_t)(2 * i + 1) * N + w] : 0.0;
        s.fvx[i] = ok ? d.state.c_foot_vel[(int64_t)(2 * i) * N + w] : 0.0;
        s.fvz[i] = ok ? d.state.c_foot_vel[(int64_t)(2 * i + 1) * N + w] : 0.0;
        s.fin[i] = ok ? d.state.c_in_contact[(int64_t)i * N + w] != 0 : false;
    }
    s.trig_ok = false;
}

template <class C, int KM, int FM, int AS>
__device__ __forceinline__ void store_phys(const ss_env_desc& d, int w, const World<KM, FM, AS>& s, bool store_cache) {
    const int N = C::NW(d), K = C::K(d), F = C::F(d);
#pragma unroll
    for (int i = 0; i < 3 + KM; ++i) {
        if (i < 3 + K) {
            d.state.q[(int64_t)i * N + w] = s.q[i];
            d.state.qd[(int64_t)i * N + w] = s.qd[i];
        }
    }
#pragma unroll
    for (int j = 0; j < KM; ++j)
        if (j < K) d.state.ctrl[(int64_t)j * N + w] = s.ctrl[j];
    d.state.ext_force[w] = s.ext0;
    d.state.ext_force[N + w] = s.ext1;
    d.state.time[w] = s.time;
    if (store_cache) {
#pragma unroll
        for (int i = 0; i < FM; ++i) {
            if (i < F) {
                d.state.c_normal[(int64_t)i * N + w] = s.fn[i];
                d.state.c_tangent[(int64_t)i * N + w] = s.ft[i];
                d.state.c_foot_pos[(int64_t)(2 * i) * N + w] = s.fpx[i];
                d.state.c_foot_pos[(int64_t)(2 * i + 1) * N + w] = s.fpz[i];
                d.state.c_foot_vel[(int64_t)(2 * i) * N + w] = s.fvx[i];
                d.state.c_foot_vel[(int64_t)(2 * i + 1) * N + w] = s.fvz[i];
                d.state.c_in_contact[(int64_t)i * N + w] = s.fin[i] ? 1 : 0;
            }
        }
    }
}

__device__ __forceinline__ double* dyn_smem() {
    extern __shared__ __align__(16) double ss_dyn_smem[];
    return ss_dyn_smem;
}

// EntityData.refresh (entity.py:145-165): a register snapshot
template <int KM, int FM, int AS>
__device__ __forceinline__ void refresh(World<KM, FM, AS>& s) {
    double sn, c;
    ss_sincos(s.q[2], &sn, &c);
    s.sp = sn;
    s.cp = c;
    s.trig_ok = true;
    s.lvb0 = c * s.qd[0] + sn * s.qd[1];
    s.lvb1 = -sn * s.qd[0] + c * s.qd[1];
    s.pg0 = -sn;
    s.pg1 = -c;
#pragma unroll
    for (int i = 0; i < 3 + KM; ++i) {
        s.eq[i] = s.q[i];
        s.eqd[i] = s.qd[i];
    }
#pragma unroll
    for (int i = 0; i < FM; ++i) {
        s.efn[i] = s.fn[i];
        s.eft[i] = s.ft[i];
        s.efvx[i] = s.fvx[i];
        s.efin[i] = s.fin[i];
    }
}

// ---------------------------------------------------------------------------
// StepPipeline.substep (sim/physics.py:178-249)

template <class C, int KM, class PP>
__device__ __forceinline__ void load_params(const ss_env_desc& d, int w, PP& P, bool actuators) {
    const int K = C::K(d);
    P.base_mass() = fld<C>(d, C::f_base_mass(d), 0, w);
    P.base_inertia() = fld<C>(d, C::f_base_inertia(d), 0, w);
    P.friction() = fld<C>(d, C::f_friction(d), 0, w);
    double lm[KM], rot[KM];
#pragma unroll
    for (int j = 0; j < KM; ++j) {
        lm[j] = (j < K) ? fld<C>(d, C::f_link_mass(d), j, w) : 0.0;
        rot[j] = (j < K) ? fld<C>(d, C::f_rotor(d), j, w) : 1.0;
        P.lm(j) = lm[j];
        P.rot(j) = rot[j];
        P.dmp(j) = (j < K) ? fld<C>(d, C::f_damping(d), j, w) : 0.0;
    }
    const double mt = P.base_mass() + np_sum<KM>(lm, K);
    P.m_total() = mt;
    P.inv_m() = 1.0 / mt;
    P.inv_inertia() = 1.0 / P.base_inertia();
#pragma unroll
    for (int j = 0; j < KM; ++j) P.inv_rot(j) = 1.0 / rot[j];
    if (actuators) {
        for_terms<C, C::kCapAct>(0, C::n_act(d), [&](auto aa) {
            const int a = ival(aa);
            if (C::act_kind(d, a) != SS_ACT_MLP) {
#pragma unroll
                for (int i = 0; i < KM; ++i) {
                    if (i < C::act_dim(d, a)) {
                        P.kp(a, i) = fld<C>(d, C::act_f_kp(d, a), i, w);
                        P.kd(a, i) = fld<C>(d, C::act_f_kd(d, a), i, w);
                    }
                }
            }
        });
    }
}

template <class C, int KM, int FM, class PP, int AS>
__device__ __forceinline__ void phys_substep(const ss_env_desc& d, int w, World<KM, FM, AS>& s, const PP& P) {
    const int K = C::K(d), F = C::F(d);
    const double friction = P.friction();

    // forward kinematics (fk_batch_trig, sim/physics.py:22-57)
    double sp, cp;
    if (s.trig_ok) {
        sp = s.sp;
        cp = s.cp;
    } else {
        ss_sincos(s.q[2], &sp, &cp);
    }
    double th[KM], st[KM], ct[KM], ax[KM], az[KM], tx[KM], tz[KM];
#pragma unroll
    for (int j = 0; j < KM; ++j) {
        th[j] = 0.0;
        if (j < K) {
            const int p = C::parent(d, j);
            double pa = s.q[2];
#pragma unroll
            for (int i = 0; i < j; ++i)
                if (p == i) pa = th[i];
            th[j] = pa + s.q[3 + j];
        }
    }
    ss_sincos_n<KM>(th, st, ct);  // th[j >= K] = 0: sin 0, cos 1 as before
#pragma unroll
    for (int j = 0; j < KM; ++j) {
        ax[j] = az[j] = tx[j] = tz[j] = 0.0;
        if (j < K) {
            const int p = C::parent(d, j);
            double sn = sp, c = cp, px = s.q[0], pz = s.q[1];
#pragma unroll
            for (int i = 0; i < j; ++i)
                if (p == i) {
                    sn = st[i];
                    c = ct[i];
                    px = ax[i];
                    pz = az[i];
                }
            const double ox = C::attach_x(d, j), oz = C::attach_z(d, j);
            ax[j] = px + (c * ox - sn * oz);
            az[j] = pz + (sn * ox + c * oz);
            tx[j] = ax[j] + C::link_len(d, j) * st[j];
            tz[j] = az[j] - C::link_len(d, j) * ct[j];
        }
    }

    // contact (compute_contact, sim/physics.py:75-111)
    double nfn[FM], nft[FM], nvx[FM], nvz[FM], npx[FM], npz[FM];
    bool ntouch[FM];
#pragma unroll
    for (int i = 0; i < FM; ++i) {
        nfn[i] = nft[i] = nvx[i] = nvz[i] = npx[i] = npz[i] = 0.0;
        ntouch[i] = false;
        if (i < F) {
            const int fj = C::foot(d, i);
            const unsigned mask = C::chain(d, i);
            const double px = sel(tx, fj), pz = sel(tz, fj);
            double vx = s.qd[0] - s.qd[2] * (pz - s.q[1]);
            double vz = s.qd[1] + s.qd[2] * (px - s.q[0]);
#pragma unroll
            for (int j = 0; j < KM; ++j) {
                if (j < K && ((mask >> j) & 1u)) {
                    vx -= s.qd[3 + j] * (pz - az[j]);
                    vz += s.qd[3 + j] * (px - ax[j]);
                }
            }
            const double phi = height<C>(d, px) - pz;
            const bool touching = phi > 0.0;
            double normal = np_max0(C::k_n(d) * phi - C::c_n(d) * vz);
            normal = touching ? normal : 0.0;
            const double bound = friction * normal;
            double tangent = np_clip(-C::k_t(d) * vx, -bound, bound);
            tangent = touching ? tangent : 0.0;
            nfn[i] = normal;
            nft[i] = tangent;
            nvx[i] = vx;
            nvz[i] = vz;
            npx[i] = px;
            npz[i] = pz;
            ntouch[i] = touching;
        }
    }

    // generalized forces (stage_forces, sim/physics.py:191-214)
    const double g = C::gravity(d);
    double tau[3 + KM];
    tau[0] = 0.0;
    tau[1] = 0.0;
    tau[2] = 0.0;
#pragma unroll
    for (int j = 0; j < KM; ++j) tau[3 + j] = 0.0 + s.ctrl[j];
#pragma unroll
    for (int j = 0; j < KM; ++j) tau[3 + j] = tau[3 + j] - P.dmp(j) * s.qd[3 + j];
    tau[1] = tau[1] - P.m_total() * g;
#pragma unroll
    for (int j = 0; j < KM; ++j) tau[3 + j] = tau[3 + j] - P.lm(j) * g * C::half_len(d, j) * st[j];
    tau[0] = tau[0] + s.ext0;
    tau[1] = tau[1] + s.ext1;
#pragma unroll
    for (int i = 0; i < FM; ++i) {
        if (i < F) {
            const double fx = nft[i], fz = nfn[i], px = npx[i], pz = npz[i];
            const unsigned mask = C::chain(d, i);
            tau[0] = tau[0] + fx;
            tau[1] = tau[1] + fz;
            tau[2] = tau[2] + ((px - s.q[0]) * fz - (pz - s.q[1]) * fx);
#pragma unroll
            for (int j = 0; j < KM; ++j)
                if (j < K && ((mask >> j) & 1u))
                    tau[3 + j] = tau[3 + j] + ((px - ax[j]) * fz - (pz - az[j]) * fx);
        }
    }
    s.ext0 = 0.0;
    s.ext1 = 0.0;

    // semi-implicit Euler (stage_integrate, sim/physics.py:216-224)
    tau[0] = tau[0] * P.inv_m();
    tau[1] = tau[1] * P.inv_m();
    tau[2] = tau[2] * P.inv_inertia();
#pragma unroll
    for (int j = 0; j < KM; ++j) tau[3 + j] = tau[3 + j] * P.inv_rot(j);
    const double dt = C::dt(d);
#pragma unroll
    for (int i = 0; i < 3 + KM; ++i)
        if (i < 3 + K) s.qd[i] = s.qd[i] + tau[i] * dt;
#pragma unroll
    for (int i = 0; i < 3 + KM; ++i)
        if (i < 3 + K) s.q[i] = s.q[i] + s.qd[i] * dt;

    // contact cache + clock (stage_finalize, sim/physics.py:226-235)
#pragma unroll
    for (int i = 0; i < FM; ++i) {
        s.fn[i] = nfn[i];
        s.ft[i] = nft[i];
        s.fvx[i] = nvx[i];
        s.fvz[i] = nvz[i];
        s.fpx[i] = npx[i];
        s.fpz[i] = npz[i];
        s.fin[i] = ntouch[i];
    }
    s.time = s.time + dt;
    s.trig_ok = false;
}

// ---------------------------------------------------------------------------
// actuators (Actuator.compute, actuators.py:279-316)

template <int KM, int FM>
__device__ __noinline__ double mlp_torque(const ss_env_desc& d, int a, int i, int w, double qdes, double qj,
                                          double qdj) {
    const ss_actuator& A = d.actuator[a];
    const int N = d.n_worlds;
    double x[2 * SS_MAX_HIST];
    for (int h = A.err_hist - 1; h >= 1; --h) {
        const double v = A.err_buf[((int64_t)(h - 1) * A.dim + i) * N + w];
        A.err_buf[((int64_t)h * A.dim + i) * N + w] = v;
        x[h] = v;
    }
    x[0] = qdes - qj;
    A.err_buf[(int64_t)i * N + w] = x[0];
    for (int h = A.vel_hist - 1; h >= 1; --h) {
        const double v = A.vel_buf[((int64_t)(h - 1) * A.dim + i) * N + w];
        A.vel_buf[((int64_t)h * A.dim + i) * N + w] = v;
        x[A.err_hist + h] = v;
    }
    x[A.err_hist] = qdj;
    A.vel_buf[(int64_t)i * N + w] = qdj;
    double buf0[32], buf1[32];
    const int n_in = A.err_hist + A.vel_hist;
    for (int k = 0; k < n_in; ++k) buf0[k] = x[k];
    double* cur = buf0;
    double* nxt = buf1;
    for (int l = 0; l < A.n_layers; ++l) {
        const ss_mlp_layer& L = A.layer[l];
        for (int o = 0; o < L.out_dim; ++o) {
            double acc = 0.0;
            for (int k = 0; k < L.in_dim; ++k) acc += cur[k] * __ldg(L.w + o * L.in_dim + k);
            acc = acc + __ldg(L.b + o);
            if (L.act == SS_MLP_RELU) acc = np_maximum(acc, 0.0);
            else if (L.act == SS_MLP_TANH) acc = tanh(acc);
            nxt[o] = acc;
        }
        double* t = cur;
        cur = nxt;
        nxt = t;
    }
    return np_clip(cur[0], -A.effort, A.effort);
}

template <class C, int KM, int FM, class PP, int AS>
__device__ __forceinline__ void apply_actuators(const ss_env_desc& d, const ss_uniforms& u, int w, int sub,
                                                World<KM, FM, AS>& s, const PP& P) {
    const int N = C::NW(d);
    for_terms<C, C::kCapAct>(0, C::n_act(d), [&](auto aa) {
        const int a = ival(aa);
        long long delay = 0;
        int head = 0;
        const int cap = C::act_cap(d, a);
        if (C::act_delayed(d, a)) {
            delay = d.actuator[a].delay_steps[w];
            head = (u.act_head0[a] + sub + 1) % cap;
        }
        const int kind = C::act_kind(d, a);
#pragma unroll
        for (int i = 0; i < KM; ++i) {
            if (i >= C::act_dim(d, a)) break;
            const int j = C::act_joint(d, a, i);
            double qdes = sel(s.targets, j);
            if (C::act_delayed(d, a)) {
                // DelayBuffer.push_and_read (actuators.py:208-213)
                double* ring = d.actuator[a].ring;
                const int dim = C::act_dim(d, a);
                ring[((int64_t)head * dim + i) * N + w] = qdes;
                int slot = (int)(((long long)head - delay) % cap);
                if (slot < 0) slot += cap;
                if (slot != head) qdes = ring[((int64_t)slot * dim + i) * N + w];
            }
            const double qj = sel(s.q, 3 + j), qdj = sel(s.qd, 3 + j);
            double tau;
            const double eff = C::act_effort(d, a);
            if (kind == SS_ACT_MLP) {
                tau = mlp_torque<KM, FM>(d, a, i, w, qdes, qj, qdj);
            } else {
                const double kp = P.kp(a, i), kd = P.kd(a, i);
                tau = kp * (qdes - qj) + kd * (0.0 - qdj);
                if (kind == SS_ACT_PD) {
                    tau = np_clip(tau, -eff, eff);
                } else {
                    // dc_motor_torque (actuators.py:110-117)
                    const double sat = C::act_sat(d, a), vl = C::act_vlim(d, a);
                    const double hi = np_clip(sat * (1.0 - qdj / vl), 0.0, eff);
                    const double lo = np_clip(sat * (-1.0 - qdj / vl), -eff, 0.0);
                    tau = np_clip(tau, lo, hi);
                }
            }
            sel_store(s.ctrl, j, tau);
        }
    });
}

// Actuator.reset (actuators.py:269-277) for one world
template <class C, int KM, class T>
__device__ __forceinline__ void reset_actuators(const ss_env_desc& d, int w, const T& targets) {
    const int N = C::NW(d);
    for (int a = 0; a < C::n_act(d); ++a) {
        const ss_actuator& A = d.actuator[a];
        if (C::act_delayed(d, a)) {
            const int dim = C::act_dim(d, a), cap = C::act_cap(d, a);
            for (int i = 0; i < dim; ++i) {
                const double v = sel(targets, C::act_joint(d, a, i));
                for (int h = 0; h < cap; ++h) A.ring[((int64_t)h * dim + i) * N + w] = v;
            }
            if (C::act_resample(d, a)) {
                double lat = C::act_lat_lo(d, a);
                if (!C::act_lat_const(d, a)) {
                    uint64_t key;
                    const int slot = C::act_lat_slot(d, a);
                    const uint64_t c = rng_begin(d, slot, w, key);
                    lat = uniform_from_word(stream_word(key, c, 0), C::act_lat_lo(d, a), C::act_lat_hi(d, a));
                    rng_end(d, slot, w, c + 1);
                }
                long long steps = (long long)rint(lat / C::dt(d));
                if (steps < 0) steps = 0;
                if (steps > cap - 1) steps = cap - 1;
                A.delay_steps[w] = steps;
            }
        }
        if (C::act_kind(d, a) == SS_ACT_MLP) {
            for (int i = 0; i < A.dim; ++i) {
                for (int h = 0; h < A.err_hist; ++h) A.err_buf[((int64_t)h * A.dim + i) * N + w] = 0.0;
                for (int h = 0; h < A.vel_hist; ++h) A.vel_buf[((int64_t)h * A.dim + i) * N + w] = 0.0;
            }
        }
    }
}

// ---------------------------------------------------------------------------
// events (mdp.py:186-220, managers/event.py:19-114)

template <class C>
__device__ __forceinline__ void randomize_world(const ss_env_desc& d, int w, int field, int dist, double r0,
                                                double r1, int op, int slot) {
    const int N = C::NW(d);
    const int size = C::fsize(d, field);
    double* ptr = d.field[field].ptr;
    uint64_t key;
    const uint64_t c = rng_begin(d, slot, w, key);
    for (int k = 0; k < size; ++k) {
        double draw;
        if (dist == SS_DIST_UNIFORM) draw = uniform_from_word(stream_word(key, c, k), r0, r1);
        else draw = r0 + normal_from_words(stream_word(key, c, k), stream_word(key, c, size + k), r1);
        const double base = C::fbase(d, field, k);
        double v = draw;
        if (op == SS_OP_SCALE) v = base * draw;
        else if (op == SS_OP_ADD) v = base + draw;
        ptr[(int64_t)k * N + w] = v;
    }
    rng_end(d, slot, w, c + (uint64_t)(dist == SS_DIST_UNIFORM ? size : 2 * size));
}

// EventManager._draw_targets for one world (managers/event.py:75-84)
template <class C>
__device__ __forceinline__ double draw_interval_target(const ss_env_desc& d, int e, int w) {
    uint64_t key;
    const int slot = C::ev_iv_slot(d, e);
    const uint64_t c = rng_begin(d, slot, w, key);
    const double draw = uniform_from_word(stream_word(key, c, 0), C::ev_iv_lo(d, e), C::ev_iv_hi(d, e));
    rng_end(d, slot, w, c + 1);
    const double dt = C::dt_control(d);
    const double quantized = rint(draw / dt) * dt;
    return np_clip(quantized, C::ev_iv_lo_q(d, e), C::ev_iv_hi_q(d, e));
}

template <class C, int KM, int FM, int AS>
__device__ __forceinline__ void apply_event(const ss_env_desc& d, int e, int w, World<KM, FM, AS>& s) {
    const int K = C::K(d);
    const int func = C::ev_func(d, e);
    if (func == SS_EVT_RANDOMIZE_FIELD) {
        randomize_world<C>(d, w, C::ev_field(d, e), C::ev_dist(d, e), C::ev_r0(d, e), C::ev_r1(d, e),
                           C::ev_op(d, e), C::ev_slot_a(d, e));
    } else if (func == SS_EVT_PUSH_BASE) {
        // push_base (mdp.py:201-211): fx then fz, one draw each per world
        uint64_t key;
        int slot = C::ev_slot_a(d, e);
        uint64_t c = rng_begin(d, slot, w, key);
        s.ext0 = s.ext0 + uniform_from_word(stream_word(key, c, 0), C::ev_r0(d, e), C::ev_r1(d, e));
        rng_end(d, slot, w, c + 1);
        slot = C::ev_slot_b(d, e);
        c = rng_begin(d, slot, w, key);
        s.ext1 = s.ext1 + uniform_from_word(stream_word(key, c, 0), C::ev_r2(d, e), C::ev_r3(d, e));
        rng_end(d, slot, w, c + 1);
    } else if (func == SS_EVT_JOINT_JITTER) {
        // reset_joints_jitter (mdp.py:214-220)
        uint64_t key;
        const int slot = C::ev_slot_a(d, e);
        const uint64_t c = rng_begin(d, slot, w, key);
#pragma unroll
        for (int j = 0; j < KM; ++j)
            if (j < K) s.q[3 + j] = s.q[3 + j] + uniform_from_word(stream_word(key, c, j), C::ev_r0(d, e), C::ev_r1(d, e));
        rng_end(d, slot, w, c + (uint64_t)K);
    }
}

// CommandManager.resample for one world (managers/command.py:33-39)
template <class C, int KM, int FM, int AS>
__device__ __forceinline__ void resample_command(const ss_env_desc& d, int w, World<KM, FM, AS>& s) {
    const int N = C::NW(d);
    uint64_t key;
    const int slot = C::cmd_slot(d);
    const uint64_t c = rng_begin(d, slot, w, key);
#pragma unroll
    for (int ch = 0; ch < SS_MAX_CMD; ++ch) {
        if (ch < C::n_cmd(d)) {
            const double lo = d.ranges[(int64_t)(2 * ch) * N + w];
            const double hi = d.ranges[(int64_t)(2 * ch + 1) * N + w];
            s.cmd[ch] = uniform_from_word(stream_word(key, c, ch), lo, hi);
            d.command[(int64_t)ch * N + w] = s.cmd[ch];
        }
    }
    rng_end(d, slot, w, c + (uint64_t)C::n_cmd(d));
    d.countdown[w] = C::period_steps(d);
}

// ---------------------------------------------------------------------------
// observation terms (mdp.py:26-89): raw values of term t into v[]

constexpr int kObsMax = SS_MAX_JOINTS > 2 * SS_MAX_FEET ? SS_MAX_JOINTS : 2 * SS_MAX_FEET;

template <class C, int KM, int FM, int AS>
__device__ __forceinline__ void obs_raw(const ss_env_desc& d, int t, int w, const World<KM, FM, AS>& s,
                                        double (&v)[kObsMax]) {
    const int N = C::NW(d), K = C::K(d), F = C::F(d);
    switch (C::obs_func(d, t)) {
        case SS_OBS_BASE_LIN_VEL:
            v[0] = s.lvb0;
            v[1] = s.lvb1;
            break;
        case SS_OBS_BASE_ANG_VEL:
            v[0] = s.eqd[2];
            break;
        case SS_OBS_BASE_LIN_ACC:
            v[0] = (s.lvb0 - s.plv0) / C::dt_control(d);
            v[1] = (s.lvb1 - s.plv1) / C::dt_control(d);
            break;
        case SS_OBS_PROJECTED_GRAVITY:
            v[0] = s.pg0;
            v[1] = s.pg1;
            break;
        case SS_OBS_JOINT_POS_REL:
#pragma unroll
            for (int j = 0; j < KM; ++j)
                if (j < K) v[j] = s.eq[3 + j] - C::joint_pos(d, j);
            break;
        case SS_OBS_JOINT_VEL:
#pragma unroll
            for (int j = 0; j < KM; ++j)
                if (j < K) v[j] = s.eqd[3 + j];
            break;
        case SS_OBS_LAST_ACTION:
#pragma unroll
            for (int k = 0; k < SS_MAX_ACTION; ++k)
                if (k < C::A(d)) v[k] = s.action[k];
            break;
        case SS_OBS_COMMAND:
#pragma unroll
            for (int c = 0; c < SS_MAX_CMD; ++c)
                if (c < C::n_cmd(d)) v[c] = s.cmd[c];
            break;
        case SS_OBS_BASE_HEIGHT:
            v[0] = s.q[1];
            break;
        case SS_OBS_SIM_TIME:
            v[0] = s.time;
            break;
        case SS_OBS_HEIGHT_SCAN: {
            // RayScanner.read (sensors.py:36-46): h(x_base + off) - z_base
            constexpr int NR = C::kJit ? C::kRays : SS_MAX_RAYS;
            double xr[NR], hr[NR];
#pragma unroll
            for (int r = 0; r < NR; ++r) xr[r] = s.eq[0] + (r < C::n_rays(d) ? C::ray_offset(d, r) : 0.0);
            height_raw_n<C, NR>(d, xr, hr);
#pragma unroll
            for (int r = 0; r < NR; ++r)
                if (r < C::n_rays(d)) v[r] = hr[r] - s.eq[1];
            break;
        }
        case SS_OBS_FOOT_CONTACT_FORCES:
#pragma unroll
            for (int i = 0; i < FM; ++i) {
                if (i < F) {
                    v[2 * i] = s.eft[i];
                    v[2 * i + 1] = s.efn[i];
                }
            }
            break;
        default: {  // SS_OBS_EXTERNAL: values of a registered Python term
            const int dim = C::obs_dim(d, t);
            for (int k = 0; k < dim; ++k) v[k] = d.obs[t].ext[(int64_t)w * dim + k];
        }
    }
}

// ObservationManager.compute, one term of one world (managers/observation.py:99-137)
template <class C, int KM, int FM, int AS>
__device__ __forceinline__ void obs_term(const ss_env_desc& d, const ss_uniforms& u, int t, int w,
                                         World<KM, FM, AS>& s, bool pending, double* out, unsigned& bad_bits) {
    const int N = C::NW(d);
    double v[kObsMax];
    obs_raw<C>(d, t, w, s, v);
    const int dim = C::obs_dim(d, t);
    const int col = C::obs_col(d, t);
    bool bad = false;
#pragma unroll
    for (int k = 0; k < kObsMax; ++k)
        if (k < dim) bad |= !finite_(v[k]);
    if (bad) bad_bits |= 1u << t;
    if (C::obs_has_clip(d, t)) {
#pragma unroll
        for (int k = 0; k < kObsMax; ++k)
            if (k < dim) v[k] = np_clip(v[k], C::obs_clip_lo(d, t), C::obs_clip_hi(d, t));
    }
    if (C::obs_has_scale(d, t)) {
#pragma unroll
        for (int k = 0; k < kObsMax; ++k)
            if (k < dim) v[k] = v[k] * C::obs_scale(d, t);
    }
    const int noise = C::obs_noise(d, t);
    if (noise != SS_NOISE_NONE) {
        const int slot = C::obs_noise_slot(d, t);
        const uint64_t key = stream_key(d.rng.base[slot], (uint64_t)(d.rng.world_id_offset + w));
        const uint64_t c = s.nctr[t];  // prefetched at kernel entry
        if (noise == SS_NOISE_UNIFORM) {
            const double hi = C::obs_noise_scale(d, t), lo = -hi;
#pragma unroll
            for (int k = 0; k < kObsMax; ++k)
                if (k < dim) v[k] = v[k] + uniform_from_word(stream_word(key, c, k), lo, hi);
            rng_end(d, slot, w, c + (uint64_t)dim);
        } else {
#pragma unroll
            for (int k = 0; k < kObsMax; ++k)
                if (k < dim)
                    v[k] = v[k] + normal_from_words(stream_word(key, c, k), stream_word(key, c, dim + k),
                                                    C::obs_noise_scale(d, t));
            rng_end(d, slot, w, c + (uint64_t)(2 * dim));
        }
    }
    const int D = C::obs_delay(d, t), H = C::obs_history(d, t);
    if (D == 0 && H == 1) {
#pragma unroll
        for (int k = 0; k < kObsMax; ++k)
            if (k < dim) out[col + k] = v[k];
        return;
    }
    // delay ring: push, then read D pushes back (flood on reset)
    if (D > 0) {
        double* ring = d.obs[t].delay_ring;
        const int D1 = D + 1;
        const int head = u.obs_delay_head[t];
        if (pending) {
            for (int h = 0; h < D1; ++h)
#pragma unroll
                for (int k = 0; k < kObsMax; ++k)
                    if (k < dim) ring[((int64_t)h * dim + k) * N + w] = v[k];
        } else {
#pragma unroll
            for (int k = 0; k < kObsMax; ++k)
                if (k < dim) ring[((int64_t)head * dim + k) * N + w] = v[k];
            int slot = (head - D) % D1;
            if (slot < 0) slot += D1;
#pragma unroll
            for (int k = 0; k < kObsMax; ++k)
                if (k < dim) v[k] = ring[((int64_t)slot * dim + k) * N + w];
        }
    }
    // history ring, oldest-first output (newest at the host-tracked head)
    if (H == 1) {
#pragma unroll
        for (int k = 0; k < kObsMax; ++k)
            if (k < dim) out[col + k] = v[k];
        return;
    }
    double* hr = d.obs[t].hist_ring;
    const int hh = u.obs_hist_head[t];
    if (pending) {
        for (int h = 0; h < H; ++h)
#pragma unroll
            for (int k = 0; k < kObsMax; ++k)
                if (k < dim) {
                    hr[((int64_t)h * dim + k) * N + w] = v[k];
                    out[col + h * dim + k] = v[k];
                }
    } else {
#pragma unroll
        for (int k = 0; k < kObsMax; ++k)
            if (k < dim) hr[((int64_t)hh * dim + k) * N + w] = v[k];
        for (int h = 0; h < H; ++h) {
            const int slot = (hh + 1 + h) % H;
#pragma unroll
            for (int k = 0; k < kObsMax; ++k)
                if (k < dim)
                    out[col + h * dim + k] = (slot == hh) ? v[k] : hr[((int64_t)slot * dim + k) * N + w];
        }
    }
}

// ---------------------------------------------------------------------------
// reward terms (mdp.py:96-160)

template <class C, int KM, int FM, int AS>
__device__ __forceinline__ double reward_value(const ss_env_desc& d, int r, int w, const World<KM, FM, AS>& s,
                                               long long sim_step_now) {
    const int K = C::K(d), F = C::F(d);
    switch (C::rew_func(d, r)) {
        case SS_REW_CONSTANT:
            return C::rew_p0(d, r);
        case SS_REW_BASE_HEIGHT:
            return s.q[1];
        case SS_REW_TRACK_VX_EXP: {
            const double err = s.cmd[0] - s.lvb0;
            const double sd = C::rew_p0(d, r);
            return exp(-(err * err) / (sd * sd));
        }
        case SS_REW_PITCH_RATE:
            return s.eqd[2] * s.eqd[2];
        case SS_REW_ANG_MOMENTUM: {
            const double m = fld<C>(d, C::f_base_inertia(d), 0, w) * s.eqd[2];
            return m * m;
        }
        case SS_REW_ACTION_RATE: {
            double sq[SS_MAX_ACTION];
#pragma unroll
            for (int k = 0; k < SS_MAX_ACTION; ++k) {
                const double dl = k < C::A(d) ? s.action[k] - s.prev_action[k] : 0.0;
                sq[k] = dl * dl;
            }
            return np_sum<SS_MAX_ACTION>(sq, C::A(d));
        }
        case SS_REW_JOINT_LIMIT: {
            double ex[KM];
#pragma unroll
            for (int j = 0; j < KM; ++j) {
                ex[j] = 0.0;
                if (j < K) {
                    const double lo = C::pos_lo(d, j), hi = C::pos_hi(d, j);
                    const double mid = 0.5 * (lo + hi);
                    const double soft_half = 0.5 * (hi - lo) * C::soft_frac(d, j);
                    ex[j] = np_max0(fabs(s.eq[3 + j] - mid) - soft_half);
                }
            }
            return np_sum<KM>(ex, K);
        }
        case SS_REW_FOOT_SLIP: {
            double sl[FM];
#pragma unroll
            for (int i = 0; i < FM; ++i) sl[i] = fabs(s.efvx[i]) * (s.efin[i] ? 1.0 : 0.0);
            return np_sum<FM>(sl, F);
        }
        case SS_REW_FEET_AIR_TIME: {
            double at[FM];
#pragma unroll
            for (int i = 0; i < FM; ++i) {
                const bool landed = s.s_td[i] > sim_step_now - C::decimation(d);
                at[i] = (s.s_last_air[i] - C::rew_p0(d, r)) * (landed ? 1.0 : 0.0);
            }
            return np_sum<FM>(at, F);
        }
        default:
            return d.reward[r].ext[w];
    }
}

// ---------------------------------------------------------------------------
// the fused step body

#ifdef SS_PROBES
#define SS_PROBE(i)                                       \
    do {                                                  \
        if (w == 0 && d.probe) d.probe[i] = clock64();    \
    } while (0)
__device__ __forceinline__ long long gtimer() {
    long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
#define SS_PROBE_SPAN(first)                                                                       \
    do {                                                                                           \
        if (d.probe && (threadIdx.x & 31) == 0) {                                                  \
            if (first) atomicMin((unsigned long long*)&d.probe[14], (unsigned long long)gtimer()); \
            else atomicMax((unsigned long long*)&d.probe[15], (unsigned long long)gtimer());       \
        }                                                                                          \
    } while (0)
#else
#define SS_PROBE_SPAN(first) \
    do {                     \
    } while (0)
#define SS_PROBE(i) \
    do {            \
    } while (0)
#endif

// FS != 0 compiles the body for exactly that stage set (the split launch of large
// envs: physics | terms + observations, each kernel with ~40 registers fewer
// than the whole body); FS == 0 takes the set from u.stages.
template <class C, int KM, int FM, unsigned FS = 0>
__device__ __forceinline__ void step_body(const ss_env_desc& d, const ss_uniforms& u) {
    const int N = C::NW(d);
    if ((int)(blockIdx.x * blockDim.x) >= N) return;  // padding block (grid rounded up to fill the SMs)
    const int w = blockIdx.x * blockDim.x + threadIdx.x;
    const bool active = w < N;
    const unsigned st = FS ? FS : u.stages;  // FS: a kernel compiled for one fixed stage set
    double stat_reward = 0.0;  // this step's reward of world w (the fused statistics, stats_tail)
    const int K = C::K(d), F = C::F(d), A = C::A(d);
    // Observation rows are staged in shared memory and leave the block as one
    // contiguous bulk copy per group (TMA, cp.async.bulk) instead of 32-way
    // scattered row stores (specialized builds whose groups fit 48 KB).
    // staging buffers: static shared memory, or one dynamic block (C::kDynSmem bytes, the layout
    // C::kDynObs / kDynParam / kDynAct in doubles) when together they exceed the 48 KB static limit
    // a fixed-stage kernel allocates only the staging its stages use (FS: step_body)
    constexpr bool kObsUsed = FS == 0 || (FS & SS_ST_OBS);
    __shared__ __align__(16) double
        obs_stage_s[(C::kStageObs && !C::kDynSmem && kObsUsed) ? C::kBlock * C::kObsTotal : 2];
    double* const obs_stage = C::kDynSmem ? dyn_smem() + C::kDynObs : obs_stage_s;
    SS_PROBE_SPAN(1);
    // JIT builds of large models keep the action / target vectors and the episodic sums in
    // shared-memory columns (Col): [action A][prev action A][targets K][ep_sum R][ep_raw R]
    constexpr int AS = C::kActSmem ? C::kBlock : 0;
    constexpr int NCOL = 2 * SS_DCAP_ACTION_COLS + KM + 2 * SS_DCAP_REWARDS;
    __shared__ double act_cols_s[(AS && !C::kDynSmem) ? NCOL * AS : 1];
    double* const act_cols = C::kDynSmem ? dyn_smem() + C::kDynAct : act_cols_s;
    World<KM, FM, AS> s;
    s.action.p = act_cols + threadIdx.x;
    s.prev_action.p = act_cols + SS_DCAP_ACTION_COLS * AS + threadIdx.x;
    s.targets.p = act_cols + 2 * SS_DCAP_ACTION_COLS * AS + threadIdx.x;
    s.ep_sum.p = act_cols + (2 * SS_DCAP_ACTION_COLS + KM) * AS + threadIdx.x;
    s.ep_rw.p = act_cols + (2 * SS_DCAP_ACTION_COLS + KM + SS_DCAP_REWARDS) * AS + threadIdx.x;
#pragma unroll
    for (int k = 0; k < SS_MAX_ACTION; ++k) {
        if (!AS || k < SS_DCAP_ACTION_COLS) s.action[k] = s.prev_action[k] = 0.0;
    }
    s.trig_bits = 0;
    s.terminated = s.truncated = s.nonfinite = s.was_reset = false;

    if (active) {
        const bool sim = (st & (SS_ST_APPLY | SS_ST_PUSH | SS_ST_PHYS | SS_ST_SENSOR)) && u.nsub > 0;
        const bool phys = (st & SS_ST_PHYS) && u.nsub > 0;
        const bool resets = st & (SS_ST_RESET | SS_ST_RESET_ALL);
        SS_PROBE(0);

        // ---- prefetch: every per-step array this launch will read, issued up
        // front so their DRAM latency overlaps (the stores that follow would
        // otherwise pin each load behind them: the pointers may alias)
        load_phys<C>(d, w, s, /*load_cache=*/!phys);
#pragma unroll
        for (int c = 0; c < SS_MAX_CMD; ++c) s.cmd[c] = (c < C::n_cmd(d)) ? d.command[(int64_t)c * N + w] : 0.0;
        const bool need_targets = st & (SS_ST_ACTION | SS_ST_APPLY | SS_ST_RESET | SS_ST_RESET_ALL);
#pragma unroll
        for (int j = 0; j < KM; ++j) s.targets[j] = (need_targets && j < K) ? d.targets[(int64_t)j * N + w] : 0.0;
        s.have_action = false;
        s.have_sensor = false;
        // per-step arrays used only after the substeps: loaded just before the
        // last substep (latency hidden behind it, registers not held through
        // the whole physics loop)
        auto late_prefetch = [&]() {
            if (st & (SS_ST_TERM | SS_ST_CURRICULUM)) {
                s.ep_steps = d.episode_steps[w];
                s.cmd_dist = d.commanded_distance[w];
            }
            if (st & (SS_ST_REWARD | SS_ST_CURRICULUM | SS_ST_RESET | SS_ST_RESET_ALL)) {
                for_terms<C, C::kCapRewards>(0, C::n_rewards(d), [&](auto rr) {
                    const int r = ival(rr);
                    s.ep_sum[r] = d.ep_sums[(int64_t)r * N + w];
                    s.ep_rw[r] = d.ep_raw[(int64_t)r * N + w];
                });
            }
            if ((st & SS_ST_COMMAND) && C::n_cmd(d) > 0) s.countdown = d.countdown[w];
            if (st & SS_ST_EVENTS) {
                for_terms<C, C::kCapEvents>(0, C::n_events(d), [&](auto ee) {
                    const int e = ival(ee);
                    if (C::ev_mode(d, e) == SS_MODE_INTERVAL) {
                        s.ev_el[e] = d.event[e].elapsed[w];
                        s.ev_tg[e] = d.event[e].target[w];
                    }
                });
            }
            if (st & SS_ST_OBS) {
                for_terms<C, C::kCapObs>(0, C::n_obs(d), [&](auto tt) {
                    const int t = ival(tt);
                    if (C::obs_noise(d, t) != SS_NOISE_NONE) s.nctr[t] = d.rng.counter[C::obs_noise_slot(d, t)][w];
                });
                s.plv0 = d.prev_lin_vel_b[w];
                s.plv1 = d.prev_lin_vel_b[N + w];
            }
        };
        // the heightfield (38 KB for the rough grid): one 128 B line per thread
        // of the first threads, so the feet's first lookups hit L2
        if (!C::flat(d) && (st & (SS_ST_PHYS | SS_ST_OBS | SS_ST_RESET | SS_ST_RESET_ALL))) {
            const int line = w;  // w < N here
            if ((int64_t)line * 16 < d.terrain.n_samples) l2_prefetch(d.terrain.samples + (int64_t)line * 16);
        }
        // L2 prefetch of everything read after the substeps or on the reset path
        if (st & (SS_ST_TERM | SS_ST_CURRICULUM)) {
            late_prefetch_line(d.episode_steps + w);
            late_prefetch_line(d.commanded_distance + w);
        }
        if (st & SS_ST_CURRICULUM) late_prefetch_line(d.episode_start_x + w);
        if (st & (SS_ST_REWARD | SS_ST_CURRICULUM | SS_ST_RESET | SS_ST_RESET_ALL)) {
            for_terms<C, C::kCapRewards>(0, C::n_rewards(d), [&](auto rr) {
                late_prefetch_line(d.ep_sums + (int64_t)ival(rr) * N + w);
                late_prefetch_line(d.ep_raw + (int64_t)ival(rr) * N + w);
            });
        }
        if ((st & (SS_ST_COMMAND | SS_ST_RESET | SS_ST_RESET_ALL)) && C::n_cmd(d) > 0) {
            late_prefetch_line(d.countdown + w);
            late_prefetch_line(d.rng.counter[C::cmd_slot(d)] + w);
            for (int c = 0; c < 2 * C::n_cmd(d); ++c) late_prefetch_line(d.ranges + (int64_t)c * N + w);
        }
        if (st & (SS_ST_EVENTS | SS_ST_RESET | SS_ST_RESET_ALL)) {
            for_terms<C, C::kCapEvents>(0, C::n_events(d), [&](auto ee) {
                const int e = ival(ee);
                if (C::ev_mode(d, e) == SS_MODE_INTERVAL) {
                    late_prefetch_line(d.event[e].elapsed + w);
                    late_prefetch_line(d.event[e].target + w);
                    late_prefetch_line(d.rng.counter[C::ev_iv_slot(d, e)] + w);
                }
                if (C::ev_mode(d, e) != SS_MODE_STARTUP && C::ev_func(d, e) != SS_EVT_EXTERNAL) {
                    late_prefetch_line(d.rng.counter[C::ev_slot_a(d, e)] + w);
                    if (C::ev_func(d, e) == SS_EVT_PUSH_BASE) late_prefetch_line(d.rng.counter[C::ev_slot_b(d, e)] + w);
                }
            });
        }
        if (st & SS_ST_OBS) {
            for_terms<C, C::kCapObs>(0, C::n_obs(d), [&](auto tt) {
                const int t = ival(tt);
                if (C::obs_noise(d, t) != SS_NOISE_NONE) late_prefetch_line(d.rng.counter[C::obs_noise_slot(d, t)] + w);
            });
            late_prefetch_line(d.prev_lin_vel_b + w);
            late_prefetch_line(d.prev_lin_vel_b + N + w);
        }
        if (resets) {
            late_prefetch_line(d.terrain_rows + w);
            late_prefetch_line(d.terrain_cols + w);
        }
        // action inputs and contact-sensor state: loaded here, ahead of the
        // ACTION stage's stores (which would otherwise order them behind)
        uint64_t pol_key = 0, pol_c = 0;
        if (st & SS_ST_ACTION) {
#pragma unroll
            for (int k = 0; k < SS_MAX_ACTION; ++k)
                if (k < A) s.prev_action[k] = d.action[(int64_t)k * N + w];
            if (u.policy_slot >= 0) {
                pol_c = rng_begin(d, u.policy_slot, w, pol_key);
            } else {
                const double* a = u.actions + (int64_t)w * A;
#pragma unroll
                for (int k = 0; k < SS_MAX_ACTION; ++k)
                    if (k < A) s.action[k] = a[k];
            }
        }
        if (sim && (st & SS_ST_SENSOR)) {
#pragma unroll
            for (int i = 0; i < FM; ++i) {
                const bool ok = i < F;
                s.s_in[i] = ok ? d.s_in_contact[(int64_t)i * N + w] != 0 : false;
                s.s_air[i] = ok ? d.s_cur_air[(int64_t)i * N + w] : 0.0;
                s.s_last_air[i] = ok ? d.s_last_air[(int64_t)i * N + w] : 0.0;
                s.s_contact[i] = ok ? d.s_cur_contact[(int64_t)i * N + w] : 0.0;
                s.s_td[i] = ok ? d.s_last_td[(int64_t)i * N + w] : kNeverTouched;
            }
            // the force history is fully overwritten when >= H updates run
            const int H = C::hist_len(d);
            const int n_upd = __popc(u.sensor_mask & ((1u << u.nsub) - 1u));
            const bool need_hist = n_upd < H;
#pragma unroll
            for (int h = 0; h < SS_MAX_HIST; ++h)
#pragma unroll
                for (int i = 0; i < FM; ++i)
                    s.s_hist[h][i] = (need_hist && h < H && i < F) ? d.s_force_hist[((int64_t)h * F + i) * N + w] : 0.0;
        }
        // JIT: the hoisted model fields live in a shared-memory column (Params, S = kBlock)
        // (the physics-only kernel of a split env has no observation staging beside them: kParamSmemAlone)
        constexpr bool kParUsed = FS == 0 || (FS & (SS_ST_PHYS | SS_ST_APPLY));
        constexpr bool kParSmem = C::kParamSmem || (FS != 0 && !(FS & SS_ST_OBS) && C::kParamSmemAlone);
        constexpr int PS = (kParSmem && kParUsed) ? C::kBlock : 0;
        using PT = Params<KM, C::kCapAct, PS>;
        __shared__ double param_cols_s[(PS && !(C::kDynSmem && C::kParamSmem)) ? PT::NV * PS : 1];
        double* const param_cols = (C::kDynSmem && C::kParamSmem) ? dyn_smem() + C::kDynParam : param_cols_s;
        PT P;
        P.p = param_cols + threadIdx.x;
        if (sim && (st & (SS_ST_PHYS | SS_ST_APPLY))) load_params<C, KM>(d, w, P, st & SS_ST_APPLY);
        if (!phys) refresh(s);  // staged launch: entity data from the stored state
        SS_PROBE(1);

        // ---- 1. ActionManager.process (managers/action.py:68-82)
        if (st & SS_ST_ACTION) {
            if (u.policy_slot >= 0) {
                // fused random_policy (policies.py:14-16): U[lo, hi) from the
                // policy stream, the same words ss_rng_draw would produce
#pragma unroll
                for (int k = 0; k < SS_MAX_ACTION; ++k)
                    if (k < A) s.action[k] = uniform_from_word(stream_word(pol_key, pol_c, k), u.policy_lo, u.policy_hi);
                rng_end(d, u.policy_slot, w, pol_c + (uint64_t)A);
            }
#pragma unroll
            for (int k = 0; k < SS_MAX_ACTION; ++k) {
                if (k < A) {
                    d.prev_action[(int64_t)k * N + w] = s.prev_action[k];
                    d.action[(int64_t)k * N + w] = s.action[k];
                }
            }
            for_terms<C, C::kCapActTerms>(0, C::n_action_terms(d), [&](auto tt) {
                const int t = ival(tt);
#pragma unroll
                for (int i = 0; i < KM; ++i) {
                    if (i >= C::at_dim(d, t)) break;
                    double x = sel(s.action, C::at_start(d, t) + i);
                    if (C::at_has_clip(d, t)) x = np_clip(x, C::at_clip_lo(d, t), C::at_clip_hi(d, t));
                    sel_store(s.targets, C::at_joint(d, t, i), C::at_offset(d, t, i) + C::at_scale(d, t) * x);
                }
            });
#pragma unroll
            for (int j = 0; j < KM; ++j)
                if (j < K) d.targets[(int64_t)j * N + w] = s.targets[j];
            s.have_action = true;
        }

        SS_PROBE(2);
        // ---- 2. decimation substeps (env.py:228-233)
        if (sim) {
            const bool sensor = st & SS_ST_SENSOR;
            const int H = C::hist_len(d);
            if (sensor) s.have_sensor = true;  // state loaded with the prefetch block
            const int nsub = u.nsub;
            auto substep = [&](int sub) {
                if (st & SS_ST_APPLY) apply_actuators<C>(d, u, w, sub, s, P);
                if (st & SS_ST_PUSH) {
                    // CaptureRing.push (capture.py:53-59): ctrl written, pre-integration
                    // capture_slot0 < capture_phys and sub < nsub <= capture_phys
                    int slot = u.capture_slot0 + sub;
                    if (slot >= C::cap_phys(d)) slot -= C::cap_phys(d);
                    const int nq = 3 + K;
#pragma unroll
                    for (int i = 0; i < 3 + KM; ++i) {
                        if (i < nq) {
                            d.cap_q[((int64_t)slot * nq + i) * N + w] = s.q[i];
                            d.cap_qd[((int64_t)slot * nq + i) * N + w] = s.qd[i];
                        }
                    }
#pragma unroll
                    for (int j = 0; j < KM; ++j)
                        if (j < K) d.cap_ctrl[((int64_t)slot * K + j) * N + w] = s.ctrl[j];
                }
                if (phys) {
                    phys_substep<C>(d, w, s, P);
                    refresh(s);
                }
                if (sensor && ((u.sensor_mask >> sub) & 1u)) {
                    // ContactSensor.update (sensors.py:91-115)
                    const long long now_step = u.sim_step + sub + (phys ? 1 : 0);
                    const double dt = C::dt(d);
#pragma unroll
                    for (int i = 0; i < FM; ++i) {
                        if (i < F) {
                            const bool now = s.fin[i], prev = s.s_in[i];
                            const bool td = now && !prev;
                            const bool lo = !now && prev;
                            s.s_last_air[i] = td ? s.s_air[i] : s.s_last_air[i];
                            s.s_td[i] = td ? now_step : s.s_td[i];
                            s.s_contact[i] = now ? (td ? dt : s.s_contact[i] + dt) : 0.0;
                            s.s_air[i] = now ? 0.0 : (lo ? dt : s.s_air[i] + dt);
                            s.s_in[i] = now;
                        }
                    }
#pragma unroll
                    for (int h = SS_MAX_HIST - 1; h >= 1; --h)
#pragma unroll
                        for (int i = 0; i < FM; ++i)
                            if (h < H) s.s_hist[h][i] = s.s_hist[h - 1][i];
#pragma unroll
                    for (int i = 0; i < FM; ++i) s.s_hist[0][i] = s.fn[i];
                }
                SS_PROBE(3 + (sub < 3 ? sub : 3));
            };
#if SS_PEEL_LAST_SUBSTEP
#pragma unroll 1
            for (int sub = 0; sub < nsub - 1; ++sub) substep(sub);
            late_prefetch();
            substep(nsub - 1);
#else
            // one copy of the substep body in the code; the late loads follow
            // the loop (their lines were pulled into L2 at kernel entry)
#pragma unroll 1
            for (int sub = 0; sub < nsub; ++sub) substep(sub);
            late_prefetch();
#endif
            if (sensor) {
#pragma unroll
                for (int i = 0; i < FM; ++i) {
                    if (i < F) {
                        d.s_in_contact[(int64_t)i * N + w] = s.s_in[i] ? 1 : 0;
                        d.s_normal[(int64_t)i * N + w] = s.fn[i];
                        d.s_tangent[(int64_t)i * N + w] = s.ft[i];
                        d.s_cur_air[(int64_t)i * N + w] = s.s_air[i];
                        d.s_last_air[(int64_t)i * N + w] = s.s_last_air[i];
                        d.s_cur_contact[(int64_t)i * N + w] = s.s_contact[i];
                        d.s_last_td[(int64_t)i * N + w] = s.s_td[i];
                    }
                }
#pragma unroll
                for (int h = 0; h < SS_MAX_HIST; ++h)
#pragma unroll
                    for (int i = 0; i < FM; ++i)
                        if (h < H && i < F) d.s_force_hist[((int64_t)h * F + i) * N + w] = s.s_hist[h][i];
            }
        }
        SS_PROBE(7);
        if (!sim) late_prefetch();
        const long long sim_step_now = u.sim_step + (phys ? u.nsub : 0);

        // ---- 3. episode bookkeeping + TerminationManager.compute (env.py:235-239)
        if (st & SS_ST_TERM) {
            if (!(u.flags & SS_FLAG_NO_EPISODE)) {
                s.ep_steps += 1;
                if (C::n_cmd(d) > 0) s.cmd_dist = s.cmd_dist + fabs(s.cmd[0]) * C::dt_control(d);
                d.episode_steps[w] = s.ep_steps;
                d.commanded_distance[w] = s.cmd_dist;
            }
            bool term = false, trunc = false;
            for_terms<C, C::kCapTerms>(0, C::n_terms(d), [&](auto tt) {
                const int t = ival(tt);
                const int f = C::term_func(d, t);
                bool m;
                if (f == SS_TERM_BASE_HEIGHT_BELOW) m = s.q[1] < C::term_p0(d, t);
                else if (f == SS_TERM_PITCH_BEYOND) m = fabs(s.q[2]) > C::term_p0(d, t);
                else if (f == SS_TERM_TIME_OUT) m = s.ep_steps >= C::max_episode_steps(d);
                else m = d.term[t].ext[w] != 0;
                if (m) s.trig_bits |= 1u << t;
                if (C::term_time_out(d, t)) trunc |= m;
                else term |= m;
            });
            // detect_nonfinite over q, qd, ctrl (sim/state.py:69-74)
            bool bad = false;
#pragma unroll
            for (int i = 0; i < 3 + KM; ++i)
                if (i < 3 + K) bad |= !finite_(s.q[i]) || !finite_(s.qd[i]);
#pragma unroll
            for (int j = 0; j < KM; ++j)
                if (j < K) bad |= !finite_(s.ctrl[j]);
            if (bad) s.trig_bits |= 1u << 31;
            term |= bad;
            s.terminated = term;
            s.truncated = trunc;
            s.nonfinite = bad;
            d.terminated[w] = term;
            d.truncated[w] = trunc;
            if (C::mirror_on(d)) {
                *mirror_of(d, d.terminated + w) = term;
                *mirror_of(d, d.truncated + w) = trunc;
            }
            d.nonfinite[(int64_t)u.nf_slot * N + w] = bad;  // per-step slot of the lag ring
        }

        SS_PROBE(8);
        auto ensure_action = [&]() {
            if (!s.have_action) {
#pragma unroll
                for (int k = 0; k < SS_MAX_ACTION; ++k) {
                    if (k < A) {
                        s.action[k] = d.action[(int64_t)k * N + w];
                        s.prev_action[k] = d.prev_action[(int64_t)k * N + w];
                    }
                }
                s.have_action = true;
            }
        };
        auto ensure_sensor = [&]() {
            if (!s.have_sensor) {
#pragma unroll
                for (int i = 0; i < FM; ++i) {
                    s.s_last_air[i] = (i < F) ? d.s_last_air[(int64_t)i * N + w] : 0.0;
                    s.s_td[i] = (i < F) ? d.s_last_td[(int64_t)i * N + w] : kNeverTouched;
                }
                s.have_sensor = true;
            }
        };

        // ---- 4. RewardManager.compute (managers/reward.py:36-49), pre-reset state
        if (st & SS_ST_REWARD) {
            ensure_action();
            ensure_sensor();
            double total = 0.0;
            for_terms<C, C::kCapRewards>(0, C::n_rewards(d), [&](auto rr) {
                const int r = ival(rr);
                const double v = reward_value<C>(d, r, w, s, sim_step_now);
                const double contribution = u.weight[r] * v * C::dt_control(d);
                total += contribution;
                s.ep_sum[r] = s.ep_sum[r] + contribution;
                s.ep_rw[r] = s.ep_rw[r] + v;
                d.last_values[(int64_t)r * N + w] = v;
            });
            d.reward_out[w] = total;
            stat_reward = total;
            if (C::mirror_on(d)) *mirror_of(d, d.reward_out + w) = total;
        }

        SS_PROBE(9);
        // ---- 5. curriculum on the finished episode, then masked reset (env.py:245-250)
        bool selected = false;
        if (st & SS_ST_RESET_ALL) selected = true;
        else if (st & (SS_ST_RESET | SS_ST_CURRICULUM)) {
            if (st & SS_ST_RESET_EXT) selected = u.reset_mask[w] != 0;
            else if (st & SS_ST_TERM) selected = s.terminated || s.truncated;
            else selected = d.terminated[w] || d.truncated[w];
        }
        const bool do_reset = selected && resets;
        if (selected && (st & SS_ST_CURRICULUM)) {
            for (int c = 0; c < C::n_curr(d); ++c) {
                if (C::cur_func(d, c) == SS_CUR_TERRAIN_LEVELS) {
                    // terrain_levels (mdp.py:227-243)
                    const double walked = fabs(s.q[0] - d.episode_start_x[w]);
                    const double commanded = s.cmd_dist;
                    long long row = d.terrain_rows[w];
                    if (walked >= C::cur_p0(d, c) * commanded) row = row + 1;
                    if (walked <= C::cur_p1(d, c) * commanded) row = row - 1;
                    if (row < 0) row = 0;
                    if (row > d.terrain.rows - 1) row = d.terrain.rows - 1;
                    d.terrain_rows[w] = row;
                } else if (C::cur_func(d, c) == SS_CUR_COMMAND_WIDEN) {
                    // command_widen (mdp.py:246-259) -> CommandManager.widen (command.py:47-50)
                    const double steps = (double)s.ep_steps;
                    double raw = 0.0;
                    for_terms<C, C::kCapRewards>(0, C::n_rewards(d), [&](auto rr) {
                        if (ival(rr) == C::cur_term(d, c)) raw = s.ep_rw[ival(rr)];
                    });
                    const double mean = raw / (steps > 1.0 ? steps : 1.0);
                    if (mean > C::cur_p0(d, c)) {
                        for (int ch = 0; ch < C::n_cmd(d); ++ch) {
                            const double blo = fabs(C::init_lo(d, ch)) * C::cap_scale(d);
                            const double bhi = fabs(C::init_hi(d, ch)) * C::cap_scale(d);
                            double* rlo = d.ranges + (int64_t)(2 * ch) * N + w;
                            double* rhi = d.ranges + (int64_t)(2 * ch + 1) * N + w;
                            *rlo = np_clip(*rlo * C::cur_p1(d, c), -blo, blo);
                            *rhi = np_clip(*rhi * C::cur_p1(d, c), -bhi, bhi);
                        }
                    }
                }
            }
        }
        if (do_reset) {
            s.was_reset = true;
            // write_default_state (entity.py:91-105)
#pragma unroll
            for (int i = 0; i < 3; ++i) {
                s.q[i] = C::base_pose(d, i);
                s.qd[i] = C::base_vel(d, i);
            }
#pragma unroll
            for (int j = 0; j < KM; ++j) {
                s.q[3 + j] = (j < K) ? C::joint_pos(d, j) : 0.0;
                s.qd[3 + j] = (j < K) ? C::joint_vel(d, j) : 0.0;
            }
            s.time = 0.0;
            // _place_on_terrain (env.py:171-180)
            {
                const long long row = d.terrain_rows[w], col = d.terrain_cols[w];
                const double origin = (double)(row * d.terrain.cols + col) * d.terrain.patch_length;
                const double spawn_x = origin + C::spawn_offset(d);
                s.q[0] = s.q[0] + spawn_x;
                s.q[1] = s.q[1] + height_raw(d, spawn_x);
            }
            // EventManager.apply_reset (managers/event.py:92-101)
            for_terms<C, C::kCapEvents>(0, C::n_events(d), [&](auto ee) {
                const int e = ival(ee);
                const int mode = C::ev_mode(d, e);
                if (mode == SS_MODE_RESET && C::ev_func(d, e) != SS_EVT_EXTERNAL) {
                    apply_event<C>(d, e, w, s);
                } else if (mode == SS_MODE_INTERVAL) {
                    s.ev_el[e] = 0.0;
                    s.ev_tg[e] = draw_interval_target<C>(d, e, w);
                    if (!(st & SS_ST_EVENTS)) {
                        d.event[e].elapsed[w] = 0.0;
                        d.event[e].target[w] = s.ev_tg[e];
                    }
                }
            });
            // CommandManager.resample
            if (C::n_cmd(d) > 0) {
                resample_command<C>(d, w, s);
                s.countdown = C::period_steps(d);
            }
            // ActionManager.reset (managers/action.py:92-97)
#pragma unroll
            for (int k = 0; k < SS_MAX_ACTION; ++k) {
                if (k < A) {
                    s.action[k] = 0.0;
                    s.prev_action[k] = 0.0;
                    d.action[(int64_t)k * N + w] = 0.0;
                    d.prev_action[(int64_t)k * N + w] = 0.0;
                }
            }
            s.have_action = true;
            for_terms<C, C::kCapActTerms>(0, C::n_action_terms(d), [&](auto tt) {
                const int t = ival(tt);
#pragma unroll
                for (int i = 0; i < KM; ++i) {
                    if (i >= C::at_dim(d, t)) break;
                    sel_store(s.targets, C::at_joint(d, t, i), C::at_offset(d, t, i));
                }
            });
#pragma unroll
            for (int j = 0; j < KM; ++j)
                if (j < K) d.targets[(int64_t)j * N + w] = s.targets[j];
            reset_actuators<C, KM>(d, w, s.targets);
            // ContactSensor.reset (sensors.py:81-89)
#pragma unroll
            for (int i = 0; i < FM; ++i) {
                s.s_last_air[i] = 0.0;
                s.s_td[i] = kNeverTouched;
                if (i < F) {
                    d.s_in_contact[(int64_t)i * N + w] = 0;
                    d.s_normal[(int64_t)i * N + w] = 0.0;
                    d.s_tangent[(int64_t)i * N + w] = 0.0;
                    d.s_cur_air[(int64_t)i * N + w] = 0.0;
                    d.s_last_air[(int64_t)i * N + w] = 0.0;
                    d.s_cur_contact[(int64_t)i * N + w] = 0.0;
                    d.s_last_td[(int64_t)i * N + w] = kNeverTouched;
                    for (int h = 0; h < C::hist_len(d); ++h) d.s_force_hist[((int64_t)h * F + i) * N + w] = 0.0;
                }
            }
            s.have_sensor = true;
            // contact cache (env.py:194-198): foot_pos is kept
#pragma unroll
            for (int i = 0; i < FM; ++i) {
                s.fn[i] = 0.0;
                s.ft[i] = 0.0;
                s.fvx[i] = 0.0;
                s.fvz[i] = 0.0;
                s.fin[i] = false;
            }
            // RewardManager.reset (managers/reward.py:55-62)
            for_terms<C, C::kCapRewards>(0, C::n_rewards(d), [&](auto rr) {
                const int r = ival(rr);
                d.finalized[(int64_t)r * N + w] = s.ep_sum[r];
                s.ep_sum[r] = 0.0;
                s.ep_rw[r] = 0.0;
            });
            s.ep_steps = 0;
            s.cmd_dist = 0.0;
            d.episode_steps[w] = 0;
            d.episode_start_x[w] = s.q[0];
            d.commanded_distance[w] = 0.0;
            refresh(s);
            if (!(st & SS_ST_OBS))
                for (int g = 0; g < C::n_groups(d); ++g) d.group[g].pending[w] = 1;
        }
        if (st & (SS_ST_REWARD | SS_ST_RESET | SS_ST_RESET_ALL)) {
            // episodic sums: one store each, after the reward update and the reset finalize
            for_terms<C, C::kCapRewards>(0, C::n_rewards(d), [&](auto rr) {
                const int r = ival(rr);
                if ((st & SS_ST_REWARD) || do_reset) {
                    d.ep_sums[(int64_t)r * N + w] = s.ep_sum[r];
                    d.ep_raw[(int64_t)r * N + w] = s.ep_rw[r];
                }
            });
        }

        SS_PROBE(10);
        // ---- 6. CommandManager.update (managers/command.py:41-45)
        if ((st & SS_ST_COMMAND) && C::n_cmd(d) > 0) {
            const long long cd = s.countdown - 1;
            if (cd <= 0) resample_command<C>(d, w, s);
            else d.countdown[w] = cd;
        }

        // ---- 7. EventManager.apply_interval (managers/event.py:103-114)
        if (st & SS_ST_EVENTS) {
            for_terms<C, C::kCapEvents>(0, C::n_events(d), [&](auto ee) {
                const int e = ival(ee);
                if (C::ev_mode(d, e) != SS_MODE_INTERVAL) return;
                double el = s.ev_el[e] + C::dt_control(d);
                const double tgt = s.ev_tg[e];
                const bool fire = el >= tgt - 0.5 * C::dt_control(d);
                if (fire) {
                    // registered Python terms run on the host for the fired ids
                    if (C::ev_func(d, e) != SS_EVT_EXTERNAL) apply_event<C>(d, e, w, s);
                    el = 0.0;
                    s.ev_tg[e] = draw_interval_target<C>(d, e, w);
                }
                if (fire || s.was_reset) d.event[e].target[w] = s.ev_tg[e];
                if (d.event[e].fired) d.event[e].fired[w] = fire;
                d.event[e].elapsed[w] = el;
            });
        }

        SS_PROBE(11);
        // ---- 8. observations (post-reset state) (managers/observation.py:139-141)
        if (st & SS_ST_PREV_BEFORE) {
            d.prev_lin_vel_b[w] = s.lvb0;
            d.prev_lin_vel_b[N + w] = s.lvb1;
            s.plv0 = s.lvb0;
            s.plv1 = s.lvb1;
        }
        if (st & SS_ST_OBS) {
            ensure_action();
            unsigned bad_bits = 0;
            for_terms<C, C::kCapGroups>(0, C::n_groups(d), [&](auto gg) {
                const int g = ival(gg);
                if (!((u.groups_mask >> g) & 1u)) return;
                bool pending = s.was_reset;
                if (u.any_pending) {
                    pending |= d.group[g].pending[w] != 0;
                    d.group[g].pending[w] = 0;
                }
                double* out = C::kStageObs
                                  ? obs_stage + C::kBlock * C::g_soff(d, g) + (int)threadIdx.x * C::g_dim(d, g)
                                  : d.group[g].out + (int64_t)w * C::g_dim(d, g);
                const int first = C::g_first(d, g);
                for_terms<C, C::kCapObs>(first, first + C::g_n(d, g), [&](auto tt) {
                    obs_term<C>(d, u, ival(tt), w, s, pending, out, bad_bits);
                });
            });
            d.obs_bad[w] = bad_bits;
            if (!C::kStageObs && C::mirror_on(d)) {
                // unstaged rows: repeat them into the host mirror
                for_terms<C, C::kCapGroups>(0, C::n_groups(d), [&](auto gg) {
                    const int g = ival(gg);
                    if (!((u.groups_mask >> g) & 1u)) return;
                    const int D = C::g_dim(d, g);
                    const double* row = d.group[g].out + (int64_t)w * D;
                    double* mrow = mirror_of(d, d.group[g].out) + (int64_t)w * D;
                    for (int k = 0; k < D; ++k) mrow[k] = row[k];
                });
            }
        }
        if (st & SS_ST_PREV_AFTER) {
            d.prev_lin_vel_b[w] = s.lvb0;
            d.prev_lin_vel_b[N + w] = s.lvb1;
        }

        SS_PROBE(12);
        store_phys<C>(d, w, s, /*store_cache=*/phys || s.was_reset);
        SS_PROBE(13);
    }

    // ---- staged observation rows -> global, one bulk copy per group
    if constexpr (C::kStageObs) {
        if (st & SS_ST_OBS) {
            __syncthreads();
            const int w0 = blockIdx.x * blockDim.x;
            const int rows = (N - w0) < (int)blockDim.x ? (N - w0) : (int)blockDim.x;
            for_terms<C, C::kCapGroups>(0, C::n_groups(d), [&](auto gg) {
                const int g = ival(gg);
                if (!((u.groups_mask >> g) & 1u)) return;
                const int D = C::g_dim(d, g);
                double* dst = d.group[g].out + (int64_t)w0 * D;
                const double* src = obs_stage + C::kBlock * C::g_soff(d, g);
                const unsigned bytes = (unsigned)rows * D * 8u;
                const bool bulk = ((bytes & 15u) == 0) && ((((unsigned long long)dst) & 15ull) == 0);
                double* mdst = C::mirror_on(d) ? mirror_of(d, dst) : nullptr;
                const bool mbulk = SS_MIRROR_TMA && ((((unsigned long long)mdst) & 15ull) == 0);
                if (bulk) {
                    if (threadIdx.x == 0) {
                        const unsigned saddr = (unsigned)__cvta_generic_to_shared(src);
                        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(saddr),
                                     "r"(bytes)
                                     : "memory");
                        if (mdst && mbulk)  // the same rows straight into the host mirror over PCIe
                            asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(mdst),
                                         "r"(saddr), "r"(bytes)
                                         : "memory");
                        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
                    }
                    if (mdst && !mbulk)
                        for (int i = threadIdx.x; i < rows * D; i += blockDim.x) mdst[i] = src[i];
                } else {
                    for (int i = threadIdx.x; i < rows * D; i += blockDim.x) dst[i] = src[i];
                    if (mdst)
                        for (int i = threadIdx.x; i < rows * D; i += blockDim.x) mdst[i] = src[i];
                }
            });
            if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
        }
    }

    // ---- warp-aggregated trigger counters (managers/termination.py:31-39)
    if (st & SS_ST_TERM) {
        const int lane = threadIdx.x & 31;
        for (int t = 0; t < C::n_terms(d); ++t) {
            const unsigned m = __ballot_sync(0xffffffffu, (s.trig_bits >> t) & 1u);
            if (lane == 0 && m) atomicAdd((unsigned long long*)&d.trigger_counts[t], (unsigned long long)__popc(m));
        }
        const unsigned m = __ballot_sync(0xffffffffu, (s.trig_bits >> 31) & 1u);
        if (lane == 0 && m) {
            atomicAdd((unsigned long long*)&d.trigger_counts[C::n_terms(d)], (unsigned long long)__popc(m));
            // zero-copy flag in mapped pinned host memory: the host notices a
            // nonfinite step without a per-step device->host copy (env.py:240-241)
            if (d.nf_flags) *((volatile uint32_t*)&d.nf_flags[u.nf_slot]) = 1u;
        }
    }

    // ---- the job statistics of metrics.build_record (metrics.py:31-45), fused into the step's tail
    // on log-interval steps: [n, sum reward, sum ep_sums[t], trigger counts, terrain-row histogram,
    // sum nonfinite] (the ss_stats_pack layout) reduced in a fixed order -- lanes by shuffle tree,
    // warps in order, blocks in order by the last block to arrive -- so the vector is deterministic,
    // ready for the single all_reduce; one launch fewer per log interval than a separate pack
    if constexpr (FS == 0 || (FS & SS_ST_REWARD))
    if (u.stats_out && (int)gridDim.x * (int)blockDim.x >= N && (int)blockDim.x <= C::kBlock) {
        // the warp partials reuse the observation staging buffer when there is one (its bulk copies
        // have been read: thread 0 waited on them before this barrier), keeping builds within 48 KB
        constexpr bool kReuse = C::kStageObs && C::kObsTotal * 32 >= SS_STATS_MAXV;
        __shared__ double red_s[kReuse ? 1 : (C::kBlock / 32) * SS_STATS_MAXV];
        double* const red = kReuse ? obs_stage : red_s;
        __shared__ bool last;
        __syncthreads();
        const int T = C::n_rewards(d), R = u.stats_rows, V = 2 + T + R;
        const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = (int)blockDim.x >> 5;
        const long long row = active ? d.terrain_rows[w] : -1;
        auto reduce_to = [&](int v, double x) {
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) x += __shfl_down_sync(0xffffffffu, x, o);
            if (lane == 0) red[warp * SS_STATS_MAXV + v] = x;
        };
        reduce_to(0, active ? stat_reward : 0.0);
        for_terms<C, C::kCapRewards>(0, C::n_rewards(d), [&](auto rr) {
            const int r = ival(rr);
            reduce_to(1 + r, active ? s.ep_sum[r] : 0.0);
        });
        reduce_to(T + 1, (active && s.nonfinite) ? 1.0 : 0.0);
        for (int k = 0; k < R; ++k) reduce_to(T + 2 + k, (row == (long long)k) ? 1.0 : 0.0);
        __syncthreads();
        for (int v = threadIdx.x; v < V; v += blockDim.x) {
            double acc = 0.0;
            for (int k = 0; k < nw; ++k) acc += red[k * SS_STATS_MAXV + v];
            u.stats_partials[(int64_t)blockIdx.x * SS_STATS_MAXV + v] = acc;
        }
        __threadfence();  // partials and this block's trigger-count atomics before the ticket
        __syncthreads();
        // atomicInc wraps the ticket back to 0 at the last arrival: ready for the next launch
        if (threadIdx.x == 0) last = atomicInc(u.stats_ticket, gridDim.x - 1) == gridDim.x - 1;
        __syncthreads();
        if (last) {
            __threadfence();
            const int Cn = C::n_terms(d) + 1;
            for (int v = threadIdx.x; v < V; v += blockDim.x) {
                double acc = 0.0;
                for (int b = 0; b < (int)gridDim.x; ++b)
                    acc += ((volatile double*)u.stats_partials)[(int64_t)b * SS_STATS_MAXV + v];
                const int o = v == 0 ? 1 : (v <= T ? 1 + v : (v == T + 1 ? 2 + T + Cn + R : 2 + T + Cn + (v - T - 2)));
                u.stats_out[o] = acc;
            }
            for (int c = threadIdx.x; c < Cn; c += blockDim.x)
                u.stats_out[2 + T + c] = (double)((volatile unsigned long long*)d.trigger_counts)[c];
            if (threadIdx.x == 0) u.stats_out[0] = (double)N;
        }
    }
    SS_PROBE_SPAN(0);
}

}  // namespace ss
