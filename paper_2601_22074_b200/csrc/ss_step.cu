// ss_step.cu -- the fused, thread-per-world ManagerBasedRlEnv.step for sm_100a.
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
// The launch is configured by a __grid_constant__ ss_env_desc (term tables,
// model constants, device pointers) and an ss_uniforms block holding the
// host-tracked per-step scalars (global_step, sim_step, ring heads, reward
// weights), so there is no device->host round trip anywhere on the path.
//
// Template parameters KM/FM bound the joint and foot counts so that the
// per-world arrays stay in registers (loops run to the compile-time bound
// with a predicate on the runtime count; runtime indices into register
// arrays are resolved with unrolled selects instead of local memory).
#include <cstdio>
#include <cstring>

#include "ss_device.cuh"

namespace ss {

constexpr int kBlock = 128;
constexpr int64_t kNeverTouched = -(1ll << 40);  // sensors.py:51

// register-array helpers: value at runtime index j of a compile-time array
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

template <int KM, int FM>
struct World {
    // BatchState (sim/state.py:20-38)
    double q[3 + KM], qd[3 + KM], ctrl[KM];
    double ext0, ext1, time;
    // ContactCache of the last substep (sim/state.py:10-17)
    double fn[FM], ft[FM], fpx[FM], fpz[FM], fvx[FM], fvz[FM];
    bool fin[FM];
    // EntityData snapshot taken at refresh (entity.py:145-165)
    double eq[3 + KM], eqd[3 + KM];
    double lvb0, lvb1, pg0, pg1;
    double efn[FM], eft[FM], efvx[FM];
    bool efin[FM];
    double sp, cp;  // sin/cos of q[2] (valid while trig_ok)
    bool trig_ok;
    // action manager
    double targets[KM];
    double action[SS_MAX_ACTION], prev_action[SS_MAX_ACTION];
    bool have_action;
    // command
    double cmd[SS_MAX_CMD];
    // contact sensor (sensors.py:68-79)
    bool s_in[FM];
    double s_air[FM], s_last_air[FM], s_contact[FM];
    int64_t s_td[FM];
    double s_hist[SS_MAX_HIST][FM];
    bool have_sensor;
    // episode
    int64_t ep_steps;
    double cmd_dist;
    // flags
    bool terminated, truncated, nonfinite, was_reset;
    uint32_t trig_bits;
};

// ---------------------------------------------------------------------------
// RNG draw for world w from purpose slot (advances that world's counter)

__device__ __forceinline__ uint64_t rng_begin(const ss_env_desc& d, int slot, int w,
                                              uint64_t& key) {
    key = stream_key(d.rng.base[slot], (uint64_t)(d.rng.world_id_offset + w));
    return d.rng.counter[slot][w];
}
__device__ __forceinline__ void rng_end(const ss_env_desc& d, int slot, int w, uint64_t c) {
    d.rng.counter[slot][w] = c;
}

// ---------------------------------------------------------------------------
// load / store of the physics state

template <int KM, int FM>
__device__ __forceinline__ void load_phys(const ss_env_desc& d, int w, World<KM, FM>& s,
                                          bool load_cache) {
    const int N = d.n_worlds, K = d.model.n_joints, F = d.model.n_feet;
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
        bool ok = load_cache && i < F;
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

template <int KM, int FM>
__device__ __forceinline__ void store_phys(const ss_env_desc& d, int w, const World<KM, FM>& s,
                                           bool store_cache) {
    const int N = d.n_worlds, K = d.model.n_joints, F = d.model.n_feet;
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

// EntityData.refresh (entity.py:145-165)
template <int KM, int FM>
__device__ __forceinline__ void refresh(World<KM, FM>& s) {
    double sn, c;
    sincos(s.q[2], &sn, &c);
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
// StepPipeline.substep (sim/physics.py:178-249): contact at the start-of-
// substep state, forces, semi-implicit Euler, contact cache, time += dt.

template <int KM, int FM>
__device__ __forceinline__ void phys_substep(const ss_env_desc& d, int w, World<KM, FM>& s) {
    const ss_model& M = d.model;
    const int N = d.n_worlds, K = M.n_joints, F = M.n_feet;
    const double base_mass = field_at(d.field[M.f_base_mass], 0, w, N);
    const double base_inertia = field_at(d.field[M.f_base_inertia], 0, w, N);
    const double friction = field_at(d.field[M.f_friction], 0, w, N);
    double lm[KM], rot[KM], dmp[KM];
#pragma unroll
    for (int j = 0; j < KM; ++j) {
        lm[j] = (j < K) ? field_at(d.field[M.f_link_mass], j, w, N) : 0.0;
        rot[j] = (j < K) ? field_at(d.field[M.f_rotor_inertia], j, w, N) : 1.0;
        dmp[j] = (j < K) ? field_at(d.field[M.f_damping], j, w, N) : 0.0;
    }

    // --- forward kinematics (fk_batch_trig, sim/physics.py:22-57)
    double sp, cp;
    if (s.trig_ok) {
        sp = s.sp;
        cp = s.cp;
    } else {
        sincos(s.q[2], &sp, &cp);
    }
    double th[KM], st[KM], ct[KM], ax[KM], az[KM], tx[KM], tz[KM];
#pragma unroll
    for (int j = 0; j < KM; ++j) {
        if (j < K) {
            const int p = M.parent[j];
            double pa = s.q[2];
#pragma unroll
            for (int i = 0; i < j; ++i)
                if (p == i) pa = th[i];
            th[j] = pa + s.q[3 + j];
        } else {
            th[j] = 0.0;
        }
    }
#pragma unroll
    for (int j = 0; j < KM; ++j) {
        if (j < K) sincos(th[j], &st[j], &ct[j]);
        else { st[j] = 0.0; ct[j] = 1.0; }
    }
#pragma unroll
    for (int j = 0; j < KM; ++j) {
        if (j < K) {
            const int p = M.parent[j];
            double sn = sp, c = cp, px = s.q[0], pz = s.q[1];
#pragma unroll
            for (int i = 0; i < j; ++i)
                if (p == i) { sn = st[i]; c = ct[i]; px = ax[i]; pz = az[i]; }
            const double ox = M.attach_x[j], oz = M.attach_z[j];
            ax[j] = px + (c * ox - sn * oz);
            az[j] = pz + (sn * ox + c * oz);
            tx[j] = ax[j] + M.link_len[j] * st[j];
            tz[j] = az[j] - M.link_len[j] * ct[j];
        } else {
            ax[j] = az[j] = tx[j] = tz[j] = 0.0;
        }
    }

    // --- contact (compute_contact, sim/physics.py:75-111)
    double nfn[FM], nft[FM], nvx[FM], nvz[FM], npx[FM], npz[FM];
    bool ntouch[FM];
#pragma unroll
    for (int i = 0; i < FM; ++i) {
        nfn[i] = nft[i] = nvx[i] = nvz[i] = npx[i] = npz[i] = 0.0;
        ntouch[i] = false;
        if (i < F) {
            const int fj = M.foot_joint[i];
            const uint32_t mask = M.chain_mask[i];
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
            const double phi = terrain_height(d.terrain, px) - pz;
            const bool touching = phi > 0.0;
            double normal = np_maximum(0.0, M.k_n * phi - M.c_n * vz);
            normal = touching ? normal : 0.0;
            const double bound = friction * normal;
            double tangent = np_clip(-M.k_t * vx, -bound, bound);
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

    // --- generalized forces (stage_forces, sim/physics.py:191-214)
    double tau[3 + KM];
    tau[0] = 0.0;
    tau[1] = 0.0;
    tau[2] = 0.0;
#pragma unroll
    for (int j = 0; j < KM; ++j) tau[3 + j] = 0.0 + s.ctrl[j];
#pragma unroll
    for (int j = 0; j < KM; ++j) tau[3 + j] = tau[3 + j] - dmp[j] * s.qd[3 + j];
    const double m_total = base_mass + np_sum<KM>(lm, K);
    tau[1] = tau[1] - m_total * M.gravity;
#pragma unroll
    for (int j = 0; j < KM; ++j) tau[3 + j] = tau[3 + j] - lm[j] * M.gravity * M.half_len[j] * st[j];
    tau[0] = tau[0] + s.ext0;
    tau[1] = tau[1] + s.ext1;
#pragma unroll
    for (int i = 0; i < FM; ++i) {
        if (i < F) {
            const double fx = nft[i], fz = nfn[i], px = npx[i], pz = npz[i];
            const uint32_t mask = M.chain_mask[i];
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

    // --- semi-implicit Euler (stage_integrate, sim/physics.py:216-224)
    const double inv_m = 1.0 / m_total;
    tau[0] = tau[0] * inv_m;
    tau[1] = tau[1] * inv_m;
    tau[2] = tau[2] * (1.0 / base_inertia);
#pragma unroll
    for (int j = 0; j < KM; ++j) tau[3 + j] = tau[3 + j] * (1.0 / rot[j]);
    const double dt = M.dt;
#pragma unroll
    for (int i = 0; i < 3 + KM; ++i)
        if (i < 3 + K) s.qd[i] = s.qd[i] + tau[i] * dt;
#pragma unroll
    for (int i = 0; i < 3 + KM; ++i)
        if (i < 3 + K) s.q[i] = s.q[i] + s.qd[i] * dt;

    // --- contact cache + clock (stage_finalize, sim/physics.py:226-235)
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
__device__ __forceinline__ void apply_actuators(const ss_env_desc& d, const ss_uniforms& u,
                                                int w, int sub, World<KM, FM>& s) {
    const int N = d.n_worlds;
    for (int a = 0; a < d.n_actuators; ++a) {
        const ss_actuator& A = d.actuator[a];
        int64_t delay = 0;
        int head = 0;
        if (A.delayed) {
            delay = A.delay_steps[w];
            head = (u.act_head0[a] + sub + 1) % A.cap;
        }
        for (int i = 0; i < A.dim; ++i) {
            const int j = A.joint[i];
            double qdes = sel(s.targets, j);
            if (A.delayed) {
                // DelayBuffer.push_and_read (actuators.py:208-213)
                A.ring[((int64_t)head * A.dim + i) * N + w] = qdes;
                int slot = (int)(((int64_t)head - delay) % A.cap);
                if (slot < 0) slot += A.cap;
                if (slot != head) qdes = A.ring[((int64_t)slot * A.dim + i) * N + w];
            }
            const double qj = sel(s.q, 3 + j), qdj = sel(s.qd, 3 + j);
            double tau;
            if (A.kind == SS_ACT_MLP) {
                // newest-first histories of position error and velocity
                double x[2 * SS_MAX_HIST];
                for (int h = A.err_hist - 1; h >= 1; --h) {
                    double v = A.err_buf[((int64_t)(h - 1) * A.dim + i) * N + w];
                    A.err_buf[((int64_t)h * A.dim + i) * N + w] = v;
                    x[h] = v;
                }
                x[0] = qdes - qj;
                A.err_buf[(int64_t)i * N + w] = x[0];
                for (int h = A.vel_hist - 1; h >= 1; --h) {
                    double v = A.vel_buf[((int64_t)(h - 1) * A.dim + i) * N + w];
                    A.vel_buf[((int64_t)h * A.dim + i) * N + w] = v;
                    x[A.err_hist + h] = v;
                }
                x[A.err_hist] = qdj;
                A.vel_buf[(int64_t)i * N + w] = qdj;
                // mlp_forward (actuators.py:177-180): x <- act(W x + b)
                double buf0[32], buf1[32];
                int n_in = A.err_hist + A.vel_hist;
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
                tau = np_clip(cur[0], -A.effort, A.effort);
            } else {
                const double kp = field_at(d.field[A.f_kp], i, w, N);
                const double kd = field_at(d.field[A.f_kd], i, w, N);
                tau = kp * (qdes - qj) + kd * (0.0 - qdj);
                if (A.kind == SS_ACT_PD) {
                    tau = np_clip(tau, -A.effort, A.effort);
                } else {
                    // dc_motor_torque (actuators.py:110-117)
                    const double hi = np_clip(A.saturation * (1.0 - qdj / A.vel_limit), 0.0, A.effort);
                    const double lo = np_clip(A.saturation * (-1.0 - qdj / A.vel_limit), -A.effort, 0.0);
                    tau = np_clip(tau, lo, hi);
                }
            }
            sel_store(s.ctrl, j, tau);
        }
    }
}

// Actuator.reset (actuators.py:269-277) for one world
__device__ __forceinline__ void reset_actuators(const ss_env_desc& d, int w, const double* targets_full,
                                                int KMAX) {
    const int N = d.n_worlds;
    for (int a = 0; a < d.n_actuators; ++a) {
        const ss_actuator& A = d.actuator[a];
        if (A.delayed) {
            for (int i = 0; i < A.dim; ++i) {
                const double v = targets_full[A.joint[i]];
                for (int h = 0; h < A.cap; ++h) A.ring[((int64_t)h * A.dim + i) * N + w] = v;
            }
            if (A.resample_on_reset) {
                double lat = A.lat_lo;
                if (!A.lat_const) {
                    uint64_t key;
                    uint64_t c = rng_begin(d, A.lat_slot, w, key);
                    lat = uniform_from_word(stream_word(key, c, 0), A.lat_lo, A.lat_hi);
                    rng_end(d, A.lat_slot, w, c + 1);
                }
                int64_t steps = (int64_t)rint(lat / d.model.dt);
                if (steps < 0) steps = 0;
                if (steps > A.cap - 1) steps = A.cap - 1;
                A.delay_steps[w] = steps;
            }
        }
        if (A.kind == SS_ACT_MLP) {
            for (int i = 0; i < A.dim; ++i) {
                for (int h = 0; h < A.err_hist; ++h) A.err_buf[((int64_t)h * A.dim + i) * N + w] = 0.0;
                for (int h = 0; h < A.vel_hist; ++h) A.vel_buf[((int64_t)h * A.dim + i) * N + w] = 0.0;
            }
        }
    }
}

// ---------------------------------------------------------------------------
// events (mdp.py:186-220, managers/event.py:19-114)

// randomize_field for one world (managers/event.py:19-52)
__device__ __forceinline__ void randomize_world(const ss_env_desc& d, int w, int field, int dist,
                                                double r0, double r1, int op, int slot) {
    const ss_field& f = d.field[field];
    const int N = d.n_worlds;
    uint64_t key;
    uint64_t c = rng_begin(d, slot, w, key);
    for (int k = 0; k < f.size; ++k) {
        double draw;
        if (dist == SS_DIST_UNIFORM) {
            draw = uniform_from_word(stream_word(key, c, k), r0, r1);
        } else {
            draw = r0 + normal_from_words(stream_word(key, c, k), stream_word(key, c, f.size + k), r1);
        }
        const double base = f.base[k];
        double v = draw;
        if (op == SS_OP_SCALE) v = base * draw;
        else if (op == SS_OP_ADD) v = base + draw;
        f.ptr[(int64_t)k * N + w] = v;
    }
    rng_end(d, slot, w, c + (uint64_t)(dist == SS_DIST_UNIFORM ? f.size : 2 * f.size));
}

// EventManager._draw_targets for one world (managers/event.py:75-84)
__device__ __forceinline__ double draw_interval_target(const ss_env_desc& d, const ss_event_term& E,
                                                       int w) {
    uint64_t key;
    uint64_t c = rng_begin(d, E.iv_slot, w, key);
    const double draw = uniform_from_word(stream_word(key, c, 0), E.iv_lo, E.iv_hi);
    rng_end(d, E.iv_slot, w, c + 1);
    const double dt = d.dt_control;
    const double quantized = rint(draw / dt) * dt;
    return np_clip(quantized, E.iv_lo_q, E.iv_hi_q);
}

template <int KM, int FM>
__device__ __forceinline__ void apply_event(const ss_env_desc& d, const ss_event_term& E, int w,
                                            World<KM, FM>& s) {
    const int K = d.model.n_joints;
    if (E.func == SS_EVT_RANDOMIZE_FIELD) {
        randomize_world(d, w, E.field, E.distribution, E.r0, E.r1, E.operation, E.slot_a);
    } else if (E.func == SS_EVT_PUSH_BASE) {
        // push_base (mdp.py:201-211): fx then fz, each one draw per world
        uint64_t key;
        uint64_t c = rng_begin(d, E.slot_a, w, key);
        s.ext0 = s.ext0 + uniform_from_word(stream_word(key, c, 0), E.r0, E.r1);
        rng_end(d, E.slot_a, w, c + 1);
        c = rng_begin(d, E.slot_b, w, key);
        s.ext1 = s.ext1 + uniform_from_word(stream_word(key, c, 0), E.r2, E.r3);
        rng_end(d, E.slot_b, w, c + 1);
    } else if (E.func == SS_EVT_JOINT_JITTER) {
        // reset_joints_jitter (mdp.py:214-220)
        uint64_t key;
        uint64_t c = rng_begin(d, E.slot_a, w, key);
#pragma unroll
        for (int j = 0; j < KM; ++j)
            if (j < K) s.q[3 + j] = s.q[3 + j] + uniform_from_word(stream_word(key, c, j), E.r0, E.r1);
        rng_end(d, E.slot_a, w, c + (uint64_t)K);
    }
}

// CommandManager.resample for one world (managers/command.py:33-39)
template <int KM, int FM>
__device__ __forceinline__ void resample_command(const ss_env_desc& d, int w, World<KM, FM>& s) {
    const int N = d.n_worlds;
    uint64_t key;
    uint64_t c = rng_begin(d, d.cmd_slot, w, key);
    for (int ch = 0; ch < d.n_cmd; ++ch) {
        const double lo = d.ranges[(int64_t)(2 * ch) * N + w];
        const double hi = d.ranges[(int64_t)(2 * ch + 1) * N + w];
        s.cmd[ch] = uniform_from_word(stream_word(key, c, ch), lo, hi);
        d.command[(int64_t)ch * N + w] = s.cmd[ch];
    }
    rng_end(d, d.cmd_slot, w, c + (uint64_t)d.n_cmd);
    d.countdown[w] = d.period_steps;
}

// ---------------------------------------------------------------------------
// observation terms (mdp.py:26-89); returns dim, values in v[]

template <int KM, int FM>
__device__ __forceinline__ int obs_raw(const ss_env_desc& d, const ss_obs_term& T, int w,
                                       const World<KM, FM>& s, double* v) {
    const int N = d.n_worlds, K = d.model.n_joints, F = d.model.n_feet;
    switch (T.func) {
        case SS_OBS_BASE_LIN_VEL:
            v[0] = s.lvb0;
            v[1] = s.lvb1;
            return 2;
        case SS_OBS_BASE_ANG_VEL:
            v[0] = s.eqd[2];
            return 1;
        case SS_OBS_BASE_LIN_ACC:
            v[0] = (s.lvb0 - d.prev_lin_vel_b[w]) / d.dt_control;
            v[1] = (s.lvb1 - d.prev_lin_vel_b[N + w]) / d.dt_control;
            return 2;
        case SS_OBS_PROJECTED_GRAVITY:
            v[0] = s.pg0;
            v[1] = s.pg1;
            return 2;
        case SS_OBS_JOINT_POS_REL:
#pragma unroll
            for (int j = 0; j < KM; ++j)
                if (j < K) v[j] = s.eq[3 + j] - d.joint_pos[j];
            return K;
        case SS_OBS_JOINT_VEL:
#pragma unroll
            for (int j = 0; j < KM; ++j)
                if (j < K) v[j] = s.eqd[3 + j];
            return K;
        case SS_OBS_LAST_ACTION:
            for (int k = 0; k < d.action_dim; ++k) v[k] = s.action[k];
            return d.action_dim;
        case SS_OBS_COMMAND:
            for (int c = 0; c < d.n_cmd; ++c) v[c] = s.cmd[c];
            return d.n_cmd;
        case SS_OBS_BASE_HEIGHT:
            v[0] = s.q[1];
            return 1;
        case SS_OBS_SIM_TIME:
            v[0] = s.time;
            return 1;
        case SS_OBS_HEIGHT_SCAN:
            // RayScanner.read (sensors.py:36-46): h(x_base + off) - z_base
            for (int r = 0; r < d.n_rays; ++r)
                v[r] = terrain_height(d.terrain, s.eq[0] + d.ray_offset[r]) - s.eq[1];
            return d.n_rays;
        case SS_OBS_FOOT_CONTACT_FORCES:
#pragma unroll
            for (int i = 0; i < FM; ++i) {
                if (i < F) {
                    v[2 * i] = s.eft[i];
                    v[2 * i + 1] = s.efn[i];
                }
            }
            return 2 * F;
        default:  // SS_OBS_EXTERNAL: values computed by a registered Python term
            for (int k = 0; k < T.dim; ++k) v[k] = T.ext[(int64_t)w * T.dim + k];
            return T.dim;
    }
}

// ObservationManager.compute for one group, one world (managers/observation.py:99-137)
template <int KM, int FM>
__device__ __forceinline__ void compute_group(const ss_env_desc& d, const ss_uniforms& u, int g, int w,
                                              const World<KM, FM>& s, bool pending, uint32_t& bad_bits) {
    const int N = d.n_worlds;
    const ss_obs_group& G = d.group[g];
    double* out = G.out + (int64_t)w * G.dim;
    for (int t = G.first_term; t < G.first_term + G.n_terms; ++t) {
        const ss_obs_term& T = d.obs[t];
        double v[SS_MAX_JOINTS > 2 * SS_MAX_FEET ? SS_MAX_JOINTS : 2 * SS_MAX_FEET];
        const int dim = obs_raw(d, T, w, s, v);
        bool bad = false;
        for (int k = 0; k < dim; ++k) bad |= !isfinite(v[k]);
        if (bad) bad_bits |= 1u << t;
        if (T.has_clip)
            for (int k = 0; k < dim; ++k) v[k] = np_clip(v[k], T.clip_lo, T.clip_hi);
        if (T.has_scale)
            for (int k = 0; k < dim; ++k) v[k] = v[k] * T.scale;
        if (T.noise == SS_NOISE_UNIFORM) {
            uint64_t key;
            uint64_t c = rng_begin(d, T.noise_slot, w, key);
            const double lo = -T.noise_scale, hi = T.noise_scale;
            for (int k = 0; k < dim; ++k) v[k] = v[k] + uniform_from_word(stream_word(key, c, k), lo, hi);
            rng_end(d, T.noise_slot, w, c + (uint64_t)dim);
        } else if (T.noise == SS_NOISE_GAUSSIAN) {
            uint64_t key;
            uint64_t c = rng_begin(d, T.noise_slot, w, key);
            for (int k = 0; k < dim; ++k)
                v[k] = v[k] + normal_from_words(stream_word(key, c, k), stream_word(key, c, dim + k), T.noise_scale);
            rng_end(d, T.noise_slot, w, c + (uint64_t)(2 * dim));
        }
        if (T.delay == 0 && T.history == 1) {
            for (int k = 0; k < dim; ++k) out[T.col + k] = v[k];
            continue;
        }
        // delay ring: push, then read `delay` pushes back (flood on reset)
        const int D1 = T.delay + 1;
        const int head = u.obs_delay_head[t];
        if (T.delay > 0) {
            if (pending) {
                for (int h = 0; h < D1; ++h)
                    for (int k = 0; k < dim; ++k) T.delay_ring[((int64_t)h * dim + k) * N + w] = v[k];
            } else {
                for (int k = 0; k < dim; ++k) T.delay_ring[((int64_t)head * dim + k) * N + w] = v[k];
                int slot = (head - T.delay) % D1;
                if (slot < 0) slot += D1;
                for (int k = 0; k < dim; ++k) v[k] = T.delay_ring[((int64_t)slot * dim + k) * N + w];
            }
        }
        // history ring, oldest-first output (newest at hist head)
        const int H = T.history;
        if (H == 1) {
            for (int k = 0; k < dim; ++k) out[T.col + k] = v[k];
            continue;
        }
        const int hh = u.obs_hist_head[t];
        if (pending) {
            for (int h = 0; h < H; ++h)
                for (int k = 0; k < dim; ++k) {
                    T.hist_ring[((int64_t)h * dim + k) * N + w] = v[k];
                    out[T.col + h * dim + k] = v[k];
                }
        } else {
            for (int k = 0; k < dim; ++k) T.hist_ring[((int64_t)hh * dim + k) * N + w] = v[k];
            for (int h = 0; h < H; ++h) {
                const int slot = (hh + 1 + h) % H;
                for (int k = 0; k < dim; ++k)
                    out[T.col + h * dim + k] = (slot == hh) ? v[k] : T.hist_ring[((int64_t)slot * dim + k) * N + w];
            }
        }
    }
}

// ---------------------------------------------------------------------------
// reward terms (mdp.py:96-160)

template <int KM, int FM>
__device__ __forceinline__ double reward_value(const ss_env_desc& d, const ss_uniforms& u,
                                               const ss_reward_term& R, int w, const World<KM, FM>& s,
                                               int64_t sim_step_now) {
    const int N = d.n_worlds, K = d.model.n_joints, F = d.model.n_feet;
    switch (R.func) {
        case SS_REW_CONSTANT:
            return R.p0;
        case SS_REW_BASE_HEIGHT:
            return s.q[1];
        case SS_REW_TRACK_VX_EXP: {
            const double err = s.cmd[0] - s.lvb0;
            return exp(-(err * err) / (R.p0 * R.p0));
        }
        case SS_REW_PITCH_RATE:
            return s.eqd[2] * s.eqd[2];
        case SS_REW_ANG_MOMENTUM: {
            const double inertia = field_at(d.field[d.model.f_base_inertia], 0, w, N);
            const double m = inertia * s.eqd[2];
            return m * m;
        }
        case SS_REW_ACTION_RATE: {
            double sq[SS_MAX_ACTION];
#pragma unroll
            for (int k = 0; k < SS_MAX_ACTION; ++k) {
                const double dl = s.action[k] - s.prev_action[k];
                sq[k] = dl * dl;
            }
            return np_sum<SS_MAX_ACTION>(sq, d.action_dim);
        }
        case SS_REW_JOINT_LIMIT: {
            double ex[KM];
#pragma unroll
            for (int j = 0; j < KM; ++j) {
                ex[j] = 0.0;
                if (j < K) {
                    const double lo = d.model.pos_lo[j], hi = d.model.pos_hi[j];
                    const double mid = 0.5 * (lo + hi);
                    const double soft_half = 0.5 * (hi - lo) * d.model.soft_frac[j];
                    ex[j] = np_maximum(0.0, fabs(s.eq[3 + j] - mid) - soft_half);
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
                const bool landed = s.s_td[i] > sim_step_now - d.decimation;
                at[i] = (s.s_last_air[i] - R.p0) * (landed ? 1.0 : 0.0);
            }
            return np_sum<FM>(at, F);
        }
        default:
            return R.ext[w];
    }
}

// ---------------------------------------------------------------------------
// the fused step kernel

template <int KM, int FM>
__global__ void __launch_bounds__(kBlock) step_kernel(const __grid_constant__ ss_env_desc d,
                                                      const __grid_constant__ ss_uniforms u) {
    const int N = d.n_worlds;
    const int w = blockIdx.x * blockDim.x + threadIdx.x;
    const bool active = w < N;
    const uint32_t st = u.stages;
    const int K = d.model.n_joints, F = d.model.n_feet;
    World<KM, FM> s;
#pragma unroll
    for (int k = 0; k < SS_MAX_ACTION; ++k) s.action[k] = s.prev_action[k] = 0.0;
    s.trig_bits = 0;
    s.terminated = s.truncated = s.nonfinite = s.was_reset = false;

    if (active) {
        const bool sim = (st & (SS_ST_APPLY | SS_ST_PUSH | SS_ST_PHYS | SS_ST_SENSOR)) && u.nsub > 0;
        const bool phys = (st & SS_ST_PHYS) && u.nsub > 0;
        load_phys(d, w, s, /*load_cache=*/!phys);
        if (!phys) refresh(s);  // staged launch: entity data from the stored state

        // command values are read by termination, reward, reset, command, obs
        for (int c = 0; c < d.n_cmd; ++c) s.cmd[c] = d.command[(int64_t)c * N + w];
        s.have_action = false;
        s.have_sensor = false;

        // targets live in registers across the substeps
        const bool need_targets = st & (SS_ST_ACTION | SS_ST_APPLY | SS_ST_RESET | SS_ST_RESET_ALL);
#pragma unroll
        for (int j = 0; j < KM; ++j) s.targets[j] = (need_targets && j < K) ? d.targets[(int64_t)j * N + w] : 0.0;

        // ---- 1. ActionManager.process (managers/action.py:68-82)
        if (st & SS_ST_ACTION) {
            const double* a = u.actions + (int64_t)w * d.action_dim;
            for (int k = 0; k < d.action_dim; ++k) {
                s.prev_action[k] = d.action[(int64_t)k * N + w];
                s.action[k] = a[k];
                d.prev_action[(int64_t)k * N + w] = s.prev_action[k];
                d.action[(int64_t)k * N + w] = s.action[k];
            }
            for (int t = 0; t < d.n_action_terms; ++t) {
                const ss_action_term& A = d.action_term[t];
                for (int i = 0; i < A.dim; ++i) {
                    double x = s.action[A.start + i];
                    if (A.has_clip) x = np_clip(x, A.clip_lo, A.clip_hi);
                    sel_store(s.targets, A.joint[i], A.offset[i] + A.scale * x);
                }
            }
#pragma unroll
            for (int j = 0; j < KM; ++j)
                if (j < K) d.targets[(int64_t)j * N + w] = s.targets[j];
            s.have_action = true;
        }

        // ---- 2. decimation substeps (env.py:228-233)
        if (sim) {
            const bool sensor = st & SS_ST_SENSOR;
            if (sensor) {
                s.have_sensor = true;
#pragma unroll
                for (int i = 0; i < FM; ++i) {
                    if (i < F) {
                        s.s_in[i] = d.s_in_contact[(int64_t)i * N + w] != 0;
                        s.s_air[i] = d.s_cur_air[(int64_t)i * N + w];
                        s.s_last_air[i] = d.s_last_air[(int64_t)i * N + w];
                        s.s_contact[i] = d.s_cur_contact[(int64_t)i * N + w];
                        s.s_td[i] = d.s_last_td[(int64_t)i * N + w];
                    } else {
                        s.s_in[i] = false;
                        s.s_air[i] = s.s_last_air[i] = s.s_contact[i] = 0.0;
                        s.s_td[i] = kNeverTouched;
                    }
                }
                // the force history is fully overwritten when >= H updates run
                const int n_upd = __popc(u.sensor_mask & ((1u << u.nsub) - 1u));
                const bool need_hist = n_upd < d.hist_len;
#pragma unroll
                for (int h = 0; h < SS_MAX_HIST; ++h)
#pragma unroll
                    for (int i = 0; i < FM; ++i)
                        s.s_hist[h][i] = (need_hist && h < d.hist_len && i < F)
                                             ? d.s_force_hist[((int64_t)h * F + i) * N + w]
                                             : 0.0;
            }
            for (int sub = 0; sub < u.nsub; ++sub) {
                if (st & SS_ST_APPLY) apply_actuators(d, u, w, sub, s);
                if (st & SS_ST_PUSH) {
                    // CaptureRing.push (capture.py:53-59): ctrl written, pre-integration
                    const int slot = (u.capture_slot0 + sub) % d.capture_phys;
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
                    phys_substep(d, w, s);
                    refresh(s);
                }
                if (sensor && ((u.sensor_mask >> sub) & 1u)) {
                    // ContactSensor.update (sensors.py:91-115)
                    const int64_t now_step = u.sim_step + sub + (phys ? 1 : 0);
                    const double dt = d.model.dt;
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
                        for (int i = 0; i < FM; ++i) s.s_hist[h][i] = s.s_hist[h - 1][i];
#pragma unroll
                    for (int i = 0; i < FM; ++i) s.s_hist[0][i] = s.fn[i];
                }
            }
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
                        if (h < d.hist_len && i < F) d.s_force_hist[((int64_t)h * F + i) * N + w] = s.s_hist[h][i];
            }
        }
        const int64_t sim_step_now = u.sim_step + (phys ? u.nsub : 0);

        // lazily loaded inputs for later stages
        auto ensure_action = [&]() {
            if (!s.have_action) {
                for (int k = 0; k < SS_MAX_ACTION; ++k) {
                    s.action[k] = (k < d.action_dim) ? d.action[(int64_t)k * N + w] : 0.0;
                    s.prev_action[k] = (k < d.action_dim) ? d.prev_action[(int64_t)k * N + w] : 0.0;
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

        // ---- 3. episode bookkeeping + TerminationManager.compute (env.py:235-239)
        bool have_ep = false;
        if (st & SS_ST_TERM) {
            s.ep_steps = d.episode_steps[w];
            s.cmd_dist = d.commanded_distance[w];
            if (!(u.flags & SS_FLAG_NO_EPISODE)) {
                s.ep_steps += 1;
                if (d.n_cmd > 0) s.cmd_dist = s.cmd_dist + fabs(s.cmd[0]) * d.dt_control;
                d.episode_steps[w] = s.ep_steps;
                d.commanded_distance[w] = s.cmd_dist;
            }
            have_ep = true;
            bool term = false, trunc = false;
            for (int t = 0; t < d.n_terms; ++t) {
                const ss_term_term& T = d.term[t];
                bool m;
                if (T.func == SS_TERM_BASE_HEIGHT_BELOW) m = s.q[1] < T.p0;
                else if (T.func == SS_TERM_PITCH_BEYOND) m = fabs(s.q[2]) > T.p0;
                else if (T.func == SS_TERM_TIME_OUT) m = s.ep_steps >= d.max_episode_steps;
                else m = T.ext[w] != 0;
                if (m) s.trig_bits |= 1u << t;
                if (T.time_out) trunc |= m;
                else term |= m;
            }
            // detect_nonfinite over q, qd, ctrl (sim/state.py:69-74)
            bool bad = false;
#pragma unroll
            for (int i = 0; i < 3 + KM; ++i)
                if (i < 3 + K) bad |= !isfinite(s.q[i]) || !isfinite(s.qd[i]);
#pragma unroll
            for (int j = 0; j < KM; ++j)
                if (j < K) bad |= !isfinite(s.ctrl[j]);
            if (bad) s.trig_bits |= 1u << 31;
            term |= bad;
            s.terminated = term;
            s.truncated = trunc;
            s.nonfinite = bad;
            d.terminated[w] = term;
            d.truncated[w] = trunc;
            d.nonfinite[w] = bad;
        }

        // ---- 4. RewardManager.compute (managers/reward.py:36-49), pre-reset state
        if (st & SS_ST_REWARD) {
            ensure_action();
            ensure_sensor();
            double total = 0.0;
            for (int r = 0; r < d.n_rewards; ++r) {
                const double v = reward_value(d, u, d.reward[r], w, s, sim_step_now);
                const double contribution = u.weight[r] * v * d.dt_control;
                total += contribution;
                d.ep_sums[(int64_t)r * N + w] += contribution;
                d.ep_raw[(int64_t)r * N + w] += v;
                d.last_values[(int64_t)r * N + w] = v;
            }
            d.reward_out[w] = total;
        }

        // ---- 5. curriculum on the finished episode, then masked reset (env.py:245-250)
        bool selected = false;
        if (st & SS_ST_RESET_ALL) selected = true;
        else if (st & (SS_ST_RESET | SS_ST_CURRICULUM)) {
            if (st & SS_ST_RESET_EXT) selected = u.reset_mask[w] != 0;
            else if (st & SS_ST_TERM) selected = s.terminated || s.truncated;
            else selected = d.terminated[w] || d.truncated[w];
        }
        const bool do_reset = selected && (st & (SS_ST_RESET | SS_ST_RESET_ALL));
        if (selected && (st & SS_ST_CURRICULUM)) {
            if (!have_ep) {
                s.ep_steps = d.episode_steps[w];
                s.cmd_dist = d.commanded_distance[w];
                have_ep = true;
            }
            for (int c = 0; c < d.n_curriculum; ++c) {
                const ss_curriculum_term& C = d.curriculum[c];
                if (C.func == SS_CUR_TERRAIN_LEVELS) {
                    // terrain_levels (mdp.py:227-243)
                    const double walked = fabs(s.q[0] - d.episode_start_x[w]);
                    const double commanded = s.cmd_dist;
                    int64_t row = d.terrain_rows[w];
                    if (walked >= C.p0 * commanded) row = row + 1;
                    if (walked <= C.p1 * commanded) row = row - 1;
                    if (row < 0) row = 0;
                    if (row > d.terrain.rows - 1) row = d.terrain.rows - 1;
                    d.terrain_rows[w] = row;
                } else if (C.func == SS_CUR_COMMAND_WIDEN) {
                    // command_widen (mdp.py:246-259) -> CommandManager.widen (command.py:47-50)
                    const double steps = (double)s.ep_steps;
                    const double mean = d.ep_raw[(int64_t)C.term * N + w] / (steps > 1.0 ? steps : 1.0);
                    if (mean > C.p0) {
                        for (int ch = 0; ch < d.n_cmd; ++ch) {
                            const double blo = fabs(d.init_lo[ch]) * d.cap_scale;
                            const double bhi = fabs(d.init_hi[ch]) * d.cap_scale;
                            double* rlo = d.ranges + (int64_t)(2 * ch) * N + w;
                            double* rhi = d.ranges + (int64_t)(2 * ch + 1) * N + w;
                            *rlo = np_clip(*rlo * C.p1, -blo, blo);
                            *rhi = np_clip(*rhi * C.p1, -bhi, bhi);
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
                s.q[i] = d.base_pose[i];
                s.qd[i] = d.base_vel[i];
            }
#pragma unroll
            for (int j = 0; j < KM; ++j) {
                s.q[3 + j] = (j < K) ? d.joint_pos[j] : 0.0;
                s.qd[3 + j] = (j < K) ? d.joint_vel[j] : 0.0;
            }
            s.time = 0.0;
            // _place_on_terrain (env.py:171-180)
            {
                const int64_t row = d.terrain_rows[w], col = d.terrain_cols[w];
                const double origin = (double)(row * d.terrain.cols + col) * d.terrain.patch_length;
                const double spawn_x = origin + d.spawn_offset;
                s.q[0] = s.q[0] + spawn_x;
                s.q[1] = s.q[1] + terrain_height(d.terrain, spawn_x);
            }
            // EventManager.apply_reset (managers/event.py:92-101)
            for (int e = 0; e < d.n_events; ++e) {
                const ss_event_term& E = d.event[e];
                if (E.mode == SS_MODE_RESET && E.func != SS_EVT_EXTERNAL) {
                    apply_event(d, E, w, s);
                } else if (E.mode == SS_MODE_INTERVAL) {
                    E.elapsed[w] = 0.0;
                    E.target[w] = draw_interval_target(d, E, w);
                }
            }
            // CommandManager.resample
            if (d.n_cmd > 0) resample_command(d, w, s);
            // ActionManager.reset (managers/action.py:92-97)
            for (int k = 0; k < d.action_dim; ++k) {
                s.action[k] = 0.0;
                s.prev_action[k] = 0.0;
                d.action[(int64_t)k * N + w] = 0.0;
                d.prev_action[(int64_t)k * N + w] = 0.0;
            }
            s.have_action = true;
            for (int t = 0; t < d.n_action_terms; ++t) {
                const ss_action_term& A = d.action_term[t];
                for (int i = 0; i < A.dim; ++i) sel_store(s.targets, A.joint[i], A.offset[i]);
            }
            double tfull[SS_MAX_JOINTS];
#pragma unroll
            for (int j = 0; j < KM; ++j) {
                tfull[j] = s.targets[j];
                if (j < K) d.targets[(int64_t)j * N + w] = s.targets[j];
            }
            reset_actuators(d, w, tfull, KM);
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
                    for (int h = 0; h < d.hist_len; ++h) d.s_force_hist[((int64_t)h * F + i) * N + w] = 0.0;
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
            for (int r = 0; r < d.n_rewards; ++r) {
                d.finalized[(int64_t)r * N + w] = d.ep_sums[(int64_t)r * N + w];
                d.ep_sums[(int64_t)r * N + w] = 0.0;
                d.ep_raw[(int64_t)r * N + w] = 0.0;
            }
            s.ep_steps = 0;
            s.cmd_dist = 0.0;
            have_ep = true;
            d.episode_steps[w] = 0;
            d.episode_start_x[w] = s.q[0];
            d.commanded_distance[w] = 0.0;
            refresh(s);
            if (!(st & SS_ST_OBS))
                for (int g = 0; g < d.n_groups; ++g) d.group[g].pending[w] = 1;
        }

        // ---- 6. CommandManager.update (managers/command.py:41-45)
        if ((st & SS_ST_COMMAND) && d.n_cmd > 0) {
            const int64_t cd = d.countdown[w] - 1;
            if (cd <= 0) resample_command(d, w, s);
            else d.countdown[w] = cd;
        }

        // ---- 7. EventManager.apply_interval (managers/event.py:103-114)
        if (st & SS_ST_EVENTS) {
            for (int e = 0; e < d.n_events; ++e) {
                const ss_event_term& E = d.event[e];
                if (E.mode != SS_MODE_INTERVAL) continue;
                double el = E.elapsed[w] + d.dt_control;
                const double tgt = E.target[w];
                const bool fire = el >= tgt - 0.5 * d.dt_control;
                if (fire) {
                    // registered Python terms run on the host for the fired ids
                    if (E.func != SS_EVT_EXTERNAL) apply_event(d, E, w, s);
                    el = 0.0;
                    E.target[w] = draw_interval_target(d, E, w);
                }
                if (E.fired) E.fired[w] = fire;
                E.elapsed[w] = el;
            }
        }

        // ---- 8. observations (post-reset state) (managers/observation.py:139-141)
        if (st & SS_ST_PREV_BEFORE) {
            d.prev_lin_vel_b[w] = s.lvb0;
            d.prev_lin_vel_b[N + w] = s.lvb1;
        }
        if (st & SS_ST_OBS) {
            ensure_action();
            uint32_t bad_bits = 0;
            for (int g = 0; g < d.n_groups; ++g) {
                if (!((u.groups_mask >> g) & 1u)) continue;
                bool pending = s.was_reset;
                if (u.any_pending) {
                    pending |= d.group[g].pending[w] != 0;
                    d.group[g].pending[w] = 0;
                }
                compute_group(d, u, g, w, s, pending, bad_bits);
            }
            d.obs_bad[w] = bad_bits;
        }
        if (st & SS_ST_PREV_AFTER) {
            d.prev_lin_vel_b[w] = s.lvb0;
            d.prev_lin_vel_b[N + w] = s.lvb1;
        }

        // ---- write back the physics state
        store_phys(d, w, s, /*store_cache=*/phys || s.was_reset);
    }

    // ---- warp-aggregated trigger counters (managers/termination.py:31-39)
    if (st & SS_ST_TERM) {
        const int lane = threadIdx.x & 31;
        for (int t = 0; t < d.n_terms; ++t) {
            const unsigned m = __ballot_sync(0xffffffffu, (s.trig_bits >> t) & 1u);
            if (lane == 0 && m) atomicAdd((unsigned long long*)&d.trigger_counts[t], (unsigned long long)__popc(m));
        }
        const unsigned m = __ballot_sync(0xffffffffu, (s.trig_bits >> 31) & 1u);
        if (lane == 0 && m) {
            atomicAdd((unsigned long long*)&d.trigger_counts[d.n_terms], (unsigned long long)__popc(m));
            // zero-copy flag in mapped pinned host memory: lets the host notice a
            // nonfinite step without a per-step device->host copy (env.py:240-241)
            if (d.nf_flags) *((volatile uint32_t*)&d.nf_flags[u.nf_slot]) = 1u;
        }
    }
}

// ---------------------------------------------------------------------------
// host-side dispatch

static thread_local char g_err[512] = "";

}  // namespace ss

using namespace ss;

extern "C" const char* ss_last_error(void) { return g_err; }

void ss_set_error(const char* what, const char* msg) { snprintf(g_err, sizeof(g_err), "%s: %s", what, msg); }

static int ss_fail(const char* what, cudaError_t e) {
    ss_set_error(what, cudaGetErrorString(e));
    return -1;
}

template <int KM, int FM>
static cudaError_t launch_step(const ss_env_desc& d, const ss_uniforms& u, cudaStream_t stream) {
    const int grid = (d.n_worlds + kBlock - 1) / kBlock;
    step_kernel<KM, FM><<<grid, kBlock, 0, stream>>>(d, u);
    return cudaGetLastError();
}

extern "C" int ss_abi_version(void) { return SS_ABI_VERSION; }

extern "C" size_t ss_sizeof(int which) {
    switch (which) {
        case 0: return sizeof(ss_env_desc);
        case 1: return sizeof(ss_uniforms);
        case 2: return sizeof(ss_rng_draw_args);
        default: return 0;
    }
}

extern "C" int ss_env_step(const ss_env_desc* desc, const ss_uniforms* u, void* stream) {
    if (!desc || !u) {
        snprintf(g_err, sizeof(g_err), "ss_env_step: null descriptor");
        return -2;
    }
    if (desc->abi_version != SS_ABI_VERSION) {
        snprintf(g_err, sizeof(g_err), "ss_env_step: abi version %d != %d", desc->abi_version, SS_ABI_VERSION);
        return -3;
    }
    if (desc->n_worlds <= 0) return 0;
    const int K = desc->model.n_joints, F = desc->model.n_feet;
    if (K > SS_MAX_JOINTS || F > SS_MAX_FEET || desc->hist_len > SS_MAX_HIST ||
        desc->action_dim > SS_MAX_ACTION || desc->n_terms > 31) {
        snprintf(g_err, sizeof(g_err), "ss_env_step: model exceeds compiled limits");
        return -4;
    }
    cudaStream_t s = (cudaStream_t)stream;
    cudaError_t e;
    if (K <= 4 && F <= 2) e = launch_step<4, 2>(*desc, *u, s);
    else if (K <= 12 && F <= 4) e = launch_step<12, 4>(*desc, *u, s);
    else e = launch_step<16, 8>(*desc, *u, s);
    if (e != cudaSuccess) return ss_fail("ss_env_step launch", e);
    return 0;
}
