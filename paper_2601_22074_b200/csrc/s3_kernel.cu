// s3_kernel.cu -- 3-D articulated-body step for sm_100a.
//
// One warp owns one world for the whole launch: its state and every
// per-world intermediate (frames, cinert/crb, cdof, the packed mass matrix and
// its factor, contacts, contact Jacobians, constraint rows) live in that
// warp's slice of shared memory; lanes split the work inside each stage
// (bodies of one tree level, dofs, geom pairs, ancestor pairs of the
// factorization, rows of the constraint problem) and __syncwarp() orders the
// stages. No block-level synchronisation: warps are independent worlds.
//
// The stages follow oracle/sim3d.py operation for operation (that file is the
// written specification; parity: tests/test_gpu_sim3d.py):
//   kinematics -> com/cinert/cdof -> CRB -> M (packed lower) -> tree-sparse
//   L^T D L -> comVel/RNE -> actuation -> qacc_smooth -> broadphase +
//   narrowphase -> limit + pyramidal contact rows -> Newton (dense Cholesky of
//   H = M + J^T D J, exact bracketed line search) -> implicitfast -> integrate.
// Templated on the element type (double: parity build; float: throughput).

#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <string.h>

#include <mutex>

#include "../../include/sim3d_b200.h"

namespace s3 {

constexpr unsigned FULL = 0xffffffffu;
constexpr int kGeomPlane = 0, kGeomHfield = 1, kGeomSphere = 2, kGeomCapsule = 3, kGeomBox = 6;
constexpr int kJntFree = 0;
constexpr int kActDC = 1, kActImplicit = 2;  // 0 = PD (the default branch)
constexpr int kConStride = 14;  // dist, pos[3], frame[9], mu

// layout slots (s3_layout.off)
enum {
    O_XPOS, O_XQUAT, O_XIPOS, O_CINERT, O_JANC, O_JAX, O_CRB, O_CDOF, O_CDOFD, O_CVEL, O_CACC,
    O_M, O_LD, O_QPOS, O_QVEL, O_SMOOTH, O_A0, O_A, O_MA, O_GRAD, O_P, O_MP, O_KVD, O_GPOS, O_GMAT,
    O_CON, O_JC, O_RAREF, O_RD, O_RJAR, O_RJP, O_CDOT, O_BIAS, O_FCON, O_CTRL, O_COM, O_CG, O_INT, O_END,
    O_INT_LIMDOF = O_END, O_INT_LIMSIGN  // int offsets inside O_INT (not element offsets)
};

__host__ __device__ inline int tri(int i, int j) { return ((i * (i + 1)) >> 1) + j; }  // packed lower, i >= j

template <class T> __device__ inline T wsum(T v) {
#pragma unroll
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
    return v;
}

template <class T> __device__ inline T rsqrt_t(T x);
template <> __device__ inline double rsqrt_t(double x) { return 1.0 / sqrt(x); }
template <> __device__ inline float rsqrt_t(float x) { return 1.0f / sqrtf(x); }

template <class T> __device__ inline void sincos_t(T x, T* s, T* c);
template <> __device__ inline void sincos_t(double x, double* s, double* c) { sincos(x, s, c); }
template <> __device__ inline void sincos_t(float x, float* s, float* c) { sincosf(x, s, c); }

// ---------------------------------------------------------------- small 3-D math (oracle/sim3d.py helpers)

template <class T> __device__ inline void qmul(const T* a, const T* b, T* r) {
    T w = a[0] * b[0] - a[1] * b[1] - a[2] * b[2] - a[3] * b[3];
    T x = a[0] * b[1] + a[1] * b[0] + a[2] * b[3] - a[3] * b[2];
    T y = a[0] * b[2] - a[1] * b[3] + a[2] * b[0] + a[3] * b[1];
    T z = a[0] * b[3] + a[1] * b[2] - a[2] * b[1] + a[3] * b[0];
    r[0] = w; r[1] = x; r[2] = y; r[3] = z;
}

template <class T> __device__ inline void qmat(const T* q, T* R) {
    T w = q[0], x = q[1], y = q[2], z = q[3];
    R[0] = T(1) - T(2) * (y * y + z * z); R[1] = T(2) * (x * y - w * z); R[2] = T(2) * (x * z + w * y);
    R[3] = T(2) * (x * y + w * z); R[4] = T(1) - T(2) * (x * x + z * z); R[5] = T(2) * (y * z - w * x);
    R[6] = T(2) * (x * z - w * y); R[7] = T(2) * (y * z + w * x); R[8] = T(1) - T(2) * (x * x + y * y);
}

template <class T> __device__ inline void mv3(const T* R, const T* v, T* r) {
    T a = R[0] * v[0] + R[1] * v[1] + R[2] * v[2];
    T b = R[3] * v[0] + R[4] * v[1] + R[5] * v[2];
    T c = R[6] * v[0] + R[7] * v[1] + R[8] * v[2];
    r[0] = a; r[1] = b; r[2] = c;
}

template <class T> __device__ inline void mm3(const T* A, const T* B, T* C) {
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j) C[3 * i + j] = A[3 * i] * B[j] + A[3 * i + 1] * B[3 + j] + A[3 * i + 2] * B[6 + j];
}

template <class T> __device__ inline void cross3(const T* a, const T* b, T* r) {
    T x = a[1] * b[2] - a[2] * b[1];
    T y = a[2] * b[0] - a[0] * b[2];
    T z = a[0] * b[1] - a[1] * b[0];
    r[0] = x; r[1] = y; r[2] = z;
}

template <class T> __device__ inline T dot3(const T* a, const T* b) { return a[0] * b[0] + a[1] * b[1] + a[2] * b[2]; }

template <class T> __device__ inline T dot6(const T* a, const T* b) {
    return a[0] * b[0] + a[1] * b[1] + a[2] * b[2] + a[3] * b[3] + a[4] * b[4] + a[5] * b[5];
}

template <class T> __device__ inline void qnormalize(T* q) {
    T r = rsqrt_t(q[0] * q[0] + q[1] * q[1] + q[2] * q[2] + q[3] * q[3]);
    q[0] *= r; q[1] *= r; q[2] *= r; q[3] *= r;
}

// motion x motion: [w x u_ang ; w x u_lin + v_lin x u_ang]
template <class T> __device__ inline void cross_motion(const T* v, const T* u, T* r) {
    T a[3], b[3], c[3];
    cross3(v, u, a);
    cross3(v, u + 3, b);
    cross3(v + 3, u, c);
    r[0] = a[0]; r[1] = a[1]; r[2] = a[2];
    r[3] = b[0] + c[0]; r[4] = b[1] + c[1]; r[5] = b[2] + c[2];
}

// motion x force: [w x f_ang + v_lin x f_lin ; w x f_lin]
template <class T> __device__ inline void cross_force(const T* v, const T* f, T* r) {
    T a[3], b[3], c[3];
    cross3(v, f, a);
    cross3(v + 3, f + 3, b);
    cross3(v, f + 3, c);
    r[0] = a[0] + b[0]; r[1] = a[1] + b[1]; r[2] = a[2] + b[2];
    r[3] = c[0]; r[4] = c[1]; r[5] = c[2];
}

// 10-vector spatial inertia times motion
template <class T> __device__ inline void inert_mul(const T* ci, const T* v, T* r) {
    const T* w = v;
    const T* vl = v + 3;
    T md[3] = {ci[6], ci[7], ci[8]};
    T a[3], b[3];
    cross3(md, vl, a);
    cross3(md, w, b);
    r[0] = ci[0] * w[0] + ci[3] * w[1] + ci[4] * w[2] + a[0];
    r[1] = ci[3] * w[0] + ci[1] * w[1] + ci[5] * w[2] + a[1];
    r[2] = ci[4] * w[0] + ci[5] * w[1] + ci[2] * w[2] + a[2];
    r[3] = ci[9] * vl[0] - b[0];
    r[4] = ci[9] * vl[1] - b[1];
    r[5] = ci[9] * vl[2] - b[2];
}

template <class T> __device__ inline T clampt(T x, T lo, T hi) { return x < lo ? lo : (x > hi ? hi : x); }

// ---------------------------------------------------------------- per-warp workspace

template <class T> struct WS {
    T *xpos, *xquat, *xipos, *cinert, *crb, *cdof, *cdofd, *cvel, *cacc, *janc, *jax, *M, *LD, *qpos, *qvel,
        *smooth, *a0, *a, *Ma, *grad, *p, *Mp, *kvd, *con, *Jc, *raref, *rD, *rjar, *rJp, *cdot,
        *bias, *fcon, *ctrl, *com, *tk, *snap, *cgm;
    int *con_pair, *lim_dof, *lim_sign;
};

template <class T> __device__ inline WS<T> make_ws(T* base, const s3_layout& l) {
    WS<T> s;
    const int* o = l.off;
    s.xpos = base + o[O_XPOS]; s.xquat = base + o[O_XQUAT]; s.xipos = base + o[O_XIPOS];
    s.cinert = base + o[O_CINERT]; s.crb = s.cinert; s.cdof = base + o[O_CDOF];
    s.tk = base + o[O_CRB];  // per-dof scratch of the level-schedule factorization (flags bit 1) only
    s.janc = base + o[O_JANC]; s.jax = base + o[O_JAX];
    // factorization snapshot (rows touched by constraints, tree entries): xipos, cinert, janc, jax are
    // contiguous and dead from the end of the mass-matrix build until the next substep's kinematics
    s.snap = s.xipos;
    // RNE scratch lives in the contact-Jacobian region (dead until build_rows)
    s.cdofd = base + o[O_JC]; s.cvel = s.cdofd + o[O_CDOFD]; s.cacc = s.cvel + o[O_CVEL];
    s.M = base + o[O_M]; s.LD = base + o[O_LD]; s.qpos = base + o[O_QPOS]; s.qvel = base + o[O_QVEL];
    s.smooth = base + o[O_SMOOTH]; s.a = base + o[O_A]; s.Ma = base + o[O_MA];
    s.grad = base + o[O_GRAD]; s.p = base + o[O_P]; s.Mp = base + o[O_MP]; s.kvd = base + o[O_KVD];
    s.a0 = s.Mp;  // qacc_smooth: parity outputs only, written before Newton (which reuses Mp as scratch)
    s.con = base + o[O_CON]; s.Jc = base + o[O_JC];
    s.raref = base + o[O_RAREF]; s.rD = base + o[O_RD]; s.rjar = base + o[O_RJAR]; s.rJp = base + o[O_RJP];
    s.cdot = base + o[O_CDOT]; s.bias = s.Ma;  // bias: RNE -> smooth_force, dead before Newton writes Ma
    s.fcon = base + o[O_FCON]; s.ctrl = base + o[O_CTRL];
    s.com = base + o[O_COM];
    s.cgm = base + o[O_CG];  // CG solver (flags bit 7): M^-1 grad, and its previous value
    int* ib = reinterpret_cast<int*>(base + o[O_INT]);
    s.con_pair = ib;
    s.lim_dof = ib + o[O_INT_LIMDOF];  // int offsets inside the int region, sized by ncon_max / nlimjnt
    s.lim_sign = ib + o[O_INT_LIMSIGN];
    return s;
}

template <class T> __device__ inline const T* F(const void* p) { return static_cast<const T*>(p); }

// The model of the launch, copied into constant memory ahead of each step kernel on the launching stream.
// The physics stages read it from here instead of through a reference to the kernel's grid-constant
// parameter: that reference is a generic pointer, so every table pointer read inside a loop that stores to
// shared memory was reloaded each iteration; constant-bank reads are cached and may be hoisted.
__constant__ s3_model c_s3m;
// The kinematics / dynamics / collision / row-building stages and Newton read the constant-bank copy in
// both builds; the factorization, solves, row products, cost and substep driver read it in float64 only
// (-5.5 % per G1 control step, -7 % motion imitation) -- in float32 the hoisted constant-bank reads there
// raised register pressure and spills (+7.5 %), while the first group alone is -3.5 %.
template <class T> __device__ __forceinline__ const s3_model& model_ref(const s3_model& param) {
    if constexpr (sizeof(T) == 8) return c_s3m;
    else return param;
}

// ---------------------------------------------------------------- stages

// mj_kinematics: body frames level by level (oracle kinematics)
template <class T> __device__ void __noinline__ kinematics(const s3_model& m_, const s3_layout& L_, T* B_, int lane) {
    const s3_model& m = c_s3m;  // constant-bank model (both dtypes; see c_s3m)
    WS<T> s = make_ws(B_, L_);
    const T* bpos = F<T>(m.body_pos);
    const T* bquat = F<T>(m.body_quat);
    const T* jpos = F<T>(m.jnt_pos);
    const T* jaxis = F<T>(m.jnt_axis);
    const T* q0 = F<T>(m.qpos0);
    if (lane == 0) {
        s.xpos[0] = s.xpos[1] = s.xpos[2] = T(0);
        s.xquat[0] = T(1); s.xquat[1] = s.xquat[2] = s.xquat[3] = T(0);
    }
    __syncwarp();
    for (int L = 1; L < m.nlevel; ++L) {
        for (int idx = m.level_ptr[L] + lane; idx < m.level_ptr[L + 1]; idx += 32) {
            int b = m.level_body[idx];
            int par = m.body_parentid[b];
            T pq[4] = {s.xquat[4 * par], s.xquat[4 * par + 1], s.xquat[4 * par + 2], s.xquat[4 * par + 3]};
            T R[9], pos[3], quat[4], v[3];
            qmat(pq, R);
            T bp[3] = {bpos[3 * b], bpos[3 * b + 1], bpos[3 * b + 2]};
            mv3(R, bp, v);
            pos[0] = s.xpos[3 * par] + v[0]; pos[1] = s.xpos[3 * par + 1] + v[1]; pos[2] = s.xpos[3 * par + 2] + v[2];
            T bq[4] = {bquat[4 * b], bquat[4 * b + 1], bquat[4 * b + 2], bquat[4 * b + 3]};
            qmul(pq, bq, quat);
            int j0 = m.body_jntadr[b], jn = m.body_jntnum[b];
            for (int j = j0; j < j0 + jn; ++j) {
                int a = m.jnt_qposadr[j];
                if (m.jnt_type[j] == kJntFree) {
                    pos[0] = s.qpos[a]; pos[1] = s.qpos[a + 1]; pos[2] = s.qpos[a + 2];
                    quat[0] = s.qpos[a + 3]; quat[1] = s.qpos[a + 4]; quat[2] = s.qpos[a + 5]; quat[3] = s.qpos[a + 6];
                    qnormalize(quat);
                    s.janc[3 * j] = pos[0]; s.janc[3 * j + 1] = pos[1]; s.janc[3 * j + 2] = pos[2];
                    s.jax[3 * j] = T(0); s.jax[3 * j + 1] = T(0); s.jax[3 * j + 2] = T(1);
                } else {
                    T jp[3] = {jpos[3 * j], jpos[3 * j + 1], jpos[3 * j + 2]};
                    T ja[3] = {jaxis[3 * j], jaxis[3 * j + 1], jaxis[3 * j + 2]};
                    T anc[3], ax[3];
                    qmat(quat, R);
                    mv3(R, jp, anc);
                    anc[0] += pos[0]; anc[1] += pos[1]; anc[2] += pos[2];
                    mv3(R, ja, ax);
                    s.janc[3 * j] = anc[0]; s.janc[3 * j + 1] = anc[1]; s.janc[3 * j + 2] = anc[2];
                    s.jax[3 * j] = ax[0]; s.jax[3 * j + 1] = ax[1]; s.jax[3 * j + 2] = ax[2];
                    T sn, cs;
                    sincos_t(T(0.5) * (s.qpos[a] - q0[a]), &sn, &cs);
                    T qa[4] = {cs, ja[0] * sn, ja[1] * sn, ja[2] * sn};
                    T nq[4];
                    qmul(quat, qa, nq);
                    quat[0] = nq[0]; quat[1] = nq[1]; quat[2] = nq[2]; quat[3] = nq[3];
                    qmat(quat, R);
                    mv3(R, jp, v);
                    pos[0] = anc[0] - v[0]; pos[1] = anc[1] - v[1]; pos[2] = anc[2] - v[2];
                }
            }
            qnormalize(quat);
            s.xquat[4 * b] = quat[0]; s.xquat[4 * b + 1] = quat[1]; s.xquat[4 * b + 2] = quat[2];
            s.xquat[4 * b + 3] = quat[3];
            s.xpos[3 * b] = pos[0]; s.xpos[3 * b + 1] = pos[1]; s.xpos[3 * b + 2] = pos[2];
        }
        __syncwarp();
    }
}

// mj_comPos: xipos, subtree com (single tree), cinert, cdof; geom frames
template <class T> __device__ void __noinline__ com_pos(const s3_model& m_, const s3_layout& L_, T* B_, int lane, T ms) {
    const s3_model& m = c_s3m;  // constant-bank model (both dtypes; see c_s3m)
    WS<T> s = make_ws(B_, L_);
    const T* ipos = F<T>(m.body_ipos);
    const T* ilmat = F<T>(m.body_ilmat);
    const T* mass = F<T>(m.body_mass);
    const T* inertia = F<T>(m.body_inertia);
    for (int b = 1 + lane; b < m.nbody; b += 32) {
        T R[9], v[3];
        qmat(s.xquat + 4 * b, R);
        T ip[3] = {ipos[3 * b], ipos[3 * b + 1], ipos[3 * b + 2]};
        mv3(R, ip, v);
        s.xipos[3 * b] = s.xpos[3 * b] + v[0];
        s.xipos[3 * b + 1] = s.xpos[3 * b + 1] + v[1];
        s.xipos[3 * b + 2] = s.xpos[3 * b + 2] + v[2];
    }
    __syncwarp();
    // subtree com of every kinematic tree (each tree's c-frame origin); body 1's mass scaled by ms
    const T* tmass = F<T>(m.tree_mass);
    for (int t = 0; t < m.nkintree; ++t) {
        T cx = T(0), cy = T(0), cz = T(0);
        for (int b = 1 + lane; b < m.nbody; b += 32) {
            if (m.body_treeid[b] != t) continue;
            T mb = b == 1 ? mass[b] * ms : mass[b];
            cx += mb * s.xipos[3 * b]; cy += mb * s.xipos[3 * b + 1]; cz += mb * s.xipos[3 * b + 2];
        }
        T inv = T(1) / (m.body_treeid[1] == t ? tmass[t] + (mass[1] * ms - mass[1]) : tmass[t]);
        cx = wsum(cx) * inv; cy = wsum(cy) * inv; cz = wsum(cz) * inv;
        if (lane == 0) { s.com[3 * t] = cx; s.com[3 * t + 1] = cy; s.com[3 * t + 2] = cz; }
    }
    __syncwarp();
    for (int b = 1 + lane; b < m.nbody; b += 32) {
        T R[9], Ri[9], IL[9];
        qmat(s.xquat + 4 * b, R);
        for (int k = 0; k < 9; ++k) IL[k] = ilmat[9 * b + k];
        mm3(R, IL, Ri);
        const T sb = b == 1 ? ms : T(1);
        T i0 = inertia[3 * b] * sb, i1 = inertia[3 * b + 1] * sb, i2 = inertia[3 * b + 2] * sb;
        // I = Ri diag(i) Ri^T
        T I[9];
#pragma unroll
        for (int r = 0; r < 3; ++r)
#pragma unroll
            for (int c = 0; c < 3; ++c) I[3 * r + c] = Ri[3 * r] * i0 * Ri[3 * c] + Ri[3 * r + 1] * i1 * Ri[3 * c + 1] +
                                                     Ri[3 * r + 2] * i2 * Ri[3 * c + 2];
        const T* com = s.com + 3 * m.body_treeid[b];
        T d[3] = {s.xipos[3 * b] - com[0], s.xipos[3 * b + 1] - com[1], s.xipos[3 * b + 2] - com[2]};
        T mb = b == 1 ? mass[b] * ms : mass[b];
        T dd = dot3(d, d);
        T* ci = s.cinert + 10 * b;
        ci[0] = I[0] + mb * (dd - d[0] * d[0]);
        ci[1] = I[4] + mb * (dd - d[1] * d[1]);
        ci[2] = I[8] + mb * (dd - d[2] * d[2]);
        ci[3] = I[1] + mb * (T(0) - d[0] * d[1]);
        ci[4] = I[2] + mb * (T(0) - d[0] * d[2]);
        ci[5] = I[5] + mb * (T(0) - d[1] * d[2]);
        ci[6] = mb * d[0]; ci[7] = mb * d[1]; ci[8] = mb * d[2]; ci[9] = mb;
    }
    // cdof, per joint
    for (int j = lane; j < m.njnt; j += 32) {
        int da = m.jnt_dofadr[j];
        const T* com = s.com + 3 * m.body_treeid[m.dof_bodyid[da]];
        T off[3] = {com[0] - s.janc[3 * j], com[1] - s.janc[3 * j + 1], com[2] - s.janc[3 * j + 2]};
        if (m.jnt_type[j] == kJntFree) {
            int b = m.dof_bodyid[da];
            T R[9];
            qmat(s.xquat + 4 * b, R);
            for (int i = 0; i < 3; ++i) {
                T* c = s.cdof + 6 * (da + i);
                c[0] = c[1] = c[2] = T(0);
                c[3] = T(i == 0); c[4] = T(i == 1); c[5] = T(i == 2);
                T ax[3] = {R[i], R[3 + i], R[6 + i]};
                T lin[3];
                cross3(ax, off, lin);
                T* r = s.cdof + 6 * (da + 3 + i);
                r[0] = ax[0]; r[1] = ax[1]; r[2] = ax[2]; r[3] = lin[0]; r[4] = lin[1]; r[5] = lin[2];
            }
        } else {
            T ax[3] = {s.jax[3 * j], s.jax[3 * j + 1], s.jax[3 * j + 2]};
            T lin[3];
            cross3(ax, off, lin);
            T* r = s.cdof + 6 * da;
            r[0] = ax[0]; r[1] = ax[1]; r[2] = ax[2]; r[3] = lin[0]; r[4] = lin[1]; r[5] = lin[2];
        }
    }
    __syncwarp();
}

// mj_crb: composite inertias (levels, deepest first, children in descending index) + packed M.
// Accumulates in place over cinert (RNE, the only other reader of cinert, has already run).
template <class T> __device__ void __noinline__ crb_mass(const s3_model& m_, const s3_layout& L_, T* B_, int lane) {
    const s3_model& m = c_s3m;  // constant-bank model (both dtypes; see c_s3m)
    WS<T> s = make_ws(B_, L_);
    for (int L = m.nlevel - 2; L >= 1; --L) {
        int n0 = m.level_ptr[L], nl = m.level_ptr[L + 1] - n0;
        for (int t = lane; t < nl * 10; t += 32) {
            int b = m.level_body[n0 + t / 10], c = t % 10;
            int k0 = m.child_ptr[b], k1 = m.child_ptr[b + 1];
            if (k0 == k1) continue;
            T acc = s.crb[10 * b + c];
            for (int k = k0; k < k1; ++k) acc += s.crb[10 * m.child_idx[k] + c];
            s.crb[10 * b + c] = acc;
        }
        __syncwarp();
    }
    const T* arm = F<T>(m.dof_armature);
    int nv = m.nv;
    int np = nv * (nv + 1) / 2;
    for (int t = lane; t < np; t += 32) s.M[t] = T(0);
    __syncwarp();
    for (int i = lane; i < nv; i += 32) {
        T f[6];
        inert_mul(s.crb + 10 * m.dof_bodyid[i], s.cdof + 6 * i, f);
        int j = i;
        while (j >= 0) {
            s.M[tri(i, j)] = dot6(s.cdof + 6 * j, f);
            j = m.dof_parentid[j];
        }
        s.M[tri(i, i)] += arm[i];
    }
    __syncwarp();
}

// mj_factorM: tree-sparse L^T D L in place on packed-lower A (oracle factor_ldl).
// Step k applies the Schur updates A[i][j] -= (A[k][i] / D[k]) A[k][j] for the (i, j) pairs of its
// precomputed list, one pair per lane, reading row k UNnormalised; row k is never read again by a later
// step (those only touch rows of ancestors), so rows are normalised in one pass at the end: one barrier
// per dof. `sel` restricts the elimination to the dofs outside (1) or inside (2) the ancestor-closed set
// U (0: all): subtrees outside U eliminate identically for M and for H = M + J^T D J when every
// constraint row lives on U, so Newton refactors only U (eliminations of disjoint subtrees commute).
template <class T>
__device__ __noinline__ void factor_ldl(const s3_model& m_, T* A, T* rk, int lane, uint64_t U = 0, int sel = 0) {
    const s3_model& m = model_ref<T>(m_);  // float64: the constant-bank copy (see c_s3m)
    if (m.flags & 4) {
        // mask-level schedule: lane owns dof rows i in {lane, lane + 32}; at height level h it applies
        // the Schur updates of the level's dofs k that descend from i to its row (j in chain(i)). Rows of
        // level-h dofs are final (their descendants sit lower) and are only read; no table loads.
        const uint64_t all = m.nv == 64 ? ~0ull : ((1ull << m.nv) - 1);
        const uint64_t selm = sel == 0 ? all : (sel == 1 ? (~U & all) : (U & all));
        const unsigned long long* cm = reinterpret_cast<const unsigned long long*>(m.dof_chainmask);
        const unsigned long long* dmk = reinterpret_cast<const unsigned long long*>(m.dof_descmask);
        const unsigned long long* hm = reinterpret_cast<const unsigned long long*>(m.hlev_mask);
        const int i0 = lane, i1 = lane + 32;
        const uint64_t am0 = i0 < m.nv ? __ldg(cm + i0) : 0, am1 = i1 < m.nv ? __ldg(cm + i1) : 0;
        const uint64_t dm0 = i0 < m.nv ? __ldg(dmk + i0) : 0, dm1 = i1 < m.nv ? __ldg(dmk + i1) : 0;
        for (int h = 0; h < m.nhlev; ++h) {
            const uint64_t lm = __ldg(hm + h) & selm;
            if (!lm) continue;
#pragma unroll
            for (int half = 0; half < 2; ++half) {
                const int i = half ? i1 : i0;
                uint64_t ks = (half ? dm1 : dm0) & lm;
                const uint64_t am = half ? am1 : am0;
                while (ks) {
                    const int k = __ffsll((long long)ks) - 1;
                    ks &= ks - 1;
                    const int rkb = tri(k, 0);
                    const T t = A[rkb + i] / A[rkb + k];
                    const int rib = tri(i, 0);
                    uint64_t js = am;
                    while (js) {
                        const int j = __ffsll((long long)js) - 1;
                        js &= js - 1;
                        A[rib + j] -= t * A[rkb + j];
                    }
                }
            }
            __syncwarp();
        }
        // normalise the selected rows: L[k][i] = A[k][i] / D[k] for strict ancestors i
#pragma unroll
        for (int half = 0; half < 2; ++half) {
            const int k = half ? i1 : i0;
            if (k >= m.nv || !((selm >> k) & 1ull)) continue;
            const int rkb = tri(k, 0);
            const T dk = A[rkb + k];
            uint64_t is = (half ? am1 : am0) & ~(1ull << k);
            while (is) {
                const int i = __ffsll((long long)is) - 1;
                is &= is - 1;
                A[rkb + i] = A[rkb + i] / dk;
            }
        }
        __syncwarp();
        return;
    }
    if (m.flags & 2) {
        // level schedule (opt-in, flags bit 1; measured SLOWER than the sequential sweep below -- 6.6 vs
        // 5.2 ms f32, 11.1 vs 8.0 ms f64 per G1 control step -- because each entry chains three dependent
        // table loads that miss the small L1 left beside 224 KB of shared memory): every dof of one height
        // level eliminates in the same step (none is an ancestor of another, and their Schur updates to
        // shared ancestor entries add); one barrier per level.
        // rk[k] = 1 / D[k]: set for every dof up front (final for leaves) and refreshed by the lane that
        // applies the last update of A[k][k] (level height(k) - 1), so no division per contribution.
        for (int k = lane; k < m.nv; k += 32) rk[k] = T(1) / A[tri(k, k)];
        __syncwarp();
        for (int L = 0; L < m.nhlev; ++L) {
            const int e0 = __ldg(m.fl_ptr + L), e1 = __ldg(m.fl_ptr + L + 1);
            for (int e = e0 + lane; e < e1; e += 32) {
                const int pr = __ldg(m.fl_ent + e);
                const int i = pr >> 8, j = pr & 255;
                const int c0 = __ldg(m.fl_kptr + e), c1 = __ldg(m.fl_kptr + e + 1);
                T acc = T(0);
                for (int c = c0; c < c1; ++c) {
                    const int k = __ldg(m.fl_k + c);
                    if (sel && (int)((U >> k) & 1ull) != (sel == 2)) continue;
                    const int rkb = tri(k, 0);
                    acc += (A[rkb + i] * rk[k]) * A[rkb + j];
                }
                const T v = A[tri(i, j)] - acc;
                A[tri(i, j)] = v;
                if (i == j) rk[i] = T(1) / v;
            }
            __syncwarp();
        }
        for (int t = lane; t < m.nldl_norm; t += 32) {
            int pr = __ldg(m.ldl_norm + t);
            int k = pr >> 8, i = pr & 255;
            if (sel && (int)((U >> k) & 1ull) != (sel == 2)) continue;
            A[tri(k, i)] = A[tri(k, i)] / A[tri(k, k)];
        }
        __syncwarp();
        return;
    }
    // dofs with ancestors (dof_parentid >= 0 <=> nonempty update list), restricted to the selection,
    // visited from the highest index down through the bit mask
    const uint64_t all = m.nv == 64 ? ~0ull : ((1ull << m.nv) - 1);
    uint64_t todo = (sel == 0 ? all : (sel == 1 ? (~U & all) : (U & all))) & m.nonroot_mask;
    // table pointers in registers: through `m` (a generic reference to the grid-constant block) every
    // use is a reload the compiler cannot hoist past the shared-memory stores
    const int32_t* __restrict__ lptr = m.ldl_ptr;
    const uint16_t* __restrict__ lpair = m.ldl_pair;
    const uint16_t* __restrict__ lnorm = m.ldl_norm;
    const int nnorm = m.nldl_norm;
    while (todo) {
        const int k = 63 - __clzll((long long)todo);
        todo &= ~(1ull << k);
        const int p0 = __ldg(lptr + k), p1 = __ldg(lptr + k + 1);
        T rk = T(1) / A[tri(k, k)];
        int rkb = tri(k, 0);
        for (int t = p0 + lane; t < p1; t += 32) {
            int pr = __ldg(lpair + t);
            int i = pr >> 8, j = pr & 255;
            A[tri(i, j)] -= (A[rkb + i] * rk) * A[rkb + j];
        }
        __syncwarp();
    }
    for (int t = lane; t < nnorm; t += 32) {
        int pr = __ldg(lnorm + t);
        int k = pr >> 8, i = pr & 255;
        if (sel && (int)((U >> k) & 1ull) != (sel == 2)) continue;
        A[tri(k, i)] = A[tri(k, i)] / A[tri(k, k)];
    }
    __syncwarp();
}

// tree entries (i, j in chain(i)) of the rows in U: A -> snap (save) or snap -> A (restore); all rows if U = ~0
template <class T>
__device__ __noinline__ void tree_copy(const s3_model& m_, T* A, T* snap, uint64_t U, bool save, int lane) {
    const s3_model& m = model_ref<T>(m_);  // float64: the constant-bank copy (see c_s3m)
    const uint16_t* __restrict__ ent = m.tree_ent;
    const int n = m.ntree;
    for (int t = lane; t < n; t += 32) {
        int pr = __ldg(ent + t);
        int i = pr >> 8, j = pr & 255;
        if (!((U >> i) & 1ull)) continue;
        if (save) snap[t] = A[tri(i, j)];
        else A[tri(i, j)] = snap[t];
    }
    __syncwarp();
}

// copy the tree entries of M into A (everything a tree factorization / solve reads)
template <class T> __device__ __noinline__ void tree_load(const s3_model& m_, const T* M, T* A, int lane) {
    const s3_model& m = model_ref<T>(m_);  // float64: the constant-bank copy (see c_s3m)
    const uint16_t* __restrict__ ent = m.tree_ent;
    const int n = m.ntree;
    for (int t = lane; t < n; t += 32) {
        int pr = __ldg(ent + t);
        int k = tri(pr >> 8, pr & 255);
        A[k] = M[k];
    }
    __syncwarp();
}

// x <- M^-1 x with the L^T D L factor (oracle solve_ldl; column-oriented forward pass)
template <class T> __device__ __noinline__ void solve_ldl(const s3_model& m_, const T* A, T* x, int lane) {
    const s3_model& m = model_ref<T>(m_);  // float64: the constant-bank copy (see c_s3m)
    int nv = m.nv;
    if (m.flags & 4) {
        // mask-level sweeps (see factor_ldl): leaf-to-root by height, each lane's dofs j gather the level's
        // descendants; root-to-leaf by depth, each lane's dof gathers its (final) ancestors
        const unsigned long long* cm = reinterpret_cast<const unsigned long long*>(m.dof_chainmask);
        const unsigned long long* dmk = reinterpret_cast<const unsigned long long*>(m.dof_descmask);
        const unsigned long long* hm = reinterpret_cast<const unsigned long long*>(m.hlev_mask);
        const unsigned long long* dlm = reinterpret_cast<const unsigned long long*>(m.dlev_mask);
        const int i0 = lane, i1 = lane + 32;
        const uint64_t am0 = i0 < nv ? __ldg(cm + i0) : 0, am1 = i1 < nv ? __ldg(cm + i1) : 0;
        const uint64_t dm0 = i0 < nv ? __ldg(dmk + i0) : 0, dm1 = i1 < nv ? __ldg(dmk + i1) : 0;
        for (int h = 0; h < m.nhlev; ++h) {
            const uint64_t lm = __ldg(hm + h);
#pragma unroll
            for (int half = 0; half < 2; ++half) {
                const int j = half ? i1 : i0;
                uint64_t src = (half ? dm1 : dm0) & lm;
                if (!src) continue;
                T acc = T(0);
                while (src) {
                    const int i = __ffsll((long long)src) - 1;
                    src &= src - 1;
                    acc += A[tri(i, j)] * x[i];
                }
                x[j] -= acc;
            }
            __syncwarp();
        }
        if (i0 < nv) x[i0] = x[i0] / A[tri(i0, i0)];
        if (i1 < nv) x[i1] = x[i1] / A[tri(i1, i1)];
        __syncwarp();
        for (int dl = 1; dl < m.ndlev; ++dl) {
            const uint64_t lm = __ldg(dlm + dl);
#pragma unroll
            for (int half = 0; half < 2; ++half) {
                const int i = half ? i1 : i0;
                if (i >= nv || !((lm >> i) & 1ull)) continue;
                uint64_t anc = (half ? am1 : am0) & ~(1ull << i);
                const int rb = tri(i, 0);
                T acc = T(0);
                while (anc) {
                    const int j = __ffsll((long long)anc) - 1;
                    anc &= anc - 1;
                    acc += A[rb + j] * x[j];
                }
                x[i] -= acc;
            }
            __syncwarp();
        }
        return;
    }
    if (m.flags & 2) {
        // leaf-to-root sweep by height levels: each target ancestor gathers the contributions of the
        // level's dofs (their values are final: all their descendants sit in lower levels)
        for (int L = 0; L < m.nhlev; ++L) {
            const int e0 = __ldg(m.bl_ptr + L), e1 = __ldg(m.bl_ptr + L + 1);
            for (int e = e0 + lane; e < e1; e += 32) {
                const int j = __ldg(m.bl_ent + e);
                const int c0 = __ldg(m.bl_iptr + e), c1 = __ldg(m.bl_iptr + e + 1);
                T acc = T(0);
                for (int c = c0; c < c1; ++c) {
                    const int i = __ldg(m.bl_i + c);
                    acc += A[tri(i, j)] * x[i];
                }
                x[j] -= acc;
            }
            __syncwarp();
        }
        for (int i = lane; i < nv; i += 32) x[i] = x[i] / A[tri(i, i)];
        __syncwarp();
        // root-to-leaf sweep by depth levels: each dof gathers over its (final) ancestors
        for (int L = 1; L < m.ndlev; ++L) {
            const int d0 = __ldg(m.fw_ptr + L), d1 = __ldg(m.fw_ptr + L + 1);
            for (int t = d0 + lane; t < d1; t += 32) {
                const int i = __ldg(m.fw_dof + t);
                const int len = __ldg(m.dof_chainlen + i) - 1;
                const uint8_t* ch = m.dof_chain + i * S3_MAX_CHAIN;
                const int rb = tri(i, 0);
                T acc = T(0);
                for (int a = 0; a < len; ++a) acc += A[rb + __ldg(ch + a)] * x[__ldg(ch + a)];
                x[i] -= acc;
            }
            __syncwarp();
        }
        return;
    }
    // register sweeps: lane l holds x[l] and x[l + 32]; step k broadcasts the (final) x[k] with a shuffle and
    // every lane applies its own update, so the serial chain per dof is shuffle -> FMA instead of a shared
    // memory store / barrier / load round trip; the factor entries and masks do not depend on x and are
    // loaded ahead. Same operations in the same order per entry as the reference sweeps (bit-identical).
    const unsigned long long* cm = reinterpret_cast<const unsigned long long*>(m.dof_chainmask);
    const unsigned long long* dmk = reinterpret_cast<const unsigned long long*>(m.dof_descmask);
    const int i0 = lane, i1 = lane + 32;
    const bool two = nv > 32;
    T x0 = i0 < nv ? x[i0] : T(0);
    T x1 = (two && i1 < nv) ? x[i1] : T(0);
    // leaf-to-root: x[j] -= L[i][j] x[i] over the ancestors j of i, i from the highest index down
#pragma unroll 4
    for (int i = nv - 1; i >= 1; --i) {
        const uint64_t anc = __ldg(cm + i) & ~(1ull << i);
        const int rb = tri(i, 0);
        const bool u0 = (anc >> i0) & 1ull, u1 = two && ((anc >> i1) & 1ull);
        const T a0 = u0 ? A[rb + i0] : T(0);
        const T a1 = u1 ? A[rb + i1] : T(0);
        const T s0 = __shfl_sync(FULL, x0, i & 31);
        const T s1 = two ? __shfl_sync(FULL, x1, i & 31) : T(0);
        const T xi = i < 32 ? s0 : s1;
        if (u0) x0 -= a0 * xi;
        if (u1) x1 -= a1 * xi;
    }
    if (i0 < nv) x0 = x0 / A[tri(i0, i0)];
    if (two && i1 < nv) x1 = x1 / A[tri(i1, i1)];
    // root-to-leaf: x[i] -= L[i][j] x[j] over the descendants i of j, j from the lowest index up
#pragma unroll 4
    for (int j = 0; j < nv - 1; ++j) {
        const uint64_t dm = __ldg(dmk + j);
        const bool u0 = (dm >> i0) & 1ull, u1 = two && ((dm >> i1) & 1ull);
        const T a0 = u0 ? A[tri(i0, j)] : T(0);
        const T a1 = u1 ? A[tri(i1, j)] : T(0);
        const T s0 = __shfl_sync(FULL, x0, j & 31);
        const T s1 = two ? __shfl_sync(FULL, x1, j & 31) : T(0);
        const T xj = j < 32 ? s0 : s1;
        if (u0) x0 -= a0 * xj;
        if (u1) x1 -= a1 * xj;
    }
    if (i0 < nv) x[i0] = x0;
    if (two && i1 < nv) x[i1] = x1;
    __syncwarp();
}

// dense Cholesky H = L L^T on packed lower (oracle cholesky), then x <- H^-1 x
template <class T> __device__ __noinline__ void cholesky(int nv, T* H, int lane) {
    for (int k = 0; k < nv; ++k) {
        T d = sqrt(H[tri(k, k)]);
        for (int i = k + 1 + lane; i < nv; i += 32) H[tri(i, k)] = H[tri(i, k)] / d;
        __syncwarp();
        if (lane == 0) H[tri(k, k)] = d;
        for (int i = k + 1 + lane; i < nv; i += 32) {
            T lik = H[tri(i, k)];
            int ri = tri(i, 0);
            for (int j = k + 1; j <= i; ++j) H[ri + j] -= lik * H[tri(j, k)];
        }
        __syncwarp();
    }
}

template <class T> __device__ __noinline__ void chol_solve(int nv, const T* L, T* x, int lane) {
    for (int i = 0; i < nv; ++i) {
        T xi = x[i] / L[tri(i, i)];
        __syncwarp();
        if (lane == 0) x[i] = xi;
        for (int r = i + 1 + lane; r < nv; r += 32) x[r] -= L[tri(r, i)] * xi;
        __syncwarp();
    }
    for (int i = nv - 1; i >= 0; --i) {
        T xi = x[i] / L[tri(i, i)];
        __syncwarp();
        if (lane == 0) x[i] = xi;
        for (int r = lane; r < i; r += 32) x[r] -= L[tri(i, r)] * xi;
        __syncwarp();
    }
}

// y = M x with packed-lower symmetric M
template <class T> __device__ __noinline__ void sym_mul(int nv, const T* M, const T* x, T* y, int lane) {
    for (int i = lane; i < nv; i += 32) {
        T acc = T(0);
        for (int j = 0; j < nv; ++j) acc += (i >= j ? M[tri(i, j)] : M[tri(j, i)]) * x[j];
        y[i] = acc;
    }
    __syncwarp();
}

// mj_comVel + mj_rne (qacc = 0): bias forces
template <class T> __device__ void __noinline__ rne(const s3_model& m_, const s3_layout& L_, T* B_, int lane) {
    const s3_model& m = c_s3m;  // constant-bank model (both dtypes; see c_s3m)
    WS<T> s = make_ws(B_, L_);
    if (lane < 6) {
        s.cvel[lane] = T(0);
        s.cacc[lane] = lane < 3 ? T(0) : T(-m.gravity[lane - 3]);
    }
    __syncwarp();
    for (int L = 1; L < m.nlevel; ++L) {
        for (int idx = m.level_ptr[L] + lane; idx < m.level_ptr[L + 1]; idx += 32) {
            int b = m.level_body[idx];
            int par = m.body_parentid[b];
            T v[6], a[6];
            for (int k = 0; k < 6; ++k) { v[k] = s.cvel[6 * par + k]; a[k] = s.cacc[6 * par + k]; }
            int j0 = m.body_jntadr[b], jn = m.body_jntnum[b];
            for (int j = j0; j < j0 + jn; ++j) {
                int da = m.jnt_dofadr[j];
                if (m.jnt_type[j] == kJntFree) {
                    for (int i = 0; i < 3; ++i)
                        for (int k = 0; k < 6; ++k) v[k] += s.cdof[6 * (da + i) + k] * s.qvel[da + i];
                    for (int i = 0; i < 3; ++i) {
                        s.cdofd[6 * (da + i)] = s.cdofd[6 * (da + i) + 1] = s.cdofd[6 * (da + i) + 2] = T(0);
                        s.cdofd[6 * (da + i) + 3] = s.cdofd[6 * (da + i) + 4] = s.cdofd[6 * (da + i) + 5] = T(0);
                        cross_motion(v, s.cdof + 6 * (da + 3 + i), s.cdofd + 6 * (da + 3 + i));
                    }
                    for (int i = 3; i < 6; ++i)
                        for (int k = 0; k < 6; ++k) v[k] += s.cdof[6 * (da + i) + k] * s.qvel[da + i];
                } else {
                    cross_motion(v, s.cdof + 6 * da, s.cdofd + 6 * da);
                    for (int k = 0; k < 6; ++k) v[k] += s.cdof[6 * da + k] * s.qvel[da];
                }
            }
            int d0 = m.body_dofadr[b], dn = m.body_dofnum[b];
            for (int d = d0; d < d0 + dn; ++d)
                for (int k = 0; k < 6; ++k) a[k] += s.cdofd[6 * d + k] * s.qvel[d];
            for (int k = 0; k < 6; ++k) { s.cvel[6 * b + k] = v[k]; s.cacc[6 * b + k] = a[k]; }
        }
        __syncwarp();
    }
    // body forces (overwrite cacc with cfrc)
    for (int b = 1 + lane; b < m.nbody; b += 32) {
        T f1[6], iv[6], f2[6];
        const T* ci = s.cinert + 10 * b;
        inert_mul(ci, s.cacc + 6 * b, f1);
        inert_mul(ci, s.cvel + 6 * b, iv);
        cross_force(s.cvel + 6 * b, iv, f2);
        for (int k = 0; k < 6; ++k) s.cacc[6 * b + k] = f1[k] + f2[k];
    }
    __syncwarp();
    // backward accumulation (children in descending index, like the oracle's reverse sweep)
    for (int L = m.nlevel - 1; L >= 1; --L) {
        int n0 = m.level_ptr[L], nl = m.level_ptr[L + 1] - n0;
        for (int t = lane; t < nl * 6; t += 32) {
            int b = m.level_body[n0 + t / 6], c = t % 6;
            T acc = s.cacc[6 * b + c];
            for (int k = m.child_ptr[b]; k < m.child_ptr[b + 1]; ++k) acc += s.cacc[6 * m.child_idx[k] + c];
            s.cacc[6 * b + c] = acc;
        }
        __syncwarp();
    }
    for (int i = lane; i < m.nv; i += 32) s.bias[i] = dot6(s.cdof + 6 * i, s.cacc + 6 * m.dof_bodyid[i]);
    __syncwarp();
}

// actuation + passive + smooth force (oracle actuation / forward)
template <class T> __device__ void __noinline__ smooth_force(const s3_model& m_, const s3_layout& L_, T* B_, const T* applied, int lane) {
    const s3_model& m = c_s3m;  // constant-bank model (both dtypes; see c_s3m)
    WS<T> s = make_ws(B_, L_);
    for (int i = lane; i < m.nv; i += 32) { s.fcon[i] = T(0); s.kvd[i] = T(0); }
    __syncwarp();
    const T* gain = F<T>(m.act_gain);
    for (int u = lane; u < m.nu; u += 32) {
        int d = m.act_dofadr[u], a = m.act_qposadr[u], kind = m.act_kind[u];
        T kp = gain[5 * u], kv = gain[5 * u + 1], eff = gain[5 * u + 2];
        T q = s.qpos[a], qd = s.qvel[d];
        T tau = kp * (s.ctrl[u] - q) + kv * (T(0) - qd);
        if (kind == kActDC) {
            T sat = gain[5 * u + 3], vmax = gain[5 * u + 4];
            T hi = fmin(fmax(sat * (T(1) - qd / vmax), T(0)), eff);
            T lo = fmin(fmax(sat * (T(-1) - qd / vmax), -eff), T(0));
            tau = fmin(fmax(tau, lo), hi);
        } else {
            bool clamped = tau > eff || tau < -eff;
            tau = fmin(fmax(tau, -eff), eff);
            if (kind == kActImplicit && !clamped) s.kvd[d] += kv;
        }
        s.fcon[d] += tau;  // fcon doubles as qfrc_actuator scratch here
    }
    __syncwarp();
    const T* damp = F<T>(m.dof_damping);
    for (int i = lane; i < m.nv; i += 32) {
        T f = s.fcon[i] - damp[i] * s.qvel[i] - s.bias[i];
        if (applied) f += applied[i];
        s.smooth[i] = f;
    }
    __syncwarp();
}

// ---------------------------------------------------------------- collision

template <class T> struct Hit { T d, n[3], pos[3]; };

template <class T> __device__ bool hfield_point(const s3_model& m, const T* q, T r, T& d, T* n) {
    const T* H = F<T>(m.hfield);
    T sp = T(m.hf_spacing);
    T fx = (q[0] - T(m.hf_origin[0])) / sp;
    T fy = (q[1] - T(m.hf_origin[1])) / sp;
    if (!(fx >= T(0) && fy >= T(0) && fx < T(m.hf_ncol - 1) && fy < T(m.hf_nrow - 1))) return false;
    int ix = (int)floor(fx), iy = (int)floor(fy);
    T u = fx - T(ix), v = fy - T(iy);
    T x0 = T(m.hf_origin[0]) + T(ix) * sp;
    T y0 = T(m.hf_origin[1]) + T(iy) * sp;
    int nc = m.hf_ncol;
    T h00 = H[iy * nc + ix], h10 = H[iy * nc + ix + 1], h01 = H[(iy + 1) * nc + ix], h11 = H[(iy + 1) * nc + ix + 1];
    if (u >= v) {
        n[0] = -(h10 - h00) * sp; n[1] = -(h11 - h10) * sp;
    } else {
        n[0] = -(h11 - h01) * sp; n[1] = -(h01 - h00) * sp;
    }
    n[2] = sp * sp;
    T rn = rsqrt_t(n[0] * n[0] + n[1] * n[1] + n[2] * n[2]);
    n[0] *= rn; n[1] *= rn; n[2] *= rn;
    T dq[3] = {q[0] - x0, q[1] - y0, q[2] - h00};
    d = dot3(n, dq) - r;
    return true;
}

template <class T> __device__ void seg_closest(const T* p1, const T* q1, const T* p2, const T* q2, T* A, T* B) {
    T d1[3] = {q1[0] - p1[0], q1[1] - p1[1], q1[2] - p1[2]};
    T d2[3] = {q2[0] - p2[0], q2[1] - p2[1], q2[2] - p2[2]};
    T r[3] = {p1[0] - p2[0], p1[1] - p2[1], p1[2] - p2[2]};
    T a = dot3(d1, d1), e = dot3(d2, d2), f = dot3(d2, r);
    T c = dot3(d1, r), b = dot3(d1, d2);
    T sN, tN;
    if (e <= T(1e-12)) {
        sN = a > T(1e-12) ? clampt(-c / a, T(0), T(1)) : T(0);
        tN = T(0);
    } else if (a <= T(1e-12)) {
        sN = T(0);
        tN = clampt(f / e, T(0), T(1));
    } else {
        T den = a * e - b * b;
        sN = den > T(1e-12) ? clampt((b * f - c * e) / den, T(0), T(1)) : T(0);
        tN = (b * sN + f) / e;
        if (tN < T(0)) {
            tN = T(0);
            sN = clampt(-c / a, T(0), T(1));
        } else if (tN > T(1)) {
            tN = T(1);
            sN = clampt((b - c) / a, T(0), T(1));
        }
    }
    for (int k = 0; k < 3; ++k) { A[k] = p1[k] + d1[k] * sN; B[k] = p2[k] + d2[k] * tN; }
}

// world frame of geom g from its body's frame (oracle kinematics: xpos + xmat @ geom_pos, xmat @ lmat);
// computed where needed instead of stored per world (saves 12 ngeom shared-memory elements)
template <class T> __device__ inline void geom_xform(const s3_model& m, const WS<T>& s, int g, T* c, T* R) {
    const int b = m.geom_bodyid[g];
    T Rb[9], v[3], L[9];
    qmat(s.xquat + 4 * b, Rb);
    const T* gp = F<T>(m.geom_pos) + 3 * g;
    const T* gl = F<T>(m.geom_lmat) + 9 * g;
    T pl[3] = {gp[0], gp[1], gp[2]};
    mv3(Rb, pl, v);
    c[0] = s.xpos[3 * b] + v[0]; c[1] = s.xpos[3 * b + 1] + v[1]; c[2] = s.xpos[3 * b + 2] + v[2];
    for (int k = 0; k < 9; ++k) L[k] = gl[k];
    mm3(Rb, L, R);
}

template <class T> __device__ inline void segment(const s3_model& m, int g, const T* c, const T* R, T* p, T* q) {
    T hl = F<T>(m.geom_size)[3 * g + 1];
    for (int k = 0; k < 3; ++k) {
        T a = R[3 * k + 2] * hl;
        p[k] = c[k] - a;
        q[k] = c[k] + a;
    }
}

// point k (0..7) of geom g's terrain point set (sphere: centre; capsule: 2 ends; box: 8 corners)
template <class T> __device__ inline int point_count(int type) {
    return type == kGeomSphere ? 1 : (type == kGeomCapsule ? 2 : 8);
}

template <class T> __device__ inline void point_of(const s3_model& m, int g, const T* c, const T* R, int type, int k,
                                                   T* q, T& r) {
    const T* sz = F<T>(m.geom_size) + 3 * g;
    if (type == kGeomSphere) {
        q[0] = c[0]; q[1] = c[1]; q[2] = c[2];
        r = sz[0];
    } else if (type == kGeomCapsule) {
        T p0[3], p1[3];
        segment(m, g, c, R, p0, p1);
        const T* pp = k == 0 ? p0 : p1;
        q[0] = pp[0]; q[1] = pp[1]; q[2] = pp[2];
        r = sz[0];
    } else {
        T loc[3] = {(k & 1) ? sz[0] : -sz[0], (k & 2) ? sz[1] : -sz[1], (k & 4) ? sz[2] : -sz[2]};
        T v[3];
        mv3(R, loc, v);
        q[0] = c[0] + v[0]; q[1] = c[1] + v[1]; q[2] = c[2] + v[2];
        r = T(0);
    }
}

// Box-box (oracle box_box): separating axes (3 + 3 face normals, 9 edge-edge cross products, parallel pairs
// skipped); a face axis clips the other box's incident face against the reference face's side planes and
// keeps the points below the reference face (at most 4: the deepest, then farthest-point selection); an edge
// axis gives one contact between the two support edges. Normal from box 1 to box 2.
constexpr double kBoxFaceBias = 0.95;  // an edge axis wins only below this fraction of the best face overlap
constexpr double kBoxTie = 1e-12;  // replace the current axis / face / point only when better by this margin

template <class T>
__device__ __noinline__ int box_box(const T* c1, const T* R1, const T* h1, const T* c2, const T* R2, const T* h2,
                                    Hit<T>* hits) {
    T dv[3] = {c2[0] - c1[0], c2[1] - c1[1], c2[2] - c1[2]};
    T A[3][3], B[3][3];
    for (int i = 0; i < 3; ++i)
        for (int k = 0; k < 3; ++k) { A[i][k] = R1[3 * k + i]; B[i][k] = R2[3 * k + i]; }
    auto overlap = [&](const T* u, T& sd) {
        T r1 = h1[0] * fabs(dot3(u, A[0])) + h1[1] * fabs(dot3(u, A[1])) + h1[2] * fabs(dot3(u, A[2]));
        T r2 = h2[0] * fabs(dot3(u, B[0])) + h2[1] * fabs(dot3(u, B[1])) + h2[2] * fabs(dot3(u, B[2]));
        sd = dot3(u, dv);
        return r1 + r2 - fabs(sd);
    };
    T fov = T(0), fsd = T(0), fu[3] = {T(0), T(0), T(0)};
    int fk = -1;
    for (int k = 0; k < 6; ++k) {
        const T* u = k < 3 ? A[k] : B[k - 3];
        T sd, ov = overlap(u, sd);
        if (ov < T(0)) return 0;
        if (fk < 0 || ov < fov - T(kBoxTie)) { fov = ov; fk = k; fsd = sd; fu[0] = u[0]; fu[1] = u[1]; fu[2] = u[2]; }
    }
    T eov = T(0), esd = T(0), eu[3] = {T(0), T(0), T(0)};
    int ek = -1;
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) {
            T u[3];
            cross3(A[i], B[j], u);
            T L = sqrt(dot3(u, u));
            if (L < T(1e-6)) continue;
            u[0] = u[0] / L; u[1] = u[1] / L; u[2] = u[2] / L;
            T sd, ov = overlap(u, sd);
            if (ov < T(0)) return 0;
            if (ek < 0 || ov < eov - T(kBoxTie)) { eov = ov; ek = 6 + 3 * i + j; esd = sd; eu[0] = u[0]; eu[1] = u[1]; eu[2] = u[2]; }
        }
    const bool use_edge = ek >= 0 && eov < T(kBoxFaceBias) * fov;
    const T ov = use_edge ? eov : fov, sd = use_edge ? esd : fsd;
    const int kk = use_edge ? ek : fk;
    const T* u = use_edge ? eu : fu;
    T n[3];
    for (int k = 0; k < 3; ++k) n[k] = sd >= T(0) ? u[k] : -u[k];
    if (kk >= 6) {
        const int i = (kk - 6) / 3, j = (kk - 6) % 3;
        T e1[3] = {c1[0], c1[1], c1[2]}, e2[3] = {c2[0], c2[1], c2[2]};
        for (int q = 0; q < 3; ++q) {
            if (q != i) {
                const T sg = dot3(A[q], n) >= T(0) ? T(1) : T(-1);
                for (int k = 0; k < 3; ++k) e1[k] = e1[k] + (sg * h1[q]) * A[q][k];
            }
            if (q != j) {
                const T sg = dot3(B[q], n) <= T(0) ? T(1) : T(-1);
                for (int k = 0; k < 3; ++k) e2[k] = e2[k] + (sg * h2[q]) * B[q][k];
            }
        }
        T p1[3], q1[3], p2[3], q2[3], P[3], Q[3];
        for (int k = 0; k < 3; ++k) {
            p1[k] = e1[k] - A[i][k] * h1[i]; q1[k] = e1[k] + A[i][k] * h1[i];
            p2[k] = e2[k] - B[j][k] * h2[j]; q2[k] = e2[k] + B[j][k] * h2[j];
        }
        seg_closest(p1, q1, p2, q2, P, Q);
        hits[0].d = -ov;
        for (int k = 0; k < 3; ++k) { hits[0].n[k] = n[k]; hits[0].pos[k] = T(0.5) * (P[k] + Q[k]); }
        return 1;
    }
    // face axis: reference box (its face along the axis) and incident box
    const bool r1 = kk < 3;
    const T* cr = r1 ? c1 : c2;
    const T* ci = r1 ? c2 : c1;
    const T* hr = r1 ? h1 : h2;
    const T* hi = r1 ? h2 : h1;
    const T(*Ar)[3] = r1 ? A : B;
    const T(*Ai)[3] = r1 ? B : A;
    const int ia = r1 ? kk : kk - 3;
    T nref[3];
    for (int k = 0; k < 3; ++k) nref[k] = r1 ? n[k] : -n[k];
    T cf[3];
    for (int k = 0; k < 3; ++k) cf[k] = cr[k] + nref[k] * hr[ia];
    int jf = 0;
    T pj = fabs(dot3(Ai[0], nref));
    for (int q = 1; q < 3; ++q) {
        const T pq = fabs(dot3(Ai[q], nref));
        if (pq > pj + T(kBoxTie)) { pj = pq; jf = q; }
    }
    const T sgi = dot3(Ai[jf], nref) >= T(0) ? T(-1) : T(1);
    T fi[3];
    for (int k = 0; k < 3; ++k) fi[k] = ci[k] + (sgi * Ai[jf][k]) * hi[jf];
    const int ua = jf == 0 ? 1 : 0, va = jf == 2 ? 1 : 2;
    T poly[8][3], tmp[8][3];
    int np = 4;
    const T su[4] = {T(-1), T(1), T(1), T(-1)}, sv[4] = {T(-1), T(-1), T(1), T(1)};
    for (int v = 0; v < 4; ++v)
        for (int k = 0; k < 3; ++k) poly[v][k] = fi[k] + (su[v] * hi[ua]) * Ai[ua][k] + (sv[v] * hi[va]) * Ai[va][k];
    for (int t = 0; t < 3; ++t) {
        if (t == ia) continue;
        for (int sgn = 0; sgn < 2; ++sgn) {
            const T sg = sgn == 0 ? T(1) : T(-1);
            int no = 0;
            for (int idx = 0; idx < np; ++idx) {
                const T* P = poly[idx];
                const T* Q = poly[idx + 1 < np ? idx + 1 : 0];
                T dpv[3] = {P[0] - cr[0], P[1] - cr[1], P[2] - cr[2]}, dqv[3] = {Q[0] - cr[0], Q[1] - cr[1], Q[2] - cr[2]};
                const T dP = hr[t] - sg * dot3(dpv, Ar[t]);
                const T dQ = hr[t] - sg * dot3(dqv, Ar[t]);
                if (dP >= T(0) && no < 8) { tmp[no][0] = P[0]; tmp[no][1] = P[1]; tmp[no][2] = P[2]; ++no; }
                if ((dP >= T(0)) != (dQ >= T(0)) && no < 8) {
                    const T f = dP / (dP - dQ);
                    for (int k = 0; k < 3; ++k) tmp[no][k] = P[k] + (Q[k] - P[k]) * f;
                    ++no;
                }
            }
            np = no;
            for (int v = 0; v < np; ++v)
                for (int k = 0; k < 3; ++k) poly[v][k] = tmp[v][k];
            if (np == 0) return 0;
        }
    }
    T dep[8];
    int nk = 0;
    for (int v = 0; v < np; ++v) {
        T dc[3] = {cf[0] - poly[v][0], cf[1] - poly[v][1], cf[2] - poly[v][2]};
        const T dd = dot3(nref, dc);
        if (dd > T(0)) {
            dep[nk] = dd;
            for (int k = 0; k < 3; ++k) tmp[nk][k] = poly[v][k];
            ++nk;
        }
    }
    if (nk == 0) return 0;
    int chosen[4], nc = 0;
    int b = 0;
    for (int q = 1; q < nk; ++q)
        if (dep[q] > dep[b] + T(kBoxTie)) b = q;
    chosen[nc++] = b;
    const int want = nk < 4 ? nk : 4;
    while (nc < want) {
        int bq = -1;
        T bd = T(-1);
        for (int q = 0; q < nk; ++q) {
            bool used = false;
            for (int c = 0; c < nc; ++c) used = used || chosen[c] == q;
            if (used) continue;
            T dm = T(0);
            for (int c = 0; c < nc; ++c) {
                T e[3] = {tmp[q][0] - tmp[chosen[c]][0], tmp[q][1] - tmp[chosen[c]][1], tmp[q][2] - tmp[chosen[c]][2]};
                const T d2 = dot3(e, e);
                dm = c == 0 ? d2 : fmin(dm, d2);
            }
            if (dm > bd + T(kBoxTie)) { bq = q; bd = dm; }
        }
        chosen[nc++] = bq;
    }
    for (int c = 0; c < nc; ++c) {
        const int q = chosen[c];
        hits[c].d = -dep[q];
        for (int k = 0; k < 3; ++k) { hits[c].n[k] = n[k]; hits[c].pos[k] = tmp[q][k] + nref[k] * (T(0.5) * dep[q]); }
    }
    return nc;
}

// Narrowphase of one pair: up to 4 contacts into `hits`, in the oracle's order.
template <class T> __device__ __noinline__ int narrow(const s3_model& m_, const s3_layout& L_, T* B_, int p, Hit<T>* hits) {
    const s3_model& m = c_s3m;  // constant-bank model (both dtypes; see c_s3m)
    WS<T> s = make_ws(B_, L_);
    int g1 = m.pair_geom[2 * p], g2 = m.pair_geom[2 * p + 1];
    int t1 = m.geom_type[g1], t2 = m.geom_type[g2];
    T c1[3], R1[9], c2[3], R2[9];
    geom_xform(m, s, g1, c1, R1);
    geom_xform(m, s, g2, c2, R2);
    const T* rb = F<T>(m.geom_rbound);
    int cnt = 0, cap = t2 == kGeomBox ? 4 : 8;
    if (t1 == kGeomPlane) {
        T n[3] = {R1[2], R1[5], R1[8]};
        T dc[3] = {c2[0] - c1[0], c2[1] - c1[1], c2[2] - c1[2]};
        if (!(dot3(n, dc) - rb[g2] < T(0))) return 0;
        int np = point_count<T>(t2);
        for (int k = 0; k < np && cnt < cap; ++k) {
            T q[3], r;
            point_of(m, g2, c2, R2, t2, k, q, r);
            T dq[3] = {q[0] - c1[0], q[1] - c1[1], q[2] - c1[2]};
            T d = dot3(n, dq) - r;
            if (d < T(0)) {
                Hit<T> h;
                h.d = d;
                for (int i = 0; i < 3; ++i) { h.n[i] = n[i]; h.pos[i] = q[i] - n[i] * (r + T(0.5) * d); }
                hits[cnt] = h;
                ++cnt;
            }
        }
    } else if (t1 == kGeomHfield) {
        if (!(c2[2] - rb[g2] < T(m.hf_max))) return 0;
        int np = point_count<T>(t2);
        for (int k = 0; k < np && cnt < cap; ++k) {
            T q[3], r, d, n[3];
            point_of(m, g2, c2, R2, t2, k, q, r);
            if (hfield_point(m, q, r, d, n) && d < T(0)) {
                Hit<T> h;
                h.d = d;
                for (int i = 0; i < 3; ++i) { h.n[i] = n[i]; h.pos[i] = q[i] - n[i] * (r + T(0.5) * d); }
                hits[cnt] = h;
                ++cnt;
            }
        }
    } else if (t1 == kGeomBox) {  // box-box: oracle box_box
        T dv[3] = {c2[0] - c1[0], c2[1] - c1[1], c2[2] - c1[2]};
        T rr = rb[g1] + rb[g2];
        if (!(dot3(dv, dv) < rr * rr)) return 0;
        const T* sz = F<T>(m.geom_size);
        T h1[3] = {sz[3 * g1], sz[3 * g1 + 1], sz[3 * g1 + 2]}, h2[3] = {sz[3 * g2], sz[3 * g2 + 1], sz[3 * g2 + 2]};
        cnt = box_box(c1, R1, h1, c2, R2, h2, hits);
    } else if (t2 == kGeomBox) {  // sphere or capsule (g1) vs box (g2): oracle sphere_box / capsule_box
        T dv[3] = {c2[0] - c1[0], c2[1] - c1[1], c2[2] - c1[2]};
        T rr = rb[g1] + rb[g2];
        if (!(dot3(dv, dv) < rr * rr)) return 0;
        const T* sz = F<T>(m.geom_size);
        const T* R = R2;
        const T* hs = sz + 3 * g2;
        T r = sz[3 * g1];
        T p[3], q[3], dq[3];
        if (t1 == kGeomCapsule) {
            // segment point closest to the box: alternating projections from the midpoint (box frame)
            T e0[3], e1[3], a[3], b[3], dd3[3];
            segment(m, g1, c1, R1, e0, e1);
            for (int k = 0; k < 3; ++k) {
                a[k] = R[k] * (e0[0] - c2[0]) + R[3 + k] * (e0[1] - c2[1]) + R[6 + k] * (e0[2] - c2[2]);
                b[k] = R[k] * (e1[0] - c2[0]) + R[3 + k] * (e1[1] - c2[1]) + R[6 + k] * (e1[2] - c2[2]);
                dd3[k] = b[k] - a[k];
            }
            T dd = dot3(dd3, dd3), t = T(0.5);
            for (int it = 0; it < 8; ++it) {
                T qq[3];
                for (int k = 0; k < 3; ++k) qq[k] = fmin(fmax(a[k] + dd3[k] * t, -hs[k]), hs[k]) - a[k];
                t = dd > T(1e-12) ? clampt(dot3(qq, dd3) / dd, T(0), T(1)) : T(0);
            }
            T cl[3] = {a[0] + dd3[0] * t, a[1] + dd3[1] * t, a[2] + dd3[2] * t}, cw[3];
            mv3(R, cl, cw);
            T cc[3] = {c2[0] + cw[0], c2[1] + cw[1], c2[2] + cw[2]};
            T dl[3] = {cc[0] - c2[0], cc[1] - c2[1], cc[2] - c2[2]};
            for (int k = 0; k < 3; ++k) p[k] = R[k] * dl[0] + R[3 + k] * dl[1] + R[6 + k] * dl[2];
        } else {
            T dl[3] = {c1[0] - c2[0], c1[1] - c2[1], c1[2] - c2[2]};
            for (int k = 0; k < 3; ++k) p[k] = R[k] * dl[0] + R[3 + k] * dl[1] + R[6 + k] * dl[2];
        }
        for (int k = 0; k < 3; ++k) {
            q[k] = fmin(fmax(p[k], -hs[k]), hs[k]);
            dq[k] = p[k] - q[k];
        }
        T L = sqrt(dot3(dq, dq));
        T nl[3], fp[3], d;
        if (L > T(1e-12)) {
            for (int k = 0; k < 3; ++k) { nl[k] = -dq[k] / L; fp[k] = q[k]; }
            d = L - r;
        } else {
            int kk = 0;
            T best = hs[0] - fabs(p[0]);
            for (int k = 1; k < 3; ++k) {
                T gk = hs[k] - fabs(p[k]);
                if (gk < best) { best = gk; kk = k; }
            }
            for (int k = 0; k < 3; ++k) { nl[k] = T(0); fp[k] = p[k]; }
            nl[kk] = p[kk] >= T(0) ? T(-1) : T(1);
            fp[kk] = p[kk] >= T(0) ? hs[kk] : -hs[kk];
            d = -best - r;
        }
        if (d < T(0)) {
            Hit<T> h;
            h.d = d;
            T n[3], wp[3];
            mv3(R, nl, n);
            mv3(R, fp, wp);
            for (int k = 0; k < 3; ++k) { h.n[k] = n[k]; h.pos[k] = c2[k] + wp[k] - n[k] * (T(0.5) * d); }
            hits[cnt] = h;
            ++cnt;
        }
    } else {
        T dv[3] = {c2[0] - c1[0], c2[1] - c1[1], c2[2] - c1[2]};
        T rr = rb[g1] + rb[g2];
        if (!(dot3(dv, dv) < rr * rr)) return 0;
        const T* sz = F<T>(m.geom_size);
        T r1 = sz[3 * g1], r2 = sz[3 * g2];
        T A[3], B[3];
        if (t1 == kGeomSphere && t2 == kGeomSphere) {
            for (int k = 0; k < 3; ++k) { A[k] = c1[k]; B[k] = c2[k]; }
        } else if (t1 == kGeomSphere) {
            T p2[3], q2[3];
            segment(m, g2, c2, R2, p2, q2);
            seg_closest(p2, q2, c1, c1, B, A);
        } else if (t2 == kGeomSphere) {
            T p1[3], q1[3];
            segment(m, g1, c1, R1, p1, q1);
            seg_closest(p1, q1, c2, c2, A, B);
        } else {
            T p1[3], q1[3], p2[3], q2[3];
            segment(m, g1, c1, R1, p1, q1);
            segment(m, g2, c2, R2, p2, q2);
            seg_closest(p1, q1, p2, q2, A, B);
        }
        T e[3] = {B[0] - A[0], B[1] - A[1], B[2] - A[2]};
        T L = sqrt(dot3(e, e));
        T n[3];
        if (L > T(1e-12)) { n[0] = e[0] / L; n[1] = e[1] / L; n[2] = e[2] / L; }
        else { n[0] = T(0); n[1] = T(0); n[2] = T(1); }
        T d = L - r1 - r2;
        if (d < T(0)) {
            Hit<T> h;
            h.d = d;
            for (int i = 0; i < 3; ++i) { h.n[i] = n[i]; h.pos[i] = A[i] + n[i] * (r1 + T(0.5) * d); }
            hits[cnt] = h;
            ++cnt;
        }
    }
    return cnt;
}

template <class T> __device__ inline void make_frame(const T* n, T* fr) {
    T e[3];
    if (fabs(n[1]) < T(0.5)) { e[0] = T(0); e[1] = T(1); e[2] = T(0); }
    else { e[0] = T(1); e[1] = T(0); e[2] = T(0); }
    T t1[3], t2[3];
    cross3(n, e, t1);
    T r = rsqrt_t(dot3(t1, t1));
    t1[0] *= r; t1[1] *= r; t1[2] *= r;
    cross3(n, t1, t2);
    for (int k = 0; k < 3; ++k) { fr[k] = n[k]; fr[3 + k] = t1[k]; fr[6 + k] = t2[k]; }
}

// broadphase + narrowphase over all pairs, compacted in pair order; returns ncon (warp-uniform)
template <class T> __device__ int __noinline__ collide(const s3_model& m_, const s3_layout& L_, T* B_, int lane, int& dropped, T fscale) {
    const s3_model& m = c_s3m;  // constant-bank model (both dtypes; see c_s3m)
    WS<T> s = make_ws(B_, L_);
    int base = 0;
    dropped = 0;
    const T* fric = F<T>(m.geom_friction);
    for (int p0 = 0; p0 < m.npair; p0 += 32) {
        int p = p0 + lane;
        Hit<T> hits[4];
        int cnt = p < m.npair ? narrow(m, L_, B_, p, hits) : 0;
        int incl = cnt;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            int y = __shfl_up_sync(FULL, incl, o);
            if (lane >= o) incl += y;
        }
        int total = __shfl_sync(FULL, incl, 31);
        int off = base + incl - cnt;
        if (cnt) {
            int g1 = m.pair_geom[2 * p], g2 = m.pair_geom[2 * p + 1];
            T mu = m.pair_condim[p] == 1 ? T(0) : fmax(fric[g1], fric[g2]) * fscale;  // condim 1: frictionless
            for (int k = 0; k < cnt; ++k) {
                int slot = off + k;
                if (slot < m.ncon_max) {
                    const Hit<T>& h = hits[k];
                    T* c = s.con + kConStride * slot;
                    c[0] = h.d;
                    c[1] = h.pos[0]; c[2] = h.pos[1]; c[3] = h.pos[2];
                    make_frame(h.n, c + 4);
                    c[13] = mu;
                    s.con_pair[slot] = p;
                }
            }
        }
        base += total;
    }
    __syncwarp();
    if (base > m.ncon_max) {
        dropped = base - m.ncon_max;
        base = m.ncon_max;
    }
    return base;
}

// ---------------------------------------------------------------- constraints

// U = union of the Jacobian column sets of every contact and every violated limit (warp-uniform)
template <class T> __device__ __noinline__ uint64_t touched_mask(const s3_model& m_, const s3_layout& L_, T* B_, int ncon,
                                                                 int lane) {
    const s3_model& m = c_s3m;  // constant-bank model (both dtypes; see c_s3m)
    WS<T> s = make_ws(B_, L_);
    const unsigned long long* pm = reinterpret_cast<const unsigned long long*>(m.pair_dofmask);
    const unsigned long long* cm = reinterpret_cast<const unsigned long long*>(m.dof_chainmask);
    uint64_t u = 0;
    for (int c = lane; c < ncon; c += 32) u |= __ldg(pm + s.con_pair[c]);
    const T* rng = F<T>(m.lim_range);
    for (int l = lane; l < m.nlimjnt; l += 32) {
        T q = s.qpos[m.lim_qposadr[l]];
        if (q - rng[2 * l] < T(0) || rng[2 * l + 1] - q < T(0)) u |= __ldg(cm + m.lim_dofadr[l]);
    }
    unsigned lo = __reduce_or_sync(FULL, (unsigned)(u & 0xffffffffu));
    unsigned hi = __reduce_or_sync(FULL, (unsigned)(u >> 32));
    return ((uint64_t)hi << 32) | lo;
}

template <class T> __device__ inline T impedance(const s3_model& m, T r) {
    T dmin = T(m.solimp[0]), dmax = T(m.solimp[1]), width = T(m.solimp[2]), mid = T(m.solimp[3]),
      power = T(m.solimp[4]);
    T x = fabs(r) / width;
    T d;
    if (x >= T(1)) d = dmax;
    else {
        T y = x <= mid ? pow(x, power) / pow(mid, power - T(1))
                       : T(1) - pow(T(1) - x, power) / pow(T(1) - mid, power - T(1));
        d = dmin + y * (dmax - dmin);
    }
    return fmin(fmax(d, T(1e-4)), T(0.9999));
}

// Contact Jacobians Jc[c][3][stride] (frame rows over the pair's chain), limit rows, aref, D.
template <class T> __device__ int __noinline__ build_rows(const s3_model& m_, const s3_layout& L_, T* B_, int ncon, int& nlim, int lane) {
    const s3_model& m = c_s3m;  // constant-bank model (both dtypes; see c_s3m)
    WS<T> s = make_ws(B_, L_);
    // limits: ballot-compact the violated sides
    const T* rng = F<T>(m.lim_range);
    nlim = 0;
    for (int l0 = 0; l0 < m.nlimjnt; l0 += 32) {
        int l = l0 + lane;
        T dlo = T(1), dhi = T(1);
        if (l < m.nlimjnt) {
            T q = s.qpos[m.lim_qposadr[l]];
            dlo = q - rng[2 * l];
            dhi = rng[2 * l + 1] - q;
        }
        bool lo = dlo < T(0), hi = dhi < T(0);
        // oracle order per joint: lower then upper (at most one is violated)
        unsigned mk = __ballot_sync(FULL, lo || hi);
        int rank = __popc(mk & ((1u << lane) - 1));
        int slot = nlim + rank;
        if ((lo || hi) && slot < S3_MAX_LIM) {
            s.lim_dof[slot] = m.lim_dofadr[l];
            s.lim_sign[slot] = lo ? 1 : -1;
            s.rjar[slot] = lo ? dlo : dhi;  // pos, stashed until aref below
        }
        nlim += __popc(mk);
    }
    if (nlim > S3_MAX_LIM) nlim = S3_MAX_LIM;
    __syncwarp();
    // contact Jacobians: serial over contacts, lanes over chain columns
    const T* iw = F<T>(m.body_invweight0);
    int stride = m.chain_stride;
    for (int t = lane; t < ncon * S3_MAX_CHAIN; t += 32) {
        int c = t / S3_MAX_CHAIN, k = t % S3_MAX_CHAIN;
        int p = s.con_pair[c];
        int len = m.pair_chainlen[p];
        if (k >= len) continue;
        int b1 = m.geom_bodyid[m.pair_geom[2 * p]], b2 = m.geom_bodyid[m.pair_geom[2 * p + 1]];
        uint64_t m1 = m.body_dofmask[b1], m2 = m.body_dofmask[b2];
        const T* cc = s.con + kConStride * c;
        {
            int d = m.pair_chain[p * S3_MAX_CHAIN + k];
            const T* com = s.com + 3 * m.body_treeid[m.dof_bodyid[d]];
            T dp[3] = {cc[1] - com[0], cc[2] - com[1], cc[3] - com[2]};
            const T* cd = s.cdof + 6 * d;
            T w[3];
            cross3(cd, dp, w);
            T jv[3] = {cd[3] + w[0], cd[4] + w[1], cd[5] + w[2]};
            T sg = T(((m2 >> d) & 1ull) ? 1 : 0) - T(((m1 >> d) & 1ull) ? 1 : 0);
            T* J = s.Jc + (3 * c) * stride;
            J[k] = sg * dot3(cc + 4, jv);
            J[stride + k] = sg * dot3(cc + 7, jv);
            J[2 * stride + k] = sg * dot3(cc + 10, jv);
        }
    }
    __syncwarp();
    int nefc = nlim + 4 * ncon;
    // J qvel per row (contact frame dots first)
    for (int t = lane; t < 3 * ncon; t += 32) {
        int c = t / 3, r = t % 3;
        int p = s.con_pair[c];
        int len = m.pair_chainlen[p];
        const T* J = s.Jc + (3 * c + r) * stride;
        T acc = T(0);
        for (int k = 0; k < len; ++k) acc += J[k] * s.qvel[m.pair_chain[p * S3_MAX_CHAIN + k]];
        s.cdot[t] = acc;
    }
    __syncwarp();
    T tc = fmax(T(m.solref[0]), T(2) * T(m.timestep));
    T dr = T(m.solref[1]);
    T dmax = T(m.solimp[1]);
    T kk = T(1) / (dmax * dmax * tc * tc * dr * dr);
    T bb = T(2) / (dmax * tc);
    const T* diw = F<T>(m.dof_invweight0);
    for (int r = lane; r < nefc; r += 32) {
        T pos, vel, A;
        if (r < nlim) {
            int d = s.lim_dof[r];
            pos = s.rjar[r];
            vel = T(s.lim_sign[r]) * s.qvel[d];
            A = diw[d];
        } else {
            int c = (r - nlim) >> 2, e = (r - nlim) & 3;
            const T* cc = s.con + kConStride * c;
            T mu = cc[13];
            T sg = (e & 1) ? -mu : mu;
            pos = cc[0];
            vel = s.cdot[3 * c] + sg * s.cdot[3 * c + 1 + (e >> 1)];
            int p = s.con_pair[c];
            int b1 = m.geom_bodyid[m.pair_geom[2 * p]], b2 = m.geom_bodyid[m.pair_geom[2 * p + 1]];
            // condim 1: mu = 0 makes the 4 pyramid rows the normal row; at 4x its R each they sum to MuJoCo's
            // single frictionless row (same cost, Hessian and total force)
            A = (m.pair_condim[p] == 1 ? T(4) : T(1) + mu * mu) * (iw[b1] + iw[b2]);
        }
        T imp = impedance(m, pos);
        T R = fmax((T(1) - imp) / imp * A, T(1e-15));
        s.rD[r] = T(1) / R;
        s.raref[r] = -bb * vel - kk * imp * pos;
    }
    __syncwarp();
    return nefc;
}

// out[r] = J_r x for all rows
template <class T> __device__ void __noinline__ rows_mul(const s3_model& m_, const s3_layout& L_, T* B_, int ncon, int nlim, const T* x, T* out,
                                            int lane) {
    const s3_model& m = model_ref<T>(m_);  // float64: the constant-bank copy (see c_s3m)
    WS<T> s = make_ws(B_, L_);
    int stride = m.chain_stride;
    for (int t = lane; t < 3 * ncon; t += 32) {
        int c = t / 3, r = t % 3;
        int p = s.con_pair[c];
        int len = m.pair_chainlen[p];
        const T* J = s.Jc + (3 * c + r) * stride;
        T acc = T(0);
        for (int k = 0; k < len; ++k) acc += J[k] * x[m.pair_chain[p * S3_MAX_CHAIN + k]];
        s.cdot[t] = acc;
    }
    __syncwarp();
    int nefc = nlim + 4 * ncon;
    for (int r = lane; r < nefc; r += 32) {
        T v;
        if (r < nlim) v = T(s.lim_sign[r]) * x[s.lim_dof[r]];
        else {
            int c = (r - nlim) >> 2, e = (r - nlim) & 3;
            T mu = s.con[kConStride * c + 13];
            T sg = (e & 1) ? -mu : mu;
            v = s.cdot[3 * c] + sg * s.cdot[3 * c + 1 + (e >> 1)];
        }
        out[r] = v;
    }
    __syncwarp();
}

// y += J^T (coef) where coef[r] is per row
template <class T> __device__ void __noinline__ rows_tmul_add(const s3_model& m_, const s3_layout& L_, T* B_, int ncon, int nlim, const T* coef, T* y,
                                                 int lane) {
    const s3_model& m = model_ref<T>(m_);  // float64: the constant-bank copy (see c_s3m)
    WS<T> s = make_ws(B_, L_);
    int stride = m.chain_stride;
    for (int r = lane; r < nlim; r += 32) y[s.lim_dof[r]] += T(s.lim_sign[r]) * coef[r];
    __syncwarp();
    for (int c0 = 0; c0 < ncon;) {
        int p0 = s.con_pair[c0];
        int cls = m.pair_class[p0];
        int c1e = c0 + 1;
        while (c1e < ncon && m.pair_class[s.con_pair[c1e]] == cls) ++c1e;
        int len = m.pair_chainlen[p0];
        for (int k = lane; k < len; k += 32) {
            T acc = T(0);
            for (int c = c0; c < c1e; ++c) {
                const T* w = coef + nlim + 4 * c;
                T mu = s.con[kConStride * c + 13];
                T cn = ((w[0] + w[1]) + w[2]) + w[3];
                T ca = mu * (w[0] - w[1]);
                T cb = mu * (w[2] - w[3]);
                const T* J = s.Jc + (3 * c) * stride;
                acc += cn * J[k] + ca * J[stride + k] + cb * J[2 * stride + k];
            }
            y[m.pair_chain[p0 * S3_MAX_CHAIN + k]] += acc;
        }
        __syncwarp();
        c0 = c1e;
    }
}

template <class T> __device__ T __noinline__ total_cost(const s3_model& m_, const s3_layout& L_, T* B_, int nefc, const T* a, const T* Ma,
                                           const T* jar, int lane) {
    const s3_model& m = model_ref<T>(m_);  // float64: the constant-bank copy (see c_s3m)
    WS<T> s = make_ws(B_, L_);
    // 1/2 a^T M a - a^T f + constraint term: the Gauss term up to a constant (oracle _cost)
    T g = T(0);
    for (int i = lane; i < m.nv; i += 32) g += a[i] * (Ma[i] - T(2) * s.smooth[i]);
    T c = T(0);
    for (int r = lane; r < nefc; r += 32)
        if (jar[r] < T(0)) c += s.rD[r] * jar[r] * jar[r];
    return T(0.5) * wsum(g) + T(0.5) * wsum(c);
}

// mj_solNewton restated (oracle newton / line_search)
template <class T> __device__ int __noinline__ newton(const s3_model& m_, const s3_layout& L_, T* B_, int ncon, int nlim, bool warm_ok, uint64_t U, int lane) {
    const s3_model& m = c_s3m;  // constant-bank model (both dtypes; see c_s3m)
    WS<T> s = make_ws(B_, L_);
    int nv = m.nv;
    int nefc = nlim + 4 * ncon;
    T scale = T(m.scale);
    T tol = T(m.tolerance);
    // start from the warm start (staged in s.p by the caller), zeros without one (oracle newton)
    for (int i = lane; i < nv; i += 32) s.a[i] = warm_ok ? s.p[i] : T(0);
    __syncwarp();
    sym_mul(nv, s.M, s.a, s.Ma, lane);
    rows_mul(m, L_, B_, ncon, nlim, s.a, s.rjar, lane);
    for (int r = lane; r < nefc; r += 32) s.rjar[r] -= s.raref[r];
    __syncwarp();
    T cost = total_cost(m, L_, B_, nefc, s.a, s.Ma, s.rjar, lane);
    // H = M + J^T D J keeps the tree pattern unless a contact couples two branches
    bool tree = true;
    for (int c = 0; c < ncon; ++c) tree = tree && m.pair_tree[s.con_pair[c]] != 0;
    int its = 0;
    for (int it = 0; it < m.iterations; ++it) {
        // gradient
        for (int r = lane; r < nefc; r += 32) s.rJp[r] = s.rjar[r] < T(0) ? s.rD[r] * s.rjar[r] : T(0);
        for (int i = lane; i < nv; i += 32) s.grad[i] = s.Ma[i] - s.smooth[i];
        __syncwarp();
        rows_tmul_add(m, L_, B_, ncon, nlim, s.rJp, s.grad, lane);
        T gn = T(0), mag = T(0);
        for (int i = lane; i < nv; i += 32) {
            gn += s.grad[i] * s.grad[i];
            if (sizeof(T) == 4) mag += s.Ma[i] * s.Ma[i] + s.smooth[i] * s.smooth[i];
        }
        gn = wsum(gn);
        if (sizeof(T) == 4) mag = wsum(mag);
        T gfloor = sizeof(T) == 4 ? T(8) * T(1.1920929e-7) * scale * sqrt(mag) : T(0);
        if (scale * sqrt(gn) < tol + gfloor) break;
        ++its;
        // H = M + J^T diag(D act) J on the packed lower LD buffer: in tree mode only the rows of U are
        // rebuilt (from the snapshot of M partially eliminated by the untouched subtrees)
        if (tree) {
            tree_copy(m, s.LD, s.snap, U, false, lane);
        } else {
            int np = nv * (nv + 1) / 2;
            for (int t = lane; t < np; t += 32) s.LD[t] = s.M[t];
            __syncwarp();
        }
        for (int r = lane; r < nlim; r += 32)
            if (s.rjar[r] < T(0)) s.LD[tri(s.lim_dof[r], s.lim_dof[r])] += s.rD[r];
        __syncwarp();
        int stride = m.chain_stride;
        for (int c0 = 0; c0 < ncon;) {
            int p0 = s.con_pair[c0];
            int cls = m.pair_class[p0];
            int c1e = c0 + 1;
            while (c1e < ncon && m.pair_class[s.con_pair[c1e]] == cls) ++c1e;
            int len = m.pair_chainlen[p0];
            const uint8_t* ch = m.pair_chain + p0 * S3_MAX_CHAIN;
            int npair = len * (len + 1) / 2;
            for (int t = lane; t < npair; t += 32) {
                int ab = m.tri_tab[t];
                int a = ab >> 8, b = ab & 255;
                T v = T(0);
                for (int c = c0; c < c1e; ++c) {
                    const T* jr = s.rjar + nlim + 4 * c;
                    const T* D = s.rD + nlim + 4 * c;
                    T w0 = jr[0] < T(0) ? D[0] : T(0), w1 = jr[1] < T(0) ? D[1] : T(0);
                    T w2 = jr[2] < T(0) ? D[2] : T(0), w3 = jr[3] < T(0) ? D[3] : T(0);
                    T mu = s.con[kConStride * c + 13];
                    T W00 = ((w0 + w1) + w2) + w3, W01 = mu * (w0 - w1), W02 = mu * (w2 - w3);
                    T W11 = mu * mu * (w0 + w1), W22 = mu * mu * (w2 + w3);
                    const T* J0 = s.Jc + (3 * c) * stride;
                    const T* J1 = J0 + stride;
                    const T* J2 = J1 + stride;
                    T x0 = J0[a], x1 = J1[a], x2 = J2[a];
                    T y0 = J0[b], y1 = J1[b], y2 = J2[b];
                    v += x0 * (W00 * y0 + W01 * y1 + W02 * y2) + x1 * (W01 * y0 + W11 * y1) +
                         x2 * (W02 * y0 + W22 * y2);
                }
                s.LD[tri(ch[a], ch[b])] += v;
            }
            __syncwarp();
            c0 = c1e;
        }
        for (int i = lane; i < nv; i += 32) s.p[i] = -s.grad[i];
        __syncwarp();
        if (tree) {
            factor_ldl(m, s.LD, s.tk, lane, U, 2);
            solve_ldl(m, s.LD, s.p, lane);
        } else {
            cholesky(nv, s.LD, lane);
            chol_solve(nv, s.LD, s.p, lane);
        }
        sym_mul(nv, s.M, s.p, s.Mp, lane);
        rows_mul(m, L_, B_, ncon, nlim, s.p, s.rJp, lane);
        // exact line search along p: bracketed Newton on phi'
        T g0 = T(0), h0 = T(0);
        for (int i = lane; i < nv; i += 32) {
            g0 += s.p[i] * (s.Ma[i] - s.smooth[i]);
            h0 += s.p[i] * s.Mp[i];
        }
        g0 = wsum(g0);
        h0 = wsum(h0);
        auto deriv = [&](T al, T& d1, T& d2) {
            T x1 = T(0), x2 = T(0);
            for (int r = lane; r < nefc; r += 32) {
                T x = s.rjar[r] + al * s.rJp[r];
                if (x < T(0)) {
                    x1 += s.rD[r] * x * s.rJp[r];
                    x2 += s.rD[r] * s.rJp[r] * s.rJp[r];
                }
            }
            d1 = g0 + al * h0 + wsum(x1);
            d2 = h0 + wsum(x2);
        };
        T d0, dd;
        deriv(T(0), d0, dd);
        T alpha = T(0);
        if (d0 < T(0)) {
            T lo = T(0), hi = T(INFINITY), al = T(1);
            for (int li = 0; li < m.ls_iterations; ++li) {
                T d1, d2;
                deriv(al, d1, d2);
                if (fabs(d1) < T(m.ls_tolerance) * fabs(d0)) break;
                if (d1 < T(0)) lo = al;
                else hi = al;
                T an = al - d1 / d2;
                if (!(lo < an && an < hi)) an = T(0.5) * (lo + hi);
                al = an;
            }
            alpha = al;
        }
        if (alpha == T(0)) break;
        T impv, floor_ = T(0);
        if (sizeof(T) == 4) {
            // float32 build: the improvement from its own small terms -- Gauss part alpha g0 + alpha^2 h0 / 2
            // and the per-row change of the constraint cost -- instead of a difference of two large costs,
            // and the rounding floor of those terms (the float64 build keeps the oracle's cost difference)
            T dc = T(0), mg = T(0);
            for (int r = lane; r < nefc; r += 32) {
                T x0 = fmin(s.rjar[r], T(0)), x1 = fmin(s.rjar[r] + alpha * s.rJp[r], T(0));
                dc += s.rD[r] * (x1 * x1 - x0 * x0);
                mg += s.rD[r] * (x1 * x1 + x0 * x0);
            }
            dc = T(0.5) * wsum(dc);
            mg = T(0.5) * wsum(mg);
            T dg1 = alpha * g0, dg2 = T(0.5) * alpha * alpha * h0;
            impv = -scale * ((dg1 + dg2) + dc);
            floor_ = T(8) * T(1.1920929e-7) * scale * (fabs(dg1) + fabs(dg2) + mg);
        }
        for (int i = lane; i < nv; i += 32) {
            s.a[i] += alpha * s.p[i];
            s.Ma[i] += alpha * s.Mp[i];
        }
        for (int r = lane; r < nefc; r += 32) s.rjar[r] += alpha * s.rJp[r];
        __syncwarp();
        if (sizeof(T) != 4) {
            T nc = total_cost(m, L_, B_, nefc, s.a, s.Ma, s.rjar, lane);
            impv = scale * (cost - nc);
            cost = nc;
        }
        if (impv < tol + floor_) break;
    }
    // forces and qfrc_constraint
    for (int r = lane; r < nefc; r += 32) s.rJp[r] = s.rjar[r] < T(0) ? -s.rD[r] * s.rjar[r] : T(0);
    for (int i = lane; i < nv; i += 32) s.fcon[i] = T(0);
    __syncwarp();
    rows_tmul_add(m, L_, B_, ncon, nlim, s.rJp, s.fcon, lane);
    return its;
}

// Primal conjugate gradient on the Newton cost (oracle cg, mj_solCG restated; s3_model.flags bit 7): the
// gradient preconditioned by M^-1 through M's L^T D L factor in s.LD, Polak-Ribiere directions (beta
// clamped at 0), the exact line search and stopping rules of newton; no Hessian is formed.
template <class T> __device__ int __noinline__ cg(const s3_model& m_, const s3_layout& L_, T* B_, int ncon, int nlim, bool warm_ok,
                                                  int lane) {
    const s3_model& m = c_s3m;
    WS<T> s = make_ws(B_, L_);
    const int nv = m.nv;
    const int nefc = nlim + 4 * ncon;
    const T scale = T(m.scale), tol = T(m.tolerance);
    T* Mg = s.cgm;
    T* Mg0 = s.cgm + nv;
    for (int i = lane; i < nv; i += 32) s.a[i] = warm_ok ? s.p[i] : T(0);
    __syncwarp();
    sym_mul(nv, s.M, s.a, s.Ma, lane);
    rows_mul(m, L_, B_, ncon, nlim, s.a, s.rjar, lane);
    for (int r = lane; r < nefc; r += 32) s.rjar[r] -= s.raref[r];
    __syncwarp();
    T cost = total_cost(m, L_, B_, nefc, s.a, s.Ma, s.rjar, lane);
    auto gradient = [&]() {  // grad = M a - smooth + J^T (D act jar), Mg = M^-1 grad
        for (int r = lane; r < nefc; r += 32) s.rJp[r] = s.rjar[r] < T(0) ? s.rD[r] * s.rjar[r] : T(0);
        for (int i = lane; i < nv; i += 32) s.grad[i] = s.Ma[i] - s.smooth[i];
        __syncwarp();
        rows_tmul_add(m, L_, B_, ncon, nlim, s.rJp, s.grad, lane);
        for (int i = lane; i < nv; i += 32) Mg[i] = s.grad[i];
        __syncwarp();
        solve_ldl(m, s.LD, Mg, lane);
    };
    gradient();
    for (int i = lane; i < nv; i += 32) s.p[i] = -Mg[i];
    __syncwarp();
    int its = 0;
    for (int it = 0; it < m.iterations; ++it) {
        T gn = T(0);
        for (int i = lane; i < nv; i += 32) gn += s.grad[i] * s.grad[i];
        gn = wsum(gn);
        if (scale * sqrt(gn) < tol) break;
        ++its;
        sym_mul(nv, s.M, s.p, s.Mp, lane);
        rows_mul(m, L_, B_, ncon, nlim, s.p, s.rJp, lane);
        T g0 = T(0), h0 = T(0);
        for (int i = lane; i < nv; i += 32) {
            g0 += s.p[i] * (s.Ma[i] - s.smooth[i]);
            h0 += s.p[i] * s.Mp[i];
        }
        g0 = wsum(g0);
        h0 = wsum(h0);
        auto deriv = [&](T al, T& d1, T& d2) {
            T x1 = T(0), x2 = T(0);
            for (int r = lane; r < nefc; r += 32) {
                T x = s.rjar[r] + al * s.rJp[r];
                if (x < T(0)) {
                    x1 += s.rD[r] * x * s.rJp[r];
                    x2 += s.rD[r] * s.rJp[r] * s.rJp[r];
                }
            }
            d1 = g0 + al * h0 + wsum(x1);
            d2 = h0 + wsum(x2);
        };
        T d0, dd;
        deriv(T(0), d0, dd);
        T alpha = T(0);
        if (d0 < T(0)) {
            T lo = T(0), hi = T(INFINITY), al = T(1);
            for (int li = 0; li < m.ls_iterations; ++li) {
                T d1, d2;
                deriv(al, d1, d2);
                if (fabs(d1) < T(m.ls_tolerance) * fabs(d0)) break;
                if (d1 < T(0)) lo = al;
                else hi = al;
                T an = al - d1 / d2;
                if (!(lo < an && an < hi)) an = T(0.5) * (lo + hi);
                al = an;
            }
            alpha = al;
        }
        if (alpha == T(0)) break;
        for (int i = lane; i < nv; i += 32) {
            s.a[i] += alpha * s.p[i];
            s.Ma[i] += alpha * s.Mp[i];
        }
        for (int r = lane; r < nefc; r += 32) s.rjar[r] += alpha * s.rJp[r];
        __syncwarp();
        const T nc = total_cost(m, L_, B_, nefc, s.a, s.Ma, s.rjar, lane);
        const T impv = scale * (cost - nc);
        cost = nc;
        // previous gradient: gold . Mgold, and Mgold kept for the Polak-Ribiere numerator
        T den = T(0);
        for (int i = lane; i < nv; i += 32) {
            den += s.grad[i] * Mg[i];
            Mg0[i] = Mg[i];
        }
        den = wsum(den);
        __syncwarp();
        gradient();
        if (impv < tol) break;
        T num = T(0);
        for (int i = lane; i < nv; i += 32) num += s.grad[i] * (Mg[i] - Mg0[i]);
        num = wsum(num);
        const T beta = fmax(T(0), num / fmax(T(1e-15), den));
        for (int i = lane; i < nv; i += 32) s.p[i] = -Mg[i] + beta * s.p[i];
        __syncwarp();
    }
    for (int r = lane; r < nefc; r += 32) s.rJp[r] = s.rjar[r] < T(0) ? -s.rD[r] * s.rjar[r] : T(0);
    for (int i = lane; i < nv; i += 32) s.fcon[i] = T(0);
    __syncwarp();
    rows_tmul_add(m, L_, B_, ncon, nlim, s.rJp, s.fcon, lane);
    return its;
}

// ---------------------------------------------------------------- one physics substep (mj_step)

template <class T>
__device__ __noinline__ int substep(const s3_model& m_, const s3_data& d, const s3_layout& L_, T* B_, int64_t w, T* gw, const T* gapp, bool last,
                        int lane, const uint8_t* psens = nullptr, uint32_t* found = nullptr) {
    const s3_model& m = model_ref<T>(m_);  // float64: the constant-bank copy (see c_s3m)
    WS<T> s = make_ws(B_, L_);
    const int nv = m.nv;
    const T dt = T(m.timestep);
    int ncon = 0, nlim = 0, dropped = 0, its = 0;
    // block phase sync (flags bits 3-5; full blocks only): the warps of a block start every substep and
    // leave the Newton solve together, so they walk the same code and model tables at the same time -- the
    // ~26 KB of L1 beside the workspace and the instruction cache then hold one stage's working set instead
    // of every stage's (G1, 4096 worlds: f32 4.24 -> 2.98 ms, f64 6.65 -> 5.87 ms per control step)
    const bool bsync = (m.flags & 56) && (int64_t)(blockIdx.x + 1) * L_.warps_per_block <= d.nworld;
    if (bsync && (m.flags & 8)) __syncthreads();
    kinematics(m, L_, B_, lane);
    com_pos(m, L_, B_, lane, d.mass_scale ? static_cast<const T*>(d.mass_scale)[w] : T(1));
    rne(m, L_, B_, lane);
    crb_mass(m, L_, B_, lane);
    int np = nv * (nv + 1) / 2;
    const T fscale = d.friction_scale ? static_cast<const T*>(d.friction_scale)[w] : T(1);
    ncon = collide(m, L_, B_, lane, dropped, fscale);
    if (psens) {
        // contact sensors (s3_task.pair_sensor): per sensor, this substep's contacts on its pairs; byte k of
        // *found keeps the most any substep of the control step saw (ncon <= S3_MAX_CON < 32: one per lane)
        const unsigned bits = lane < ncon ? psens[s.con_pair[lane]] : 0u;
#pragma unroll
        for (int k = 0; k < S3_MAX_SENSOR; ++k) {
            const uint32_t n = (uint32_t)__popc(__ballot_sync(FULL, (bits >> k) & 1u));
            if (n > ((*found >> (8 * k)) & 255u)) *found = (*found & ~(255u << (8 * k))) | (n << (8 * k));
        }
    }
    uint64_t U = (m.flags & 1) ? (nv == 64 ? ~0ull : ((1ull << nv) - 1)) : touched_mask(m, L_, B_, ncon, lane);
    tree_load(m, s.M, s.LD, lane);
    factor_ldl(m, s.LD, s.tk, lane, U, 1);          // subtrees no constraint touches: shared by M and H
    tree_copy(m, s.LD, s.snap, U, true, lane);
    smooth_force(m, L_, B_, gapp, lane);
    if (last && d.qM) {
        // parity outputs only: finish M's factor and qacc_smooth = M^-1 f (the solver does not need them:
        // Newton starts from the warm start and its first iteration factors H over the touched rows)
        factor_ldl(m, s.LD, s.tk, lane, U, 2);
        T* o = static_cast<T*>(d.qLD) + w * np;
        const unsigned long long* cm = reinterpret_cast<const unsigned long long*>(m.dof_chainmask);
        for (int i = lane; i < nv; i += 32) {
            uint64_t mk = __ldg(cm + i);
            for (int j = 0; j <= i; ++j) o[tri(i, j)] = ((mk >> j) & 1ull) ? s.LD[tri(i, j)] : T(0);
        }
        for (int i = lane; i < nv; i += 32) s.a0[i] = s.smooth[i];
        __syncwarp();
        solve_ldl(m, s.LD, s.a0, lane);
        // bias and qacc_smooth alias Newton scratch: emit them now
        for (int i = lane; i < nv; i += 32) {
            static_cast<T*>(d.qfrc_bias)[w * nv + i] = s.bias[i];
            static_cast<T*>(d.qacc_smooth)[w * nv + i] = s.a0[i];
        }
    }
    if (last && d.qM) {  // parity output; the constraint-force row buffer may reuse cdof's slot from here on
        for (int i = lane; i < nv; i += 32)
            for (int k = 0; k < 6; ++k) static_cast<T*>(d.cdof)[(w * nv + i) * 6 + k] = s.cdof[6 * i + k];
        __syncwarp();
    }
    build_rows(m, L_, B_, ncon, nlim, lane);
    if (bsync && (m.flags & 16)) __syncthreads();
    if (gw) {
        for (int i = lane; i < nv; i += 32) s.p[i] = gw[i];
        __syncwarp();
    }
    if (m.flags & 128) {  // CG: the solver preconditions with M's full factor
        if (!(last && d.qM)) factor_ldl(m, s.LD, s.tk, lane, U, 2);  // (the parity path finished it above)
        its = cg(m, L_, B_, ncon, nlim, gw != nullptr, lane);
    } else {
        its = newton(m, L_, B_, ncon, nlim, gw != nullptr, U, lane);
    }
    if (gw) {
        for (int i = lane; i < nv; i += 32) gw[i] = s.a[i];
    }
    if (bsync && (m.flags & 32)) __syncthreads();
    // implicitfast: (M + dt diag(damping + kv)) acc = smooth + constraint
    const T* damp = F<T>(m.dof_damping);
    tree_load(m, s.M, s.LD, lane);
    for (int i = lane; i < nv; i += 32) s.LD[tri(i, i)] += dt * (damp[i] + s.kvd[i]);
    for (int i = lane; i < nv; i += 32) s.grad[i] = s.smooth[i] + s.fcon[i];
    __syncwarp();
    if (last && d.qM) {  // parity outputs (pre-integration quantities)
        T* oM = static_cast<T*>(d.qM) + w * np;
        for (int t = lane; t < np; t += 32) oM[t] = s.M[t];
        for (int i = lane; i < nv; i += 32) {
            static_cast<T*>(d.qfrc_smooth)[w * nv + i] = s.smooth[i];
            static_cast<T*>(d.qacc)[w * nv + i] = s.a[i];
            static_cast<T*>(d.qfrc_constraint)[w * nv + i] = s.fcon[i];
        }
        for (int b = lane; b < m.nbody; b += 32) {
            for (int k = 0; k < 3; ++k) static_cast<T*>(d.xpos)[(w * m.nbody + b) * 3 + k] = s.xpos[3 * b + k];
            for (int k = 0; k < 4; ++k) static_cast<T*>(d.xquat)[(w * m.nbody + b) * 4 + k] = s.xquat[4 * b + k];
        }
        for (int k = lane; k < 3 * m.nkintree; k += 32) static_cast<T*>(d.com)[w * 3 * S3_MAX_TREE + k] = s.com[k];
        for (int c = lane; c < ncon; c += 32) {
            const T* cc = s.con + kConStride * c;
            static_cast<T*>(d.con_dist)[w * S3_MAX_CON + c] = cc[0];
            for (int k = 0; k < 3; ++k) static_cast<T*>(d.con_pos)[(w * S3_MAX_CON + c) * 3 + k] = cc[1 + k];
            for (int k = 0; k < 9; ++k) static_cast<T*>(d.con_frame)[(w * S3_MAX_CON + c) * 9 + k] = cc[4 + k];
            d.con_pair[w * S3_MAX_CON + c] = s.con_pair[c];
        }
        for (int r = lane; r < nlim + 4 * ncon; r += 32) static_cast<T*>(d.efc_force)[w * S3_MAX_ROWS + r] = s.rJp[r];
        if (lane == 0) {
            d.ncon[w] = ncon;
            d.ndropped[w] = dropped;
            d.nefc[w] = nlim + 4 * ncon;
            d.solver_niter[w] = its;
        }
    }
    __syncwarp();
    factor_ldl(m, s.LD, s.tk, lane);
    solve_ldl(m, s.LD, s.grad, lane);
    for (int i = lane; i < nv; i += 32) s.qvel[i] += dt * s.grad[i];
    __syncwarp();
    // integrate positions (oracle integrate_pos)
    for (int j = lane; j < m.njnt; j += 32) {
        int a = m.jnt_qposadr[j], dd = m.jnt_dofadr[j];
        if (m.jnt_type[j] == kJntFree) {
            for (int k = 0; k < 3; ++k) s.qpos[a + k] = s.qpos[a + k] + dt * s.qvel[dd + k];
            T wv[3] = {s.qvel[dd + 3], s.qvel[dd + 4], s.qvel[dd + 5]};
            T nw = sqrt(dot3(wv, wv));
            T qt[4] = {s.qpos[a + 3], s.qpos[a + 4], s.qpos[a + 5], s.qpos[a + 6]};
            if (nw > T(1e-15)) {
                T sn, cs;
                sincos_t(T(0.5) * (nw * dt), &sn, &cs);
                T inv = T(1) / nw;
                T qa[4] = {cs, wv[0] * inv * sn, wv[1] * inv * sn, wv[2] * inv * sn};
                T r[4];
                qmul(qt, qa, r);
                qt[0] = r[0]; qt[1] = r[1]; qt[2] = r[2]; qt[3] = r[3];
            }
            qnormalize(qt);
            for (int k = 0; k < 4; ++k) s.qpos[a + 3 + k] = qt[k];
        } else {
            s.qpos[a] = s.qpos[a] + dt * s.qvel[dd];
        }
    }
    __syncwarp();
    if (d.time && lane == 0) static_cast<T*>(d.time)[w] += dt;
    return its;
}

template <class T> __device__ __noinline__ void store_geom_frames(const s3_model& m, const s3_data& d, const s3_layout& L_, T* B_, int64_t w,
                                                     int lane) {
    WS<T> s = make_ws(B_, L_);
    // frames at the FINAL state of the launch (what sensors see)
    kinematics(m, L_, B_, lane);
    for (int g = lane; g < m.ngeom; g += 32) {
        T c[3], R[9];
        geom_xform(m, s, g, c, R);
        for (int k = 0; k < 3; ++k) static_cast<T*>(d.geom_xpos)[(w * m.ngeom + g) * 3 + k] = c[k];
        for (int k = 0; k < 9; ++k) static_cast<T*>(d.geom_xmat)[(w * m.ngeom + g) * 9 + k] = R[k];
    }
}

// ---------------------------------------------------------------- the step kernel

template <class T>
__global__ void __launch_bounds__(32 * 16) step_kernel(const __grid_constant__ s3_model m, const __grid_constant__ s3_data d,
                                                      const __grid_constant__ s3_layout l, int nsub) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    int lane = threadIdx.x & 31;
    int wib = threadIdx.x >> 5;
    int64_t w = (int64_t)blockIdx.x * l.warps_per_block + wib;
    if (w >= d.nworld) return;
    T* base = reinterpret_cast<T*>(smem_raw) + (size_t)wib * l.elems_per_world;
    WS<T> s = make_ws(base, l);
    const s3_layout& L_ = l;
    T* B_ = base;
    const int nq = m.nq, nv = m.nv, nu = m.nu;
    T* gq = static_cast<T*>(d.qpos) + w * nq;
    T* gv = static_cast<T*>(d.qvel) + w * nv;
    T* gw = d.qacc_warmstart ? static_cast<T*>(d.qacc_warmstart) + w * nv : nullptr;
    const T* gapp = d.qfrc_applied ? static_cast<const T*>(d.qfrc_applied) + w * nv : nullptr;
    for (int i = lane; i < nq; i += 32) s.qpos[i] = gq[i];
    for (int i = lane; i < nv; i += 32) s.qvel[i] = gv[i];
    for (int i = lane; i < nu; i += 32) s.ctrl[i] = static_cast<const T*>(d.ctrl)[w * nu + i];
    __syncwarp();
    for (int sub = 0; sub < nsub; ++sub) substep(m, d, L_, B_, w, gw, gapp, sub == nsub - 1, lane);
    if (d.geom_xpos) store_geom_frames(m, d, L_, B_, w, lane);
    for (int i = lane; i < nq; i += 32) gq[i] = s.qpos[i];
    for (int i = lane; i < nv; i += 32) gv[i] = s.qvel[i];
}

// ---------------------------------------------------------------- the fused velocity task (task.py)

__device__ inline uint64_t mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}
constexpr uint64_t kGolden = 0x9E3779B97F4A7C15ull;
constexpr uint64_t kSalt = 0xD1B54A32D192ED03ull;

__device__ inline uint64_t stream_key(uint64_t seed, int64_t world, uint64_t purpose) {
    return mix64(mix64(seed * kGolden) ^ ((uint64_t)(world + 1) * kSalt) ^ mix64(purpose));
}

template <class T> __device__ inline T uniform01(uint64_t key, uint64_t ctr) {
    uint64_t wd = mix64(key + ctr * kGolden);
    return T((double)(wd >> 11) * (1.0 / 9007199254740992.0));
}

template <class T> __device__ inline T terrain_height(const s3_model& m, T x, T y) {
    if (!m.terrain_hfield) return T(0);
    T q[3] = {x, y, T(0)}, dd, n[3];
    if (!hfield_point(m, q, T(0), dd, n)) return T(0);
    return -dd / n[2];
}

// base-frame linear velocity, angular velocity, projected gravity from the free joint
template <class T> __device__ inline void base_frame(const T* qpos, const T* qvel, T* vb, T* om, T* g) {
    T q[4] = {qpos[3], qpos[4], qpos[5], qpos[6]};
    qnormalize(q);
    T R[9];
    qmat(q, R);
    for (int k = 0; k < 3; ++k) {
        vb[k] = R[k] * qvel[0] + R[3 + k] * qvel[1] + R[6 + k] * qvel[2];
        om[k] = qvel[3 + k];
        g[k] = -R[6 + k];
    }
}

template <class T>
__device__ __noinline__ void task_reset(const s3_model& m, const s3_task& tk, const s3_layout& L_, T* B_, int64_t w, uint64_t ctr, int lane) {
    WS<T> s = make_ws(B_, L_);
    const T* dq = static_cast<const T*>(tk.default_qpos);
    uint64_t kr = stream_key(tk.seed, tk.world_offset + w, 1);
    for (int i = lane; i < m.nq; i += 32) s.qpos[i] = dq[i];
    __syncwarp();
    for (int j = lane; j < m.njnt; j += 32) {
        if (m.jnt_type[j] == kJntFree) continue;
        // hinge index among hinge joints (joint order; the free joint, if any, comes first)
        int hi = j - (m.jnt_type[0] == kJntFree ? 1 : 0);
        int a = m.jnt_qposadr[j];
        s.qpos[a] = dq[a] + T(tk.reset_joint_jitter) * (T(2) * uniform01<T>(kr, ctr * 256 + hi) - T(1));
    }
    if (lane == 0) {
        T x = T(tk.spawn_half_extent) * (T(2) * uniform01<T>(kr, ctr * 256 + 200) - T(1));
        T y = T(tk.spawn_half_extent) * (T(2) * uniform01<T>(kr, ctr * 256 + 201) - T(1));
        T yaw = T(3.141592653589793) * (T(2) * uniform01<T>(kr, ctr * 256 + 202) - T(1));
        if (tk.curriculum) {  // centre of the world's (level row, world_id % cols) patch
            x += (T((tk.world_offset + w) % tk.terrain_cols) + T(0.5)) * T(tk.patch_size);
            y += (T(tk.terrain_level[w]) + T(0.5)) * T(tk.patch_size);
            static_cast<T*>(tk.spawn_xy)[2 * w] = x;
            static_cast<T*>(tk.spawn_xy)[2 * w + 1] = y;
            static_cast<T*>(tk.cmd_dist)[w] = T(0);
        }
        s.qpos[0] = x;
        s.qpos[1] = y;
        s.qpos[2] = dq[2] + terrain_height(m, x, y);
        T sn, cs;
        sincos_t(T(0.5) * yaw, &sn, &cs);
        s.qpos[3] = cs; s.qpos[4] = T(0); s.qpos[5] = T(0); s.qpos[6] = sn;
    }
    for (int i = lane; i < m.nv; i += 32) s.qvel[i] = T(0);
    __syncwarp();
}

template <class T>
__device__ void task_resample(const s3_task& tk, T* cmd, int64_t w, uint64_t ctr, int lane) {
    uint64_t kc = stream_key(tk.seed, tk.world_offset + w, 2);
    if (lane < 3) cmd[lane] = T(tk.cmd_lo[lane]) + T(tk.cmd_hi[lane] - tk.cmd_lo[lane]) * uniform01<T>(kc, ctr * 4 + lane);
}

template <class T>
__device__ __noinline__ void task_observe(const s3_model& m, const s3_task& tk, const s3_layout& L_, T* B_, int64_t w, uint64_t ctr, const T* cmd,
                             const T* action, int lane) {
    WS<T> s = make_ws(B_, L_);
    T vb[3], om[3], g[3];
    base_frame(s.qpos, s.qvel, vb, om, g);
    const T* dq = static_cast<const T*>(tk.default_qpos);
    uint64_t ko = stream_key(tk.seed, tk.world_offset + w, 3);
    T* out = static_cast<T*>(tk.obs) + w * tk.obs_dim;
    int nu = m.nu;
    T yaw = T(0), cy = T(1), sy = T(0);
    if (tk.nscan) {
        T q[4] = {s.qpos[3], s.qpos[4], s.qpos[5], s.qpos[6]};
        qnormalize(q);
        yaw = atan2(T(2) * (q[0] * q[3] + q[1] * q[2]), T(1) - T(2) * (q[2] * q[2] + q[3] * q[3]));
        sincos_t(yaw, &sy, &cy);
    }
    for (int i = lane; i < tk.obs_dim; i += 32) {
        T v, ns;
        if (i < 12) {
            int g3 = i / 3, k = i % 3;
            v = g3 == 0 ? vb[k] : (g3 == 1 ? om[k] : (g3 == 2 ? g[k] : cmd[k]));
            ns = T(tk.noise[g3]);
        } else if (i < 12 + nu) {
            int a = m.act_qposadr[i - 12];
            v = s.qpos[a] - dq[a];
            ns = T(tk.noise[4]);
        } else if (i < 12 + 2 * nu) {
            v = s.qvel[m.act_dofadr[i - 12 - nu]];
            ns = T(tk.noise[5]);
        } else if (i < 12 + 3 * nu) {
            v = action[i - 12 - 2 * nu];
            ns = T(tk.noise[6]);
        } else {
            int r = i - 12 - 3 * nu;
            T ox = T(tk.scan_xy[2 * r]), oy = T(tk.scan_xy[2 * r + 1]);
            T x = s.qpos[0] + cy * ox - sy * oy;
            T y = s.qpos[1] + sy * ox + cy * oy;
            T h = s.qpos[2] - terrain_height(m, x, y) - T(tk.scan_offset);
            v = fmin(fmax(h, T(-1)), T(1));
            ns = T(tk.scan_noise);
        }
        if (ns > T(0)) v += ns * (T(2) * uniform01<T>(ko, ctr * 1024 + i) - T(1));
        out[i] = v;
    }
}

// ---- domain-randomisation events (velocity and motion kinds; s3_task.events, purpose 5)

// startup: per-world friction and base-mass scales, and the first push timer (reset-all launch, counter 0)
template <class T> __device__ inline void events_startup(const s3_data& d, const s3_task& tk, int64_t w, int lane) {
    if (!tk.events || lane != 0) return;
    uint64_t k5 = stream_key(tk.seed, tk.world_offset + w, 5);
    static_cast<T*>(d.friction_scale)[w] =
        T(tk.friction_range[0]) + T(tk.friction_range[1] - tk.friction_range[0]) * uniform01<T>(k5, 0);
    static_cast<T*>(d.mass_scale)[w] =
        T(tk.base_mass_range[0]) + T(tk.base_mass_range[1] - tk.base_mass_range[0]) * uniform01<T>(k5, 5);
    static_cast<T*>(tk.event_timer)[w] =
        T(tk.push_interval[0]) + T(tk.push_interval[1] - tk.push_interval[0]) * uniform01<T>(k5, 1);
}

// masked reset: a fresh push timer (slot 1 of the step's counter)
template <class T> __device__ inline void events_reset(const s3_task& tk, int64_t w, uint64_t ctr, int lane) {
    if (!tk.events || lane != 0) return;
    uint64_t k5 = stream_key(tk.seed, tk.world_offset + w, 5);
    static_cast<T*>(tk.event_timer)[w] =
        T(tk.push_interval[0]) + T(tk.push_interval[1] - tk.push_interval[0]) * uniform01<T>(k5, ctr * 8 + 1);
}

// interval push (EventManager.apply_interval): every world after resets -- U(-v, v) on the base's planar
// velocity when its timer runs out, then a new timer
template <class T>
__device__ inline void events_interval(const s3_model& m, const s3_task& tk, T* qvel, int64_t w, uint64_t ctr, int lane) {
    if (!tk.events) return;
    T tmr = static_cast<T*>(tk.event_timer)[w] - T(m.timestep) * T(tk.decimation);
    __syncwarp();
    if (lane == 0) {
        uint64_t k5 = stream_key(tk.seed, tk.world_offset + w, 5);
        if (tmr <= T(0)) {
            T pv = T(tk.push_velocity);
            qvel[0] += pv * (T(2) * uniform01<T>(k5, ctr * 8 + 2) - T(1));
            qvel[1] += pv * (T(2) * uniform01<T>(k5, ctr * 8 + 3) - T(1));
            tmr = T(tk.push_interval[0]) + T(tk.push_interval[1] - tk.push_interval[0]) * uniform01<T>(k5, ctr * 8 + 4);
        }
        static_cast<T*>(tk.event_timer)[w] = tmr;
    }
    __syncwarp();
}

// ---- motion imitation (kind 1): reference-motion command, cmd = (motion time, anchor x, anchor y)

// reference qpos -> qr[nq], qvel -> vr[nv] at motion time t (oracle motion_ref)
template <class T>
__device__ __noinline__ void motion_ref(const s3_model& m, const s3_task& tk, T t, T* qr, T* vr, int lane) {
    const T* Q = static_cast<const T*>(tk.motion_qpos);
    const T* V = static_cast<const T*>(tk.motion_qvel);
    const int F = tk.nframes;
    T f = t / T(tk.frame_dt);
    int i0 = (int)floor(f);
    i0 = i0 < 0 ? 0 : (i0 > F - 2 ? F - 2 : i0);
    T a = f - T(i0);
    const T* q0 = Q + (size_t)i0 * m.nq;
    const T* q1 = q0 + m.nq;
    for (int i = lane; i < m.nq; i += 32) qr[i] = (T(1) - a) * q0[i] + a * q1[i];
    for (int i = lane; i < m.nv; i += 32) vr[i] = (T(1) - a) * V[(size_t)i0 * m.nv + i] + a * V[(size_t)(i0 + 1) * m.nv + i];
    __syncwarp();
    if (lane == 0) {
        T u[4] = {q0[3], q0[4], q0[5], q0[6]}, w[4] = {q1[3], q1[4], q1[5], q1[6]};
        T d = u[0] * w[0] + u[1] * w[1] + u[2] * w[2] + u[3] * w[3];
        if (d < T(0)) { w[0] = -w[0]; w[1] = -w[1]; w[2] = -w[2]; w[3] = -w[3]; }
        T qq[4];
        for (int k = 0; k < 4; ++k) qq[k] = (T(1) - a) * u[k] + a * w[k];
        T r = rsqrt_t(qq[0] * qq[0] + qq[1] * qq[1] + qq[2] * qq[2] + qq[3] * qq[3]);
        for (int k = 0; k < 4; ++k) qr[3 + k] = qq[k] * r;
    }
    __syncwarp();
}

// root position error in the base frame and orientation error (rotation vector of conj(q) q_ref)
template <class T>
__device__ inline void motion_errors(const s3_model& m, const T* qpos, const T* qr, const T* cmd, T* pe, T* re) {
    T px = qr[0] + cmd[1], py = qr[1] + cmd[2];
    T pz = qr[2] + terrain_height(m, px, py);
    T q[4] = {qpos[3], qpos[4], qpos[5], qpos[6]};
    qnormalize(q);
    T R[9];
    qmat(q, R);
    T d[3] = {px - qpos[0], py - qpos[1], pz - qpos[2]};
    for (int k = 0; k < 3; ++k) pe[k] = R[k] * d[0] + R[3 + k] * d[1] + R[6 + k] * d[2];
    T qc[4] = {q[0], -q[1], -q[2], -q[3]};
    T qf[4] = {qr[3], qr[4], qr[5], qr[6]};
    qnormalize(qf);
    T e[4];
    qmul(qc, qf, e);
    if (e[0] < T(0)) { e[0] = -e[0]; e[1] = -e[1]; e[2] = -e[2]; e[3] = -e[3]; }
    T sn = sqrt(e[1] * e[1] + e[2] * e[2] + e[3] * e[3]);
    T sc = sn < T(1e-12) ? T(2) : T(2) * atan2(sn, e[0]) / sn;
    re[0] = e[1] * sc; re[1] = e[2] * sc; re[2] = e[3] * sc;
}

// ---- BeyondMimic's relative body terms

// World state of body b (S3_BODY_STATE values: position, orientation, origin linear velocity, angular
// velocity) from the workspace's kinematics + com_pos and s.qvel: the body's spatial velocity is the sum of
// the motion vectors (cdof, about the tree's com) of the dofs on its chain (oracle body_state).
template <class T> __device__ inline void body_state(const s3_model& m, const WS<T>& s, int b, T* o) {
    for (int k = 0; k < 3; ++k) o[k] = s.xpos[3 * b + k];
    for (int k = 0; k < 4; ++k) o[3 + k] = s.xquat[4 * b + k];
    T v[6] = {T(0), T(0), T(0), T(0), T(0), T(0)};
    uint64_t mk = m.body_dofmask[b];
    while (mk) {
        const int i = __ffsll((long long)mk) - 1;
        mk &= mk - 1;
        const T qd = s.qvel[i];
        for (int k = 0; k < 6; ++k) v[k] += s.cdof[6 * i + k] * qd;
    }
    const T* com = s.com + 3 * m.body_treeid[b];
    T r[3] = {o[0] - com[0], o[1] - com[1], o[2] - com[2]}, wr[3];
    cross3(v, r, wr);
    for (int k = 0; k < 3; ++k) {
        o[7 + k] = v[3 + k] + wr[k];
        o[10 + k] = v[k];
    }
}

// body k's (0: the anchor) clip state at motion time t: the s3_motion_bodies table interpolated like
// motion_ref (linear; quaternion nlerp with sign alignment)
template <class T> __device__ inline void motion_body_ref(const s3_task& tk, T t, int k, T* o) {
    const T* Bt = static_cast<const T*>(tk.motion_body);
    const int F = tk.nframes, K1 = tk.ntrack + 1;
    T f = t / T(tk.frame_dt);
    int i0 = (int)floor(f);
    i0 = i0 < 0 ? 0 : (i0 > F - 2 ? F - 2 : i0);
    const T a = f - T(i0);
    const T* b0 = Bt + ((size_t)i0 * K1 + k) * S3_BODY_STATE;
    const T* b1 = b0 + (size_t)K1 * S3_BODY_STATE;
    for (int c = 0; c < S3_BODY_STATE; ++c) o[c] = (T(1) - a) * b0[c] + a * b1[c];
    T d = b0[3] * b1[3] + b0[4] * b1[4] + b0[5] * b1[5] + b0[6] * b1[6];
    if (d < T(0))
        for (int c = 3; c < 7; ++c) o[c] = (T(1) - a) * b0[c] - a * b1[c];
    T r = rsqrt_t(o[3] * o[3] + o[4] * o[4] + o[5] * o[5] + o[6] * o[6]);
    for (int c = 3; c < 7; ++c) o[c] *= r;
}

// squared angle of the rotation conj(a) b (quat_error_magnitude^2)
template <class T> __device__ inline T quat_err2(const T* a, const T* b) {
    T ac[4] = {a[0], -a[1], -a[2], -a[3]}, e[4];
    qmul(ac, b, e);
    T sn = sqrt(e[1] * e[1] + e[2] * e[2] + e[3] * e[3]);
    T ang = T(2) * atan2(sn, fabs(e[0]));
    return ang * ang;
}

// The four BeyondMimic body-tracking errors at the final state of the control step: the clip's tracked body
// poses re-expressed about the robot's anchor (the robot anchor's xy, the clip anchor's height above the
// terrain under the spawn anchor, the yaw between the two anchors), compared with the robot's body poses;
// body velocities compared in the world frame. Means over the tracked bodies: out[0] position (squared
// distance), out[1] orientation (squared angle), out[2] linear velocity, out[3] angular velocity.
template <class T>
__device__ __noinline__ void motion_body_errors(const s3_model& m, const s3_task& tk, const s3_layout& L_, T* B_, T tnow,
                                                const T* cmd, T* out, int lane) {
    WS<T> s = make_ws(B_, L_);
    kinematics(m, L_, B_, lane);
    com_pos(m, L_, B_, lane, T(1));
    const int K1 = tk.ntrack + 1;
    T rb[S3_BODY_STATE], rf[S3_BODY_STATE];
    if (lane < K1) {
        body_state(m, s, lane ? tk.track_body[lane - 1] : tk.anchor_body, rb);
        motion_body_ref(tk, tnow, lane, rf);
    }
    T pa[3], qa[4], pr[3], qr[4];
    for (int k = 0; k < 3; ++k) {
        pa[k] = __shfl_sync(FULL, rb[k], 0);
        pr[k] = __shfl_sync(FULL, rf[k], 0);
    }
    for (int k = 0; k < 4; ++k) {
        qa[k] = __shfl_sync(FULL, rb[3 + k], 0);
        qr[k] = __shfl_sync(FULL, rf[3 + k], 0);
    }
    // yaw of qa conj(qr)
    T qrc[4] = {qr[0], -qr[1], -qr[2], -qr[3]}, dq[4];
    qmul(qa, qrc, dq);
    T yaw = atan2(T(2) * (dq[0] * dq[3] + dq[1] * dq[2]), T(1) - T(2) * (dq[2] * dq[2] + dq[3] * dq[3]));
    T sy, cy;
    sincos_t(T(0.5) * yaw, &sy, &cy);
    const T dy[4] = {cy, T(0), T(0), sy};
    const T tz = pr[2] + terrain_height(m, pr[0] + cmd[1], pr[1] + cmd[2]);
    T e[4] = {T(0), T(0), T(0), T(0)};
    if (lane >= 1 && lane < K1) {
        T R[9], rel[3] = {rf[0] - pr[0], rf[1] - pr[1], rf[2] - pr[2]}, rot[3];
        qmat(dy, R);
        mv3(R, rel, rot);
        T p[3] = {pa[0] + rot[0], pa[1] + rot[1], tz + rot[2]};
        T qh[4];
        qmul(dy, rf + 3, qh);
        for (int k = 0; k < 3; ++k) {
            e[0] += (p[k] - rb[k]) * (p[k] - rb[k]);
            e[2] += (rf[7 + k] - rb[7 + k]) * (rf[7 + k] - rb[7 + k]);
            e[3] += (rf[10 + k] - rb[10 + k]) * (rf[10 + k] - rb[10 + k]);
        }
        e[1] = quat_err2(qh, rb + 3);
    }
    const T inv = T(1) / T(tk.ntrack);
    for (int k = 0; k < 4; ++k) out[k] = wsum(e[k]) * inv;
}

template <class T>
__device__ __noinline__ void motion_reset(const s3_model& m, const s3_task& tk, const s3_layout& L_, T* B_, int64_t w,
                                          uint64_t ctr, T* cmd, int lane) {
    WS<T> s = make_ws(B_, L_);
    uint64_t kr = stream_key(tk.seed, tk.world_offset + w, 1);
    const T clip_end = T(tk.nframes - 1) * T(tk.frame_dt);
    T t0;
    if (tk.nbins > 0) {  // adaptive sampling: a bin by the cumulative weights of the last fold, a time inside it
        const T* cum = static_cast<const T*>(tk.bin_cum);
        const T target = uniform01<T>(kr, ctr * 256 + 203) * cum[tk.nbins - 1];
        int b = 0;
        while (b < tk.nbins - 1 && !(target < cum[b])) ++b;
        t0 = (T(b) + uniform01<T>(kr, ctr * 256 + 204)) / T(tk.nbins) * clip_end;
    } else {
        t0 = T(tk.motion_start_frac) * clip_end * uniform01<T>(kr, ctr * 256 + 203);
    }
    T ax = T(tk.spawn_half_extent) * (T(2) * uniform01<T>(kr, ctr * 256 + 200) - T(1));
    T ay = T(tk.spawn_half_extent) * (T(2) * uniform01<T>(kr, ctr * 256 + 201) - T(1));
    motion_ref(m, tk, t0, s.qpos, s.qvel, lane);
    if (lane == 0) {
        s.qpos[0] += ax;
        s.qpos[1] += ay;
        s.qpos[2] += terrain_height(m, s.qpos[0], s.qpos[1]);
        cmd[0] = t0; cmd[1] = ax; cmd[2] = ay;
    }
    __syncwarp();
}

template <class T>
__device__ __noinline__ void motion_observe(const s3_model& m, const s3_task& tk, const s3_layout& L_, T* B_, int64_t w,
                                            uint64_t ctr, const T* cmd, const T* action, int lane) {
    WS<T> s = make_ws(B_, L_);
    T* qr = s.LD;
    T* vr = s.LD + m.nq;
    motion_ref(m, tk, cmd[0], qr, vr, lane);
    T vb[3], om[3], g[3], pe[3], re[3];
    base_frame(s.qpos, s.qvel, vb, om, g);
    motion_errors(m, s.qpos, qr, cmd, pe, re);
    const T* dq = static_cast<const T*>(tk.default_qpos);
    uint64_t ko = stream_key(tk.seed, tk.world_offset + w, 3);
    T* out = static_cast<T*>(tk.obs) + w * tk.obs_dim;
    const int nu = m.nu;
    // [ref joint pos - default, ref joint vel, v_b, w_b, g_b, pos err_b, rot err, joint pos - default, joint vel, action]
    for (int i = lane; i < tk.obs_dim; i += 32) {
        T v, ns = T(0);
        if (i < nu) {
            int a = m.act_qposadr[i];
            v = qr[a] - dq[a];
        } else if (i < 2 * nu) {
            v = vr[m.act_dofadr[i - nu]];
        } else if (i < 2 * nu + 15) {
            int r = i - 2 * nu, g3 = r / 3, k = r % 3;
            v = g3 == 0 ? vb[k] : (g3 == 1 ? om[k] : (g3 == 2 ? g[k] : (g3 == 3 ? pe[k] : re[k])));
            ns = g3 < 3 ? T(tk.noise[g3]) : T(0);
        } else if (i < 3 * nu + 15) {
            int a = m.act_qposadr[i - 2 * nu - 15];
            v = s.qpos[a] - dq[a];
            ns = T(tk.noise[4]);
        } else if (i < 4 * nu + 15) {
            v = s.qvel[m.act_dofadr[i - 3 * nu - 15]];
            ns = T(tk.noise[5]);
        } else {
            v = action[i - 4 * nu - 15];
            ns = T(tk.noise[6]);
        }
        if (ns > T(0)) v += ns * (T(2) * uniform01<T>(ko, ctr * 1024 + i) - T(1));
        out[i] = v;
    }
}

template <class T>
__device__ __noinline__ void motion_post(const s3_model& m, const s3_task& tk, const s3_layout& L_, T* B_, int64_t w,
                                         uint64_t ctr, T* cmd, T* act, T rate, T* gq, T* gv, T* gw, T* prev,
                                         uint32_t found, int lane) {
    WS<T> s = make_ws(B_, L_);
    const int nu = m.nu, nq = m.nq, nv = m.nv;
    const T dtc = T(m.timestep) * T(tk.decimation);
    T tnow = cmd[0] + dtc;
    __syncwarp();
    if (lane == 0) cmd[0] = tnow;
    __syncwarp();
    T* qr = s.LD;
    T* vr = s.LD + nq;
    motion_ref(m, tk, tnow, qr, vr, lane);
    T pe[3], re[3];
    T c3[3] = {tnow, cmd[1], cmd[2]};
    motion_errors(m, s.qpos, qr, c3, pe, re);
    T ej = T(0), ev = T(0);
    for (int i = lane; i < nu; i += 32) {
        int a = m.act_qposadr[i], d = m.act_dofadr[i];
        T dq = s.qpos[a] - qr[a], dv = s.qvel[d] - vr[d];
        ej += dq * dq;
        ev += dv * dv;
    }
    ej = wsum(ej);
    ev = wsum(ev);
    T be[4] = {T(0), T(0), T(0), T(0)};
    if (tk.ntrack) motion_body_errors(m, tk, L_, B_, tnow, cmd, be, lane);
    // joint pos / vel, anchor pos / ori, action rate, body pos / ori / lin vel / ang vel, self contacts
    T terms[10] = {exp(-ej / T(tk.motion_sigmas[0])), exp(-ev / T(tk.motion_sigmas[1])),
                   exp(-(pe[0] * pe[0] + pe[1] * pe[1] + pe[2] * pe[2]) / T(tk.motion_sigmas[2])),
                   exp(-(re[0] * re[0] + re[1] * re[1] + re[2] * re[2]) / T(tk.motion_sigmas[3])), rate,
                   T(0), T(0), T(0), T(0), T(found & 255u)};
    if (tk.ntrack)
        for (int k = 0; k < 4; ++k) terms[5 + k] = exp(-be[k] / T(tk.motion_sigmas[4 + k]));
    T r = T(0);
    for (int k = 0; k < 10; ++k) r += T(tk.reward_weights[k]) * terms[k] * dtc;
    bool finite = true;
    for (int i = lane; i < nq; i += 32) finite = finite && isfinite(s.qpos[i]);
    for (int i = lane; i < nv; i += 32) finite = finite && isfinite(s.qvel[i]);
    finite = __all_sync(FULL, finite);
    T rot = sqrt(re[0] * re[0] + re[1] * re[1] + re[2] * re[2]);
    bool term = fabs(pe[2]) > T(tk.max_height_error) || rot > T(tk.max_ori_error) || !finite;
    int es = tk.episode_step[w] + 1;
    const T clip_end = T(tk.nframes - 1) * T(tk.frame_dt);
    if (tk.nbins > 0 && term && lane == 0) {  // adaptive sampling: a failure in the bin of its motion time
        int b = (int)floor(tnow / clip_end * T(tk.nbins));
        b = b < 0 ? 0 : (b > tk.nbins - 1 ? tk.nbins - 1 : b);
        atomicAdd(tk.bin_fail_now + b, 1u);
    }
    bool trunc = es >= tk.episode_steps || tnow >= clip_end - T(1e-9);
    __syncwarp();
    if (lane == 0) {
        static_cast<T*>(tk.reward)[w] = r;
        static_cast<T*>(tk.episode_return)[w] += r;
        tk.terminated[w] = term;
        tk.truncated[w] = trunc;
        tk.episode_step[w] = es;
    }
    if (term || trunc) {
        motion_reset(m, tk, L_, B_, w, ctr, cmd, lane);
        events_reset<T>(tk, w, ctr, lane);
        for (int i = lane; i < nv; i += 32) gw[i] = T(0);
        for (int i = lane; i < nu; i += 32) { act[i] = T(0); prev[i] = T(0); }
        if (lane == 0) {
            tk.episode_step[w] = 0;
            static_cast<T*>(tk.episode_return)[w] = T(0);
        }
    }
    __syncwarp();
    events_interval(m, tk, s.qvel, w, ctr, lane);  // pushes after resets, like the velocity kind
    motion_observe(m, tk, L_, B_, w, ctr, cmd, act, lane);
    for (int i = lane; i < nq; i += 32) gq[i] = s.qpos[i];
    for (int i = lane; i < nv; i += 32) gv[i] = s.qvel[i];
}

// ---- cube lift (kind 2): cmd = goal position; claw position = mean of the two fingertip spheres

template <class T>
__device__ __noinline__ void lift_ee(const s3_model& m, const s3_task& tk, const s3_layout& L_, T* B_, T* ee, int lane) {
    WS<T> s = make_ws(B_, L_);
    kinematics(m, L_, B_, lane);
    T c0[3], c1[3], R[9];
    geom_xform(m, s, tk.tip_geom[0], c0, R);
    geom_xform(m, s, tk.tip_geom[1], c1, R);
    for (int k = 0; k < 3; ++k) ee[k] = T(0.5) * (c0[k] + c1[k]);
}

template <class T>
__device__ __noinline__ void lift_reset(const s3_model& m, const s3_task& tk, const s3_layout& L_, T* B_, int64_t w,
                                        uint64_t ctr, T* cmd, int lane) {
    WS<T> s = make_ws(B_, L_);
    const T* dq = static_cast<const T*>(tk.default_qpos);
    uint64_t kr = stream_key(tk.seed, tk.world_offset + w, 1);
    for (int i = lane; i < m.nq; i += 32) s.qpos[i] = dq[i];
    __syncwarp();
    int nh = 0;  // hinge index among hinge joints, in joint order (the oracle's enumeration)
    for (int j = 0; j < m.njnt; ++j) {
        if (m.jnt_type[j] == kJntFree) continue;
        if ((nh & 31) == lane) {
            int a = m.jnt_qposadr[j];
            s.qpos[a] = dq[a] + T(tk.reset_joint_jitter) * (T(2) * uniform01<T>(kr, ctr * 256 + nh) - T(1));
        }
        ++nh;
    }
    if (lane == 0) {
        const int ca = tk.cube_qposadr;
        s.qpos[ca] = T(tk.cube_x[0]) + T(tk.cube_x[1] - tk.cube_x[0]) * uniform01<T>(kr, ctr * 256 + 200);
        s.qpos[ca + 1] = T(tk.cube_y[0]) + T(tk.cube_y[1] - tk.cube_y[0]) * uniform01<T>(kr, ctr * 256 + 201);
        s.qpos[ca + 2] = T(tk.cube_half);
        T yaw = T(3.141592653589793) * (T(2) * uniform01<T>(kr, ctr * 256 + 202) - T(1));
        T sn, cs;
        sincos_t(T(0.5) * yaw, &sn, &cs);
        s.qpos[ca + 3] = cs; s.qpos[ca + 4] = T(0); s.qpos[ca + 5] = T(0); s.qpos[ca + 6] = sn;
    }
    for (int i = lane; i < m.nv; i += 32) s.qvel[i] = T(0);
    task_resample(tk, cmd, w, ctr, lane);  // goal ~ U(cmd_lo, cmd_hi), purpose 2
    __syncwarp();
}

template <class T>
__device__ __noinline__ void lift_observe(const s3_model& m, const s3_task& tk, const s3_layout& L_, T* B_, int64_t w,
                                          uint64_t ctr, const T* cmd, const T* action, int lane) {
    WS<T> s = make_ws(B_, L_);
    T ee[3];
    lift_ee(m, tk, L_, B_, ee, lane);
    const T* dq = static_cast<const T*>(tk.default_qpos);
    uint64_t ko = stream_key(tk.seed, tk.world_offset + w, 3);
    T* out = static_cast<T*>(tk.obs) + w * tk.obs_dim;
    const int nu = m.nu, ca = tk.cube_qposadr;
    // [joint pos - default, joint vel, cube pos, cube quat, claw pos, goal, action]
    for (int i = lane; i < tk.obs_dim; i += 32) {
        T v, ns = T(0);
        if (i < nu) {
            int a = m.act_qposadr[i];
            v = s.qpos[a] - dq[a];
            ns = T(tk.noise[4]);
        } else if (i < 2 * nu) {
            v = s.qvel[m.act_dofadr[i - nu]];
            ns = T(tk.noise[5]);
        } else if (i < 2 * nu + 7) {
            v = s.qpos[ca + i - 2 * nu];
        } else if (i < 2 * nu + 10) {
            v = ee[i - 2 * nu - 7];
        } else if (i < 2 * nu + 13) {
            v = cmd[i - 2 * nu - 10];
        } else {
            v = action[i - 2 * nu - 13];
            ns = T(tk.noise[6]);
        }
        if (ns > T(0)) v += ns * (T(2) * uniform01<T>(ko, ctr * 1024 + i) - T(1));
        out[i] = v;
    }
}

template <class T>
__device__ __noinline__ void lift_post(const s3_model& m, const s3_task& tk, const s3_layout& L_, T* B_, int64_t w,
                                       uint64_t ctr, T* cmd, T* act, T rate, T* gq, T* gv, T* gw, T* prev,
                                       uint32_t found, int lane) {
    WS<T> s = make_ws(B_, L_);
    const int nu = m.nu, nq = m.nq, nv = m.nv, ca = tk.cube_qposadr;
    const T dtc = T(m.timestep) * T(tk.decimation);
    T ee[3];
    lift_ee(m, tk, L_, B_, ee, lane);
    T cube[3] = {s.qpos[ca], s.qpos[ca + 1], s.qpos[ca + 2]};
    T de[3] = {ee[0] - cube[0], ee[1] - cube[1], ee[2] - cube[2]};
    T dg[3] = {cube[0] - cmd[0], cube[1] - cmd[1], cube[2] - cmd[2]};
    T d_ee = sqrt(dot3(de, de)), d_goal = sqrt(dot3(dg, dg));
    T lifted = cube[2] > T(tk.lift_height) ? T(1) : T(0);
    T jv = T(0);
    for (int i = lane; i < nu; i += 32) {
        T v = s.qvel[m.act_dofadr[i]];
        jv += v * v;
    }
    jv = wsum(jv);
    // reach, lifted, goal tracking, action rate, joint velocity, end-effector / ground contacts (sensor 1)
    T terms[6] = {T(1) - tanh(d_ee / T(tk.reach_std)), lifted, lifted * (T(1) - tanh(d_goal / T(tk.goal_std))), rate, jv,
                  T((found >> 8) & 255u)};
    T r = T(0);
    for (int k = 0; k < 6; ++k) r += T(tk.reward_weights[k]) * terms[k] * dtc;
    bool finite = true;
    for (int i = lane; i < nq; i += 32) finite = finite && isfinite(s.qpos[i]);
    for (int i = lane; i < nv; i += 32) finite = finite && isfinite(s.qvel[i]);
    finite = __all_sync(FULL, finite);
    bool term = cube[2] < T(tk.min_cube_z) || !finite;
    int es = tk.episode_step[w] + 1;
    bool trunc = es >= tk.episode_steps;
    __syncwarp();
    if (lane == 0) {
        static_cast<T*>(tk.reward)[w] = r;
        static_cast<T*>(tk.episode_return)[w] += r;
        tk.terminated[w] = term;
        tk.truncated[w] = trunc;
        tk.episode_step[w] = es;
    }
    if (term || trunc) {
        lift_reset(m, tk, L_, B_, w, ctr, cmd, lane);
        for (int i = lane; i < nv; i += 32) gw[i] = T(0);
        for (int i = lane; i < nu; i += 32) { act[i] = T(0); prev[i] = T(0); }
        if (lane == 0) {
            tk.episode_step[w] = 0;
            static_cast<T*>(tk.episode_return)[w] = T(0);
        }
    }
    __syncwarp();
    lift_observe(m, tk, L_, B_, w, ctr, cmd, act, lane);
    for (int i = lane; i < nq; i += 32) gq[i] = s.qpos[i];
    for (int i = lane; i < nv; i += 32) gv[i] = s.qvel[i];
}

// mjlab's velocity-task penalties beyond the base-frame terms, at the final state of the control step:
// out[0] |centroidal angular momentum|^2 of the robot (tree 0: sum over its bodies of the angular part of
// cinert x cvel, about the tree's com), out[1] joint-limit violation (sum over limited joints of the distance
// outside [lo, hi]), out[2] foot slip (sum over feet in contact -- contact sensors 0..nfeet-1 -- of the
// foot body's squared horizontal velocity). Kinematics + com_pos run only when a weight needs them.
template <class T>
__device__ __noinline__ void velocity_extra_terms(const s3_model& m, const s3_data& d, const s3_task& tk, const s3_layout& L_,
                                                  T* B_, int64_t w, uint32_t found, T* out, int lane) {
    WS<T> s = make_ws(B_, L_);
    T lim = T(0);
    if (tk.reward_weights[7] != 0.0) {
        const T* rg = F<T>(m.lim_range);
        for (int l = lane; l < m.nlimjnt; l += 32) {
            const T q = s.qpos[m.lim_qposadr[l]];
            lim += fmax(rg[2 * l] - q, T(0)) + fmax(q - rg[2 * l + 1], T(0));
        }
        lim = wsum(lim);
    }
    T h[3] = {T(0), T(0), T(0)}, slip = T(0);
    if (tk.reward_weights[6] != 0.0 || (tk.reward_weights[8] != 0.0 && tk.nfeet > 0)) {
        kinematics(m, L_, B_, lane);
        com_pos(m, L_, B_, lane, d.mass_scale ? static_cast<const T*>(d.mass_scale)[w] : T(1));
        if (tk.reward_weights[6] != 0.0) {
            for (int b = 1 + lane; b < m.nbody; b += 32) {
                if (m.body_treeid[b] != 0) continue;
                T v[6] = {T(0), T(0), T(0), T(0), T(0), T(0)}, f[6];
                uint64_t mk = m.body_dofmask[b];
                while (mk) {
                    const int i = __ffsll((long long)mk) - 1;
                    mk &= mk - 1;
                    for (int k = 0; k < 6; ++k) v[k] += s.cdof[6 * i + k] * s.qvel[i];
                }
                inert_mul(s.cinert + 10 * b, v, f);
                h[0] += f[0]; h[1] += f[1]; h[2] += f[2];
            }
            h[0] = wsum(h[0]); h[1] = wsum(h[1]); h[2] = wsum(h[2]);
        }
        if (tk.reward_weights[8] != 0.0 && lane < tk.nfeet && ((found >> (8 * lane)) & 255u)) {
            T o[S3_BODY_STATE];
            body_state(m, s, tk.foot_body[lane], o);
            slip = o[7] * o[7] + o[8] * o[8];
        }
        slip = wsum(slip);
    }
    out[0] = h[0] * h[0] + h[1] * h[1] + h[2] * h[2];
    out[1] = lim;
    out[2] = slip;
}

// Adaptive sampling (s3_task.nbins): the last world of the launch to finish (a per-warp ticket, so no block
// barrier) folds the launch's failure counts into the exponential average and rebuilds the cumulative
// sampling weights for the next launch -- one thread, bins in order (oracle MotionTaskOracle.fold_bins)
template <class T> __device__ __noinline__ void adaptive_fold(const s3_task& tk, int64_t nworld, int lane) {
    __syncwarp();
    unsigned last = 0;
    if (lane == 0) {
        __threadfence();  // this world's failure count before its ticket
        last = atomicInc(tk.bin_ticket, (unsigned)(nworld - 1)) == (unsigned)(nworld - 1);
    }
    last = __shfl_sync(FULL, last, 0);
    if (!last || lane != 0) return;
    __threadfence();
    T* F = static_cast<T*>(tk.bin_failed);
    T* C = static_cast<T*>(tk.bin_cum);
    const int nb = tk.nbins;
    const T a = T(tk.adaptive_alpha);
    for (int b = 0; b < nb; ++b) {
        const T now = T(atomicExch(tk.bin_fail_now + b, 0u));
        F[b] = a * now + (T(1) - a) * F[b];
    }
    const T u = T(tk.adaptive_uniform) / T(nb);
    T acc = T(0);
    for (int b = 0; b < nb; ++b) {
        T q = T(0);
        for (int i = 0; i < tk.nkernel; ++i) {
            const int j = b + i < nb - 1 ? b + i : nb - 1;
            q += T(tk.adaptive_kernel[i]) * (F[j] + u);
        }
        acc += q;
        C[b] = acc;
    }
}

template <class T>
__global__ void __launch_bounds__(32 * 16) env_kernel(const __grid_constant__ s3_model m, const __grid_constant__ s3_data d,
                                                     const __grid_constant__ s3_layout l,
                                                     const __grid_constant__ s3_task tk, const T* __restrict__ actions,
                                                     int mode, int64_t global_step) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    int lane = threadIdx.x & 31;
    int wib = threadIdx.x >> 5;
    int64_t w = (int64_t)blockIdx.x * l.warps_per_block + wib;
    if (w >= d.nworld) return;
    if (tk.order && mode == 0) w = tk.order[w];  // cost-ordered schedule (s3_task.order; sorted before each step)
    T* base = reinterpret_cast<T*>(smem_raw) + (size_t)wib * l.elems_per_world;
    WS<T> s = make_ws(base, l);
    const s3_layout& L_ = l;
    T* B_ = base;
    const int nq = m.nq, nv = m.nv, nu = m.nu;
    T* gq = static_cast<T*>(d.qpos) + w * nq;
    T* gv = static_cast<T*>(d.qvel) + w * nv;
    T* gw = static_cast<T*>(d.qacc_warmstart) + w * nv;
    T* act = static_cast<T*>(tk.action) + w * nu;
    T* prev = static_cast<T*>(tk.prev_action) + w * nu;
    T* cmd = static_cast<T*>(tk.command) + w * 3;
    const T* dq = static_cast<const T*>(tk.default_qpos);
    uint64_t ctr = (uint64_t)global_step;
    if (mode == 1) {  // reset every world, counter 0
        if (tk.kind == 1) {
            motion_reset(m, tk, L_, B_, w, 0, cmd, lane);
        } else if (tk.kind == 2) {
            lift_reset(m, tk, L_, B_, w, 0, cmd, lane);
        } else {
            if (tk.curriculum && lane == 0) {  // initial terrain level (purpose 6, counter 0)
                int lv = (int)(uniform01<T>(stream_key(tk.seed, tk.world_offset + w, 6), 0) *
                               T(tk.curriculum_max_init_level + 1));
                tk.terrain_level[w] = lv < tk.terrain_rows - 1 ? lv : tk.terrain_rows - 1;
            }
            __syncwarp();
            task_reset(m, tk, L_, B_, w, 0, lane);
            task_resample(tk, cmd, w, 0, lane);
        }
        if (tk.kind != 2) events_startup<T>(d, tk, w, lane);  // friction / mass scales, first push timer
        for (int i = lane; i < nv; i += 32) gw[i] = T(0);
        for (int i = lane; i < nu; i += 32) { act[i] = T(0); prev[i] = T(0); }
        if (lane == 0) {
            tk.cmd_timer[w] = tk.kind == 0 ? tk.cmd_resample_steps : 0;
            tk.episode_step[w] = 0;
            static_cast<T*>(tk.episode_return)[w] = T(0);
        }
        __syncwarp();
        if (tk.kind == 1) motion_observe(m, tk, L_, B_, w, 0, cmd, act, lane);
        else if (tk.kind == 2) lift_observe(m, tk, L_, B_, w, 0, cmd, act, lane);
        else task_observe(m, tk, L_, B_, w, 0, cmd, act, lane);
        if (d.geom_xpos) store_geom_frames(m, d, L_, B_, w, lane);
        for (int i = lane; i < nq; i += 32) gq[i] = s.qpos[i];
        for (int i = lane; i < nv; i += 32) gv[i] = s.qvel[i];
        return;
    }
    for (int i = lane; i < nq; i += 32) s.qpos[i] = gq[i];
    for (int i = lane; i < nv; i += 32) s.qvel[i] = gv[i];
    // ActionManager.process: clip, remember the previous action, position targets
    T rate = T(0);
    for (int i = lane; i < nu; i += 32) {
        T a = fmin(fmax(actions[w * nu + i], T(-tk.action_clip)), T(tk.action_clip));
        T p = act[i];
        prev[i] = p;
        act[i] = a;
        rate += (a - p) * (a - p);
        s.ctrl[i] = dq[m.act_qposadr[i]] + T(tk.action_scale) * a;
    }
    rate = wsum(rate);
    __syncwarp();
    int cost = 0;
    uint32_t found = 0;  // contact sensors: byte k = sensor k's most contacts in one substep
    const uint8_t* psens = tk.nsensor ? tk.pair_sensor : nullptr;
    for (int sub = 0; sub < tk.decimation; ++sub)
        cost += substep(m, d, L_, B_, w, gw, (const T*)nullptr, false, lane, psens, &found);
    if (tk.cost && lane == 0) tk.cost[w] = cost;
    if (tk.nsensor && lane < tk.nsensor) static_cast<T*>(tk.sensor)[w * tk.nsensor + lane] = T((found >> (8 * lane)) & 255u);
    if (tk.kind == 1) {
        motion_post(m, tk, L_, B_, w, ctr, cmd, act, rate, gq, gv, gw, prev, found, lane);
        if (tk.nbins > 0) adaptive_fold<T>(tk, d.nworld, lane);
        return;
    }
    if (tk.kind == 2) {
        lift_post(m, tk, L_, B_, w, ctr, cmd, act, rate, gq, gv, gw, prev, found, lane);
        if (d.geom_xpos) store_geom_frames(m, d, L_, B_, w, lane);
        return;
    }
    // rewards, terminations (pre-reset state)
    T vb[3], om[3], g[3];
    base_frame(s.qpos, s.qvel, vb, om, g);
    T c0 = cmd[0], c1 = cmd[1], c2 = cmd[2];
    T dtc = T(m.timestep) * T(tk.decimation);
    T e_xy = (c0 - vb[0]) * (c0 - vb[0]) + (c1 - vb[1]) * (c1 - vb[1]);
    T sig = T(tk.track_sigma);
    T extra[3];
    velocity_extra_terms(m, d, tk, L_, B_, w, found, extra, lane);
    // track lin vel xy, track ang vel z, lin vel z, ang vel xy, action rate, flat orientation, angular
    // momentum, joint limits, foot slip
    T terms[9] = {exp(-e_xy / sig), exp(-((c2 - om[2]) * (c2 - om[2])) / sig), vb[2] * vb[2],
                  om[0] * om[0] + om[1] * om[1], rate, g[0] * g[0] + g[1] * g[1], extra[0], extra[1], extra[2]};
    T r = T(0);
    for (int k = 0; k < 9; ++k) r += T(tk.reward_weights[k]) * terms[k] * dtc;
    bool finite = true;
    for (int i = lane; i < nq; i += 32) finite = finite && isfinite(s.qpos[i]);
    for (int i = lane; i < nv; i += 32) finite = finite && isfinite(s.qvel[i]);
    finite = __all_sync(FULL, finite);
    T h = s.qpos[2] - terrain_height(m, s.qpos[0], s.qpos[1]);
    bool term = h < T(tk.min_height) || g[2] > T(tk.max_tilt_cos) || !finite;
    int es = tk.episode_step[w] + 1;
    bool trunc = es >= tk.episode_steps;
    __syncwarp();
    if (lane == 0) {
        static_cast<T*>(tk.reward)[w] = r;
        static_cast<T*>(tk.episode_return)[w] += r;
        tk.terminated[w] = term;
        tk.truncated[w] = trunc;
        tk.episode_step[w] = es;
        if (tk.curriculum) {
            T cd = static_cast<T*>(tk.cmd_dist)[w] + sqrt(c0 * c0 + c1 * c1) * dtc;
            static_cast<T*>(tk.cmd_dist)[w] = cd;
            if (term || trunc) {  // terrain levels on the finished episode, before the reset
                T dx = s.qpos[0] - static_cast<T*>(tk.spawn_xy)[2 * w];
                T dy = s.qpos[1] - static_cast<T*>(tk.spawn_xy)[2 * w + 1];
                T walked = sqrt(dx * dx + dy * dy);
                int lv = tk.terrain_level[w];
                if (walked > T(tk.curriculum_promote) * cd) lv = lv + 1 < tk.terrain_rows ? lv + 1 : tk.terrain_rows - 1;
                else if (walked < T(tk.curriculum_demote) * cd) lv = lv > 0 ? lv - 1 : 0;
                tk.terrain_level[w] = lv;
            }
        }
    }
    __syncwarp();
    if (term || trunc) {  // masked reset (warp-uniform)
        task_reset(m, tk, L_, B_, w, ctr, lane);
        events_reset<T>(tk, w, ctr, lane);
        for (int i = lane; i < nv; i += 32) gw[i] = T(0);
        for (int i = lane; i < nu; i += 32) { act[i] = T(0); prev[i] = T(0); }
        task_resample(tk, cmd, w, ctr, lane);
        if (lane == 0) {
            tk.cmd_timer[w] = tk.cmd_resample_steps;
            tk.episode_step[w] = 0;
            static_cast<T*>(tk.episode_return)[w] = T(0);
        }
    } else {
        int tm = tk.cmd_timer[w] - 1;
        if (tm <= 0) {
            task_resample(tk, cmd, w, ctr, lane);
            tm = tk.cmd_resample_steps;
        }
        __syncwarp();
        if (lane == 0) tk.cmd_timer[w] = tm;
    }
    __syncwarp();
    events_interval(m, tk, s.qvel, w, ctr, lane);  // after resets and commands (EventManager.apply_interval)
    task_observe(m, tk, L_, B_, w, ctr, cmd, act, lane);
    if (d.geom_xpos) store_geom_frames(m, d, L_, B_, w, lane);  // sensors see the post-reset state, like obs
    for (int i = lane; i < nq; i += 32) gq[i] = s.qpos[i];
    for (int i = lane; i < nv; i += 32) gv[i] = s.qvel[i];
}

// s3_motion_bodies: one warp per clip frame -- the frame's qpos / qvel into the workspace, kinematics +
// com_pos, then the anchor's and each tracked body's state (lanes over bodies)
template <class T>
__global__ void __launch_bounds__(32 * 16) motion_table_kernel(const __grid_constant__ s3_model m, const __grid_constant__ s3_layout l,
                                                              const __grid_constant__ s3_task tk, T* __restrict__ out) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int lane = threadIdx.x & 31;
    const int64_t f = (int64_t)blockIdx.x * l.warps_per_block + (threadIdx.x >> 5);
    if (f >= tk.nframes) return;
    T* B_ = reinterpret_cast<T*>(smem_raw) + (size_t)(threadIdx.x >> 5) * l.elems_per_world;
    const s3_layout& L_ = l;
    WS<T> s = make_ws(B_, L_);
    const T* q = static_cast<const T*>(tk.motion_qpos) + f * m.nq;
    const T* v = static_cast<const T*>(tk.motion_qvel) + f * m.nv;
    for (int i = lane; i < m.nq; i += 32) s.qpos[i] = q[i];
    for (int i = lane; i < m.nv; i += 32) s.qvel[i] = v[i];
    __syncwarp();
    kinematics(m, L_, B_, lane);
    com_pos(m, L_, B_, lane, T(1));
    const int K1 = tk.ntrack + 1;
    if (lane < K1) {
        T o[S3_BODY_STATE];
        body_state(m, s, lane ? tk.track_body[lane - 1] : tk.anchor_body, o);
        for (int c = 0; c < S3_BODY_STATE; ++c) out[(f * K1 + lane) * S3_BODY_STATE + c] = o[c];
    }
}

// cost-ordered schedule: counting sort of the worlds by their last solver cost, heaviest first, so the
// warps of one block get worlds of similar Newton work (one block; order within a cost bucket is arbitrary
// and does not affect results -- every world is computed independently)
constexpr int kCostBuckets = 64;
__global__ void __launch_bounds__(1024) order_kernel(const int32_t* __restrict__ cost, int32_t* __restrict__ order,
                                                      int64_t n) {
    __shared__ int hist[kCostBuckets];
    for (int b = threadIdx.x; b < kCostBuckets; b += blockDim.x) hist[b] = 0;
    __syncthreads();
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
        const int c = cost[i];
        atomicAdd(&hist[c < 0 ? 0 : (c >= kCostBuckets ? kCostBuckets - 1 : c)], 1);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        int acc = 0;
        for (int b = kCostBuckets - 1; b >= 0; --b) {
            const int h = hist[b];
            hist[b] = acc;
            acc += h;
        }
    }
    __syncthreads();
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
        const int c = cost[i];
        order[atomicAdd(&hist[c < 0 ? 0 : (c >= kCostBuckets ? kCostBuckets - 1 : c)], 1)] = (int32_t)i;
    }
}

// ---------------------------------------------------------------- ray casting (oracle raycast)

constexpr double kHfMarch = 0.5;
constexpr int kHfBisect = 24;

template <class T> __device__ inline T ray_plane(const T* n, const T* p0, const T* o, const T* d) {
    T den = dot3(n, d);
    if (!(den < T(0))) return T(INFINITY);
    T dp[3] = {p0[0] - o[0], p0[1] - o[1], p0[2] - o[2]};
    T t = dot3(n, dp) / den;
    return t > T(0) ? t : T(INFINITY);
}

template <class T> __device__ inline T ray_sphere(const T* c, T r, const T* o, const T* d) {
    T oc[3] = {o[0] - c[0], o[1] - c[1], o[2] - c[2]};
    T b = dot3(oc, d);
    T cc = dot3(oc, oc) - r * r;
    T disc = b * b - cc;
    if (disc < T(0)) return T(INFINITY);
    T sq = sqrt(disc);
    T t = -b - sq;
    if (t > T(0)) return t;
    t = -b + sq;
    return t > T(0) ? t : T(INFINITY);
}

template <class T> __device__ inline T ray_capsule(const T* c, const T* ax, T hl, T r, const T* o, const T* d) {
    T e0[3] = {c[0] - ax[0] * hl, c[1] - ax[1] * hl, c[2] - ax[2] * hl};
    T e1[3] = {c[0] + ax[0] * hl, c[1] + ax[1] * hl, c[2] + ax[2] * hl};
    T best = fmin(ray_sphere(e0, r, o, d), ray_sphere(e1, r, o, d));
    T oc[3] = {o[0] - c[0], o[1] - c[1], o[2] - c[2]};
    T da = dot3(d, ax), oa = dot3(oc, ax);
    T dd[3] = {d[0] - ax[0] * da, d[1] - ax[1] * da, d[2] - ax[2] * da};
    T oo[3] = {oc[0] - ax[0] * oa, oc[1] - ax[1] * oa, oc[2] - ax[2] * oa};
    T a = dot3(dd, dd);
    if (a > T(1e-12)) {
        T b = dot3(oo, dd);
        T cc = dot3(oo, oo) - r * r;
        T disc = b * b - a * cc;
        if (disc >= T(0)) {
            T sq = sqrt(disc);
            T ts[2] = {(-b - sq) / a, (-b + sq) / a};
            for (int k = 0; k < 2; ++k) {
                T t = ts[k];
                if (t > T(0)) {
                    T p[3] = {oc[0] + d[0] * t, oc[1] + d[1] * t, oc[2] + d[2] * t};
                    T z = dot3(p, ax);
                    if (-hl <= z && z <= hl && t < best) best = t;
                    break;
                }
            }
        }
    }
    return best;
}

template <class T> __device__ inline T ray_box(const T* c, const T* R, const T* size, const T* o, const T* d) {
    T oc[3] = {o[0] - c[0], o[1] - c[1], o[2] - c[2]};
    T tmin = T(-INFINITY), tmax = T(INFINITY);
    for (int k = 0; k < 3; ++k) {
        T ol = R[k] * oc[0] + R[3 + k] * oc[1] + R[6 + k] * oc[2];
        T dl = R[k] * d[0] + R[3 + k] * d[1] + R[6 + k] * d[2];
        if (fabs(dl) < T(1e-12)) {
            if (ol < -size[k] || ol > size[k]) return T(INFINITY);
            continue;
        }
        T t1 = (-size[k] - ol) / dl, t2 = (size[k] - ol) / dl;
        if (t1 > t2) { T x = t1; t1 = t2; t2 = x; }
        tmin = fmax(tmin, t1);
        tmax = fmin(tmax, t2);
    }
    if (tmax < tmin || tmax <= T(0)) return T(INFINITY);
    return tmin > T(0) ? tmin : tmax;
}

template <class T> __device__ inline T hf_f(const s3_model& m, const T* p) {
    T dd, n[3];
    if (!hfield_point(m, p, T(0), dd, n)) return T(1);
    return dd;
}

template <class T> __device__ T ray_hfield(const s3_model& m, const T* o, const T* d, T tmax) {
    T step = T(kHfMarch) * T(m.hf_spacing);
    T t0 = T(0);
    if (hf_f(m, o) < T(0)) return T(INFINITY);
    int nstep = (int)ceil(tmax / step);
    for (int i = 1; i <= nstep; ++i) {
        T t1 = fmin(T(i) * step, tmax);
        T p[3] = {o[0] + d[0] * t1, o[1] + d[1] * t1, o[2] + d[2] * t1};
        if (hf_f(m, p) < T(0)) {
            T a = t0, b = t1;
            for (int k = 0; k < kHfBisect; ++k) {
                T mid = T(0.5) * (a + b);
                T q[3] = {o[0] + d[0] * mid, o[1] + d[1] * mid, o[2] + d[2] * mid};
                if (hf_f(m, q) < T(0)) b = mid;
                else a = mid;
            }
            return b;
        }
        t0 = t1;
    }
    return T(INFINITY);
}

template <class T>
__device__ void raycast1(const s3_model& m, const T* gpos, const T* gmat, const T* o, const T* d, T maxd, int excl,
                         T& dist, int& gid) {
    const T* sz = F<T>(m.geom_size);
    T best = T(INFINITY);
    int bg = -1;
    for (int g = 0; g < m.ngeom; ++g) {
        if (m.geom_bodyid[g] == excl) continue;
        int t = m.geom_type[g];
        const T* c = gpos + 3 * g;
        const T* R = gmat + 9 * g;
        T tt;
        if (t == kGeomPlane) {
            T n[3] = {R[2], R[5], R[8]};
            tt = ray_plane(n, c, o, d);
        } else if (t == kGeomHfield) {
            tt = ray_hfield(m, o, d, maxd);
        } else if (t == kGeomSphere) {
            tt = ray_sphere(c, sz[3 * g], o, d);
        } else if (t == kGeomCapsule) {
            T ax[3] = {R[2], R[5], R[8]};
            tt = ray_capsule(c, ax, sz[3 * g + 1], sz[3 * g], o, d);
        } else {
            tt = ray_box(c, R, sz + 3 * g, o, d);
        }
        if (tt < best) { best = tt; bg = g; }
    }
    if (!(best <= maxd)) { dist = T(-1); gid = -1; }
    else { dist = best; gid = bg; }
}

template <class T>
__global__ void raycast_kernel(const __grid_constant__ s3_model m, const T* __restrict__ gpos, const T* __restrict__ gmat,
                               int64_t nworld, int nray, const T* __restrict__ origin, const T* __restrict__ dir,
                               T maxd, int excl, T* __restrict__ out, int* __restrict__ gout) {
    int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= nworld * nray) return;
    int64_t w = t / nray;
    T o[3] = {origin[3 * t], origin[3 * t + 1], origin[3 * t + 2]};
    T d[3] = {dir[3 * t], dir[3 * t + 1], dir[3 * t + 2]};
    T dist;
    int g;
    raycast1(m, gpos + w * m.ngeom * 3, gmat + w * m.ngeom * 9, o, d, maxd, excl, dist, g);
    out[t] = dist;
    if (gout) gout[t] = g;
}

template <class T>
__global__ void depth_kernel(const __grid_constant__ s3_model m, const T* __restrict__ gpos, const T* __restrict__ gmat,
                             int64_t nworld, int cam, T ox, T oy, T oz, int W, int H, T tx, T ty, T maxd, int excl,
                             T* __restrict__ out, int* __restrict__ gout) {
    int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    int64_t npix = (int64_t)W * H;
    if (t >= nworld * npix) return;
    int64_t w = t / npix;
    int pix = (int)(t - w * npix);
    int i = pix / W, j = pix % W;
    const T* gp = gpos + w * m.ngeom * 3;
    const T* gm = gmat + w * m.ngeom * 9;
    const T* R = gm + 9 * cam;
    T off[3] = {ox, oy, oz}, v[3];
    mv3(R, off, v);
    T o[3] = {gp[3 * cam] + v[0], gp[3 * cam + 1] + v[1], gp[3 * cam + 2] + v[2]};
    T a = (T(2) * (T(j) + T(0.5)) / T(W) - T(1)) * tx;
    T b = (T(1) - T(2) * (T(i) + T(0.5)) / T(H)) * ty;
    T dl[3] = {T(1), -a, b};
    T rn = rsqrt_t(dot3(dl, dl));
    dl[0] *= rn; dl[1] *= rn; dl[2] *= rn;
    T d[3];
    mv3(R, dl, d);
    T dist;
    int g;
    raycast1(m, gp, gm, o, d, maxd, excl, dist, g);
    out[t] = dist;
    if (gout) gout[t] = g;
}

}  // namespace s3

// ---------------------------------------------------------------- C-ABI

namespace {
thread_local char g_err[512] = "";
int fail(int code, const char* msg) {
    snprintf(g_err, sizeof(g_err), "%s", msg);
    return code;
}
}  // namespace

extern "C" {

int s3_abi_version(void) { return S3_ABI_VERSION; }

size_t s3_sizeof(int which) {
    switch (which) {
        case 0: return sizeof(s3_model);
        case 1: return sizeof(s3_data);
        case 2: return sizeof(s3_layout);
        case 3: return sizeof(s3_task);
        default: return 0;
    }
}

const char* s3_last_error(void) { return g_err; }

int s3_plan(const s3_model* m, int32_t warps_per_block, s3_layout* out) {
    using namespace s3;
    if (!m || !out) return fail(S3_ERR_ARG, "null argument");
    if (m->nv > S3_MAX_NV || m->nbody > S3_MAX_NBODY || m->chain_stride > S3_MAX_CHAIN || m->nlimjnt > 64 ||
        m->ncon_max < 1 || m->ncon_max > S3_MAX_CON)
        return fail(S3_ERR_BOUNDS, "model exceeds kernel bounds");
    int nb = m->nbody, nv = m->nv, nj = m->njnt, ng = m->ngeom, nq = m->nq, nu = m->nu;
    int np = nv * (nv + 1) / 2;
    int sizes[O_END] = {};
    sizes[O_XPOS] = 3 * nb; sizes[O_XQUAT] = 4 * nb; sizes[O_XIPOS] = 3 * nb; sizes[O_CINERT] = 10 * nb;
    sizes[O_CRB] = S3_MAX_NV; sizes[O_CDOF] = 6 * nv; sizes[O_JANC] = 3 * nj; sizes[O_JAX] = 3 * nj; sizes[O_M] = np; sizes[O_LD] = np;
    sizes[O_QPOS] = nq; sizes[O_QVEL] = nv; sizes[O_SMOOTH] = nv; sizes[O_A0] = 0; sizes[O_A] = nv;
    sizes[O_MA] = nv; sizes[O_GRAD] = nv; sizes[O_P] = nv; sizes[O_MP] = nv; sizes[O_KVD] = nv;
    const int nc = m->ncon_max;  // per-model contact capacity (<= S3_MAX_CON)
    const int nrow = (m->nlimjnt < S3_MAX_LIM ? m->nlimjnt : S3_MAX_LIM) + 4 * nc;
    sizes[O_GPOS] = 0; sizes[O_GMAT] = 0; sizes[O_CON] = kConStride * nc;  // geom frames: computed on the fly
    int jc = 3 * nc * m->chain_stride, rne = 6 * nv + 12 * nb;
    sizes[O_JC] = jc > rne ? jc : rne; sizes[O_RAREF] = nrow; sizes[O_RD] = nrow;
    sizes[O_RJAR] = nrow; sizes[O_RJP] = nrow; sizes[O_CDOT] = 3 * nc; sizes[O_BIAS] = 0;  // bias aliases Ma
    sizes[O_FCON] = nv; sizes[O_CTRL] = nu; sizes[O_COM] = 3 * (m->nkintree > 0 ? m->nkintree : 1);
    sizes[O_CG] = (m->flags & 128) ? 2 * nv : 0;
    // the per-dof reciprocal scratch (tk, in the O_CRB slot) is used by the level-schedule variants only
    if (!(m->flags & 6)) sizes[O_CRB] = 0;
    int region = sizes[O_XIPOS] + sizes[O_CINERT] + sizes[O_JANC] + sizes[O_JAX];
    if (region < m->ntree) sizes[O_JAX] += m->ntree - region;  // room for the factorization snapshot
    // row buffers are live from build_rows to the end of Newton only: aref / D / J·a go after the factorization
    // snapshot in the xipos .. jax region and the force / J·p buffer into cdof's slot (cdof is last read by
    // build_rows; its parity copy is written before) -- each when the host slot is large enough
    auto ev = [](int x) { return (x + 1) & ~1; };
    const int nre = ev(nrow);
    const int snap_region = ev(sizes[O_XIPOS]) + ev(sizes[O_CINERT]) + ev(sizes[O_JANC]) + ev(sizes[O_JAX]);
    const bool rows_in_snap = ev(m->ntree) + 3 * nre <= snap_region;
    const bool jp_in_cdof = 6 * nv >= nrow;
    if (rows_in_snap) sizes[O_RAREF] = sizes[O_RD] = sizes[O_RJAR] = 0;
    if (jp_in_cdof) sizes[O_RJP] = 0;
    int esz = m->dtype == S3_F64 ? 8 : 4;
    const int nlim_cap = m->nlimjnt < S3_MAX_LIM ? m->nlimjnt : S3_MAX_LIM;
    int ints = nc + 2 * nlim_cap;  // con_pair, lim_dof, lim_sign
    sizes[O_INT] = (ints * 4 + esz - 1) / esz;
    int off = 0;
    for (int k = 0; k < O_END; ++k) {
        out->off[k] = off;
        off += (sizes[k] + 1) & ~1;  // keep 8-byte alignment for the float build's int region
    }
    if (rows_in_snap) {
        const int t = out->off[O_XIPOS] + ev(m->ntree);
        out->off[O_RAREF] = t;
        out->off[O_RD] = t + nre;
        out->off[O_RJAR] = t + 2 * nre;
    }
    if (jp_in_cdof) out->off[O_RJP] = out->off[O_CDOF];
    out->off[O_INT_LIMDOF] = nc;
    out->off[O_INT_LIMSIGN] = nc + nlim_cap;
    out->off[O_CDOFD] = 6 * nv;  // RNE scratch offsets relative to the Jacobian region
    out->off[O_CVEL] = 6 * nb;
    out->off[O_CACC] = 0;
    out->elems_per_world = off;
    int per = off * esz;
    int dev = 0;
    cudaGetDevice(&dev);
    int maxsm = 0;
    if (cudaDeviceGetAttribute(&maxsm, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev) != cudaSuccess || maxsm <= 0)
        maxsm = 227 * 1024;
    int wpb = warps_per_block > 0 ? warps_per_block : maxsm / per;
    if (wpb > 16) wpb = 16;
    if (wpb < 1 || wpb * per > maxsm) return fail(S3_ERR_BOUNDS, "one world does not fit in shared memory");
    out->warps_per_block = wpb;
    out->bytes_per_block = wpb * per;
    return S3_OK;
}

// The constant-memory model slot (s3::c_s3m) is one per device and shared by every model and stream.
// ModelSlot serializes its use: it holds a per-device lock from the upload through the kernel launch;
// a launch from a different stream than the previous one first waits (on the GPU) for the previous
// launch's kernels, so no running kernel ever sees the slot change under it; an identical model on the
// same stream skips the upload; uploads go through a small pinned staging ring (a pageable source could
// make the async copy synchronous), each slot reused only after its previous copy has completed.
namespace {
constexpr int kStageSlots = 8;
struct DeviceSlot {
    std::mutex mu;
    bool init = false, valid = false;
    cudaStream_t stream = nullptr;  // stream of the last launch that used the slot
    cudaEvent_t last = nullptr;     // recorded after that launch's kernels
    s3_model model;                 // contents of c_s3m as of the last upload
    s3_model* stage = nullptr;      // pinned staging ring
    cudaEvent_t stage_done[kStageSlots] = {};
    int next = 0;
};
DeviceSlot g_slots[64];

class ModelSlot {
  public:
    ModelSlot(const s3_model* m, cudaStream_t st) : st_(st) {
        int dev = 0;
        cudaGetDevice(&dev);
        s_ = &g_slots[dev & 63];
        lk_ = std::unique_lock<std::mutex>(s_->mu);
        if (!s_->init) {
            if ((err_ = cudaEventCreateWithFlags(&s_->last, cudaEventDisableTiming)) != cudaSuccess) return;
            if ((err_ = cudaMallocHost(&s_->stage, kStageSlots * sizeof(s3_model))) != cudaSuccess) return;
            for (int i = 0; i < kStageSlots; ++i)
                if ((err_ = cudaEventCreateWithFlags(&s_->stage_done[i], cudaEventDisableTiming)) != cudaSuccess) return;
            s_->init = true;
        }
        if (s_->valid && s_->stream != st && (err_ = cudaStreamWaitEvent(st, s_->last, 0)) != cudaSuccess) return;
        if (s_->valid && s_->stream == st && memcmp(&s_->model, m, sizeof(s3_model)) == 0) return;
        s_->stream = st;  // from here on the slot's latest work is on st (even if the launch fails later)
        const int k = s_->next;
        s_->next = (k + 1) % kStageSlots;
        if ((err_ = cudaEventSynchronize(s_->stage_done[k])) != cudaSuccess) return;
        s_->stage[k] = *m;
        if ((err_ = cudaMemcpyToSymbolAsync(s3::c_s3m, &s_->stage[k], sizeof(s3_model), 0, cudaMemcpyHostToDevice,
                                            st)) != cudaSuccess)
            return;
        if ((err_ = cudaEventRecord(s_->stage_done[k], st)) != cudaSuccess) return;
        s_->model = *m;
        s_->valid = true;
        err_ = cudaEventRecord(s_->last, st);
    }
    cudaError_t error() const { return err_; }
    // after the launch's kernels are enqueued: later launches from other streams wait for them
    cudaError_t done() {
        s_->stream = st_;
        return cudaEventRecord(s_->last, st_);
    }

  private:
    cudaStream_t st_;
    DeviceSlot* s_ = nullptr;
    std::unique_lock<std::mutex> lk_;
    cudaError_t err_ = cudaSuccess;
};
}  // namespace

// Launch layout: the planned (maximal) warps per block packs the most worlds per SM; when all worlds fit
// in one partial wave, smaller blocks spread them over every SM instead (G1 f32, 1024 worlds: 147 blocks of
// 7 warps instead of 64 blocks of 16, 1.62 -> 1.50 ms). Over several waves, flags bit 6 also balances the
// waves (same wave count, fewer warps per block): a win for latency-bound models (G1 f32 at 4096 worlds:
// 2 waves of 14 instead of 16, 3.03 -> 2.98 ms) and a loss for light ones (arm: +6 %), so the Python layer
// sets it by model size.
struct DeviceAttrs {
    std::once_flag once;
    int nsm = 0, smem_sm = 0;
};
static DeviceAttrs g_attrs[64];

extern "C++" s3_layout balanced_layout(const s3_layout& l, int64_t nworld, int flags) {
    int dev = 0;
    cudaGetDevice(&dev);
    DeviceAttrs& a = g_attrs[dev & 63];
    std::call_once(a.once, [&] {
        cudaDeviceGetAttribute(&a.nsm, cudaDevAttrMultiProcessorCount, dev);
        cudaDeviceGetAttribute(&a.smem_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev);
    });
    const int nsm = a.nsm, smem_sm = a.smem_sm;
    s3_layout o = l;
    const int wmax = l.warps_per_block;
    if (nsm <= 0 || wmax <= 1 || nworld <= 0) return o;
    const int per_world = l.bytes_per_block / wmax;
    int per_sm = 16 / wmax;  // 128 registers per thread: at most 16 resident warps per SM
    const int by_smem = smem_sm > 0 ? smem_sm / l.bytes_per_block : 1;
    if (by_smem < per_sm) per_sm = by_smem;
    if (per_sm < 1) per_sm = 1;
    const int64_t slots = (int64_t)nsm * per_sm;  // resident blocks
    if (nworld > slots * wmax && !(flags & 64)) return o;  // several waves: keep the maximal block
    const int64_t waves = (nworld + slots * wmax - 1) / (slots * wmax);
    int64_t w = (nworld + slots * waves - 1) / (slots * waves);
    if (w < 1) w = 1;
    if (w > wmax) w = wmax;
    o.warps_per_block = (int32_t)w;
    o.bytes_per_block = (int32_t)(w * per_world);
    return o;
}

int s3_env_step(const s3_model* m, const s3_data* d, const s3_layout* l, const s3_task* t, const void* actions,
                int32_t mode, int64_t global_step, void* stream) {
    using namespace s3;
    if (!m || !d || !l || !t) return fail(S3_ERR_ARG, "null argument");
    if (d->nworld == 0) return S3_OK;
    if (!d->qpos || !d->qvel || !d->qacc_warmstart) return fail(S3_ERR_ARG, "qpos/qvel/qacc_warmstart required");
    if (mode == 0 && !actions) return fail(S3_ERR_ARG, "actions required");
    if (t->kind != 2 && t->events && (!d->friction_scale || !d->mass_scale || !t->event_timer))
        return fail(S3_ERR_ARG, "events need friction_scale, mass_scale and event_timer");
    const int want = t->kind == 1 ? 15 + 5 * m->nu : (t->kind == 2 ? 13 + 3 * m->nu : 12 + 3 * m->nu + t->nscan);
    if (t->obs_dim != want || t->nscan > S3_MAX_RAYS || t->decimation < 1 ||
        (t->kind == 1 && (t->nframes < 2 || !t->motion_qpos || !t->motion_qvel || m->nq + m->nv > m->nv * (m->nv + 1) / 2)))
        return fail(S3_ERR_ARG, "task layout does not match the model");
    if (d->qM) return fail(S3_ERR_ARG, "parity outputs are not written by s3_env_step");
    if (t->kind == 1 && t->ntrack && (t->ntrack > S3_MAX_TRACK || !t->motion_body))
        return fail(S3_ERR_ARG, "tracked bodies need the s3_motion_bodies table");
    if (t->nsensor < 0 || t->nsensor > S3_MAX_SENSOR || (t->nsensor && (!t->pair_sensor || !t->sensor)))
        return fail(S3_ERR_ARG, "contact sensors need pair_sensor and sensor");
    if (t->kind == 1 && t->nbins && (t->nbins < 0 || t->nkernel < 1 || t->nkernel > S3_MAX_KERNEL || !t->bin_failed ||
                                     !t->bin_cum || !t->bin_fail_now || !t->bin_ticket))
        return fail(S3_ERR_ARG, "adaptive sampling needs its bin buffers and 1..S3_MAX_KERNEL kernel weights");
    if ((t->cost == nullptr) != (t->order == nullptr)) return fail(S3_ERR_ARG, "cost and order go together");
    if ((m->flags & 6) && l->off[O_CDOF] - l->off[O_CRB] < m->nv)
        return fail(S3_ERR_ARG, "layout planned without the level-schedule scratch (flags bits 1-2): re-plan");
    if (t->order && d->nworld > INT32_MAX) return fail(S3_ERR_BOUNDS, "cost-ordered schedule needs < 2^31 worlds");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    // the physics stages read the model from constant memory (s3::c_s3m): take the slot on this stream
    ModelSlot slot(m, st);
    if (slot.error() != cudaSuccess) return fail(S3_ERR_CUDA, cudaGetErrorString(slot.error()));
    const s3_layout ll = balanced_layout(*l, d->nworld, m->flags);
    int wpb = ll.warps_per_block;
    unsigned grid = (unsigned)((d->nworld + wpb - 1) / wpb);
    size_t smem = (size_t)ll.bytes_per_block;
    cudaError_t e;
    if (t->order && mode == 0) {  // sort by the previous step's solver cost (reset launches keep the order)
        order_kernel<<<1, 1024, 0, st>>>(t->cost, t->order, d->nworld);
    }
    if (m->dtype == S3_F64) {
        e = cudaFuncSetAttribute(env_kernel<double>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e == cudaSuccess)
            env_kernel<double><<<grid, 32 * wpb, smem, st>>>(*m, *d, ll, *t, static_cast<const double*>(actions), mode,
                                                              global_step);
    } else {
        e = cudaFuncSetAttribute(env_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e == cudaSuccess)
            env_kernel<float><<<grid, 32 * wpb, smem, st>>>(*m, *d, ll, *t, static_cast<const float*>(actions), mode,
                                                             global_step);
    }
    if (e == cudaSuccess) e = cudaGetLastError();
    if (e == cudaSuccess) e = slot.done();
    if (e != cudaSuccess) return fail(S3_ERR_CUDA, cudaGetErrorString(e));
    return S3_OK;
}

int s3_motion_bodies(const s3_model* m, const s3_layout* l, const s3_task* t, void* out, void* stream) {
    using namespace s3;
    if (!m || !l || !t || !out || !t->motion_qpos || !t->motion_qvel) return fail(S3_ERR_ARG, "null argument");
    if (t->nframes < 1 || t->ntrack < 1 || t->ntrack > S3_MAX_TRACK) return fail(S3_ERR_ARG, "bad frame / body count");
    for (int k = -1; k < t->ntrack; ++k) {
        const int b = k < 0 ? t->anchor_body : t->track_body[k];
        if (b < 1 || b >= m->nbody) return fail(S3_ERR_ARG, "tracked body out of range");
    }
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    ModelSlot slot(m, st);
    if (slot.error() != cudaSuccess) return fail(S3_ERR_CUDA, cudaGetErrorString(slot.error()));
    const int wpb = l->warps_per_block;
    const unsigned grid = (unsigned)((t->nframes + wpb - 1) / wpb);
    const size_t smem = (size_t)l->bytes_per_block;
    cudaError_t e;
    if (m->dtype == S3_F64) {
        e = cudaFuncSetAttribute(motion_table_kernel<double>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e == cudaSuccess) motion_table_kernel<double><<<grid, 32 * wpb, smem, st>>>(*m, *l, *t, static_cast<double*>(out));
    } else {
        e = cudaFuncSetAttribute(motion_table_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e == cudaSuccess) motion_table_kernel<float><<<grid, 32 * wpb, smem, st>>>(*m, *l, *t, static_cast<float*>(out));
    }
    if (e == cudaSuccess) e = cudaGetLastError();
    if (e == cudaSuccess) e = slot.done();
    if (e != cudaSuccess) return fail(S3_ERR_CUDA, cudaGetErrorString(e));
    return S3_OK;
}

int s3_step(const s3_model* m, const s3_data* d, const s3_layout* l, int32_t nsub, void* stream) {
    using namespace s3;
    if (!m || !d || !l || nsub < 0) return fail(S3_ERR_ARG, "null argument");
    if (d->nworld == 0 || nsub == 0) return S3_OK;
    if (!d->qpos || !d->qvel || (!d->ctrl && m->nu > 0)) return fail(S3_ERR_ARG, "qpos/qvel/ctrl required");
    if (d->qM && (!d->qLD || !d->qfrc_bias || !d->qfrc_smooth || !d->qacc_smooth || !d->qacc || !d->qfrc_constraint ||
                  !d->cdof || !d->xpos || !d->xquat || !d->com || !d->ncon || !d->ndropped || !d->nefc ||
                  !d->con_pair || !d->con_dist || !d->con_pos || !d->con_frame || !d->efc_force || !d->solver_niter))
        return fail(S3_ERR_ARG, "qM set: every parity output is required");
    if (d->geom_xpos && !d->geom_xmat) return fail(S3_ERR_ARG, "geom_xmat required with geom_xpos");
    if ((m->flags & 6) && l->off[O_CDOF] - l->off[O_CRB] < m->nv)
        return fail(S3_ERR_ARG, "layout planned without the level-schedule scratch (flags bits 1-2): re-plan");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    // the physics stages read the model from constant memory (s3::c_s3m): take the slot on this stream
    ModelSlot slot(m, st);
    if (slot.error() != cudaSuccess) return fail(S3_ERR_CUDA, cudaGetErrorString(slot.error()));
    const s3_layout ll = balanced_layout(*l, d->nworld, m->flags);
    int wpb = ll.warps_per_block;
    unsigned grid = (unsigned)((d->nworld + wpb - 1) / wpb);
    size_t smem = (size_t)ll.bytes_per_block;
    cudaError_t e;
    if (m->dtype == S3_F64) {
        e = cudaFuncSetAttribute(step_kernel<double>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e == cudaSuccess) step_kernel<double><<<grid, 32 * wpb, smem, st>>>(*m, *d, ll, nsub);
    } else {
        e = cudaFuncSetAttribute(step_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e == cudaSuccess) step_kernel<float><<<grid, 32 * wpb, smem, st>>>(*m, *d, ll, nsub);
    }
    if (e == cudaSuccess) e = cudaGetLastError();
    if (e == cudaSuccess) e = slot.done();
    if (e != cudaSuccess) return fail(S3_ERR_CUDA, cudaGetErrorString(e));
    return S3_OK;
}

int s3_raycast(const s3_model* m, const void* geom_xpos, const void* geom_xmat, int64_t nworld, int32_t nray,
               const void* origin, const void* dir, double max_dist, int32_t exclude_body, void* dist, int32_t* geom,
               void* stream) {
    using namespace s3;
    if (!m || !geom_xpos || !geom_xmat || !origin || !dir || !dist || nray < 0) return fail(S3_ERR_ARG, "null argument");
    int64_t n = nworld * nray;
    if (n == 0) return S3_OK;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    unsigned grid = (unsigned)((n + 127) / 128);
    if (m->dtype == S3_F64)
        raycast_kernel<double><<<grid, 128, 0, st>>>(*m, (const double*)geom_xpos, (const double*)geom_xmat, nworld, nray,
                                                     (const double*)origin, (const double*)dir, max_dist, exclude_body,
                                                     (double*)dist, geom);
    else
        raycast_kernel<float><<<grid, 128, 0, st>>>(*m, (const float*)geom_xpos, (const float*)geom_xmat, nworld, nray,
                                                    (const float*)origin, (const float*)dir, (float)max_dist,
                                                    exclude_body, (float*)dist, geom);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return fail(S3_ERR_CUDA, cudaGetErrorString(e));
    return S3_OK;
}

int s3_depth(const s3_model* m, const void* geom_xpos, const void* geom_xmat, int64_t nworld, int32_t cam_geom,
             const double* offset, int32_t width, int32_t height, double fovy, double max_dist, int32_t exclude_body,
             void* dist, int32_t* geom, void* stream) {
    using namespace s3;
    if (!m || !geom_xpos || !geom_xmat || !offset || !dist || width <= 0 || height <= 0)
        return fail(S3_ERR_ARG, "null argument");
    if (cam_geom < 0 || cam_geom >= m->ngeom) return fail(S3_ERR_ARG, "camera geom out of range");
    int64_t n = nworld * (int64_t)width * height;
    if (n == 0) return S3_OK;
    double ty = tan(0.5 * fovy), tx = ty * width / height;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    unsigned grid = (unsigned)((n + 127) / 128);
    if (m->dtype == S3_F64)
        depth_kernel<double><<<grid, 128, 0, st>>>(*m, (const double*)geom_xpos, (const double*)geom_xmat, nworld,
                                                   cam_geom, offset[0], offset[1], offset[2], width, height, tx, ty,
                                                   max_dist, exclude_body, (double*)dist, geom);
    else
        depth_kernel<float><<<grid, 128, 0, st>>>(*m, (const float*)geom_xpos, (const float*)geom_xmat, nworld,
                                                  cam_geom, (float)offset[0], (float)offset[1], (float)offset[2], width,
                                                  height, (float)tx, (float)ty, (float)max_dist, exclude_body,
                                                  (float*)dist, geom);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return fail(S3_ERR_CUDA, cudaGetErrorString(e));
    return S3_OK;
}

}  // extern "C"
