// ss_aux.cu -- the small kernels around the fused step: stream draws for
// user code (StreamPack.uniform/normal, rng.py:86-119), batched forward
// kinematics (fk_batch_trig, sim/physics.py:22-57), heightfield queries
// (terrain.py:159-169), field randomization for startup / explicit calls
// (randomize_field, managers/event.py:19-52) and the pure torque laws
// (actuators.py:104-117). All are one thread per world (or per element).
#include <cstdio>

#include "ss_device.cuh"

namespace ss {
constexpr int kAuxBlock = 128;
}  // namespace ss

using namespace ss;

void ss_set_error(const char* what, const char* msg);  // ss_step.cu

static int aux_fail(const char* what, cudaError_t e) {
    ss_set_error(what, cudaGetErrorString(e));
    return -1;
}

// ---------------------------------------------------------------------------
// StreamPack draws

__global__ void __launch_bounds__(kAuxBlock) rng_draw_kernel(const __grid_constant__ ss_rng_draw_args a,
                                                              int n_rows) {
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= n_rows) return;
    const int64_t w = a.sel ? a.sel[r] : r;
    const uint64_t key = stream_key(a.base, (uint64_t)(a.world_id_offset + w));
    const uint64_t c = a.counter[w];
    const int dim = a.dim;
    if (a.kind == 0) {
        for (int k = 0; k < dim; ++k) {
            double lo = a.lo, hi = a.hi;
            if (a.lohi_mode == 1) {
                lo = a.lo_arr[r];
                hi = a.hi_arr[r];
            } else if (a.lohi_mode == 2) {
                lo = a.lo_arr[(int64_t)r * dim + k];
                hi = a.hi_arr[(int64_t)r * dim + k];
            }
            a.out[(int64_t)r * dim + k] = uniform_from_word(stream_word(key, c, k), lo, hi);
        }
        a.counter[w] = c + (uint64_t)dim;
    } else {
        for (int k = 0; k < dim; ++k)
            a.out[(int64_t)r * dim + k] = normal_from_words(stream_word(key, c, k), stream_word(key, c, dim + k), a.lo);
        a.counter[w] = c + (uint64_t)(2 * dim);
    }
}

extern "C" int ss_rng_draw(const ss_rng_draw_args* a, void* stream) {
    const int n = a->n_sel;
    if (n <= 0 || a->dim <= 0) return 0;
    rng_draw_kernel<<<(n + kAuxBlock - 1) / kAuxBlock, kAuxBlock, 0, (cudaStream_t)stream>>>(*a, n);
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? 0 : aux_fail("ss_rng_draw", e);
}

// ---------------------------------------------------------------------------
// forward kinematics: thetas (N,K), attach (N,K,2), tips (N,K,2) row-major

__global__ void __launch_bounds__(kAuxBlock) fk_kernel(const __grid_constant__ ss_model m, const double* q,
                                                        double* thetas, double* attach, double* tips, int n) {
    const int w = blockIdx.x * blockDim.x + threadIdx.x;
    if (w >= n) return;
    const int K = m.n_joints;
    const int nq = 3 + K;
    const double* qr = q + (int64_t)w * nq;  // row-major (N, nq) input
    double th[SS_MAX_JOINTS], st[SS_MAX_JOINTS], ct[SS_MAX_JOINTS], ax[SS_MAX_JOINTS], az[SS_MAX_JOINTS];
    double sp, cp;
    ss_sincos(qr[2], &sp, &cp);
    for (int j = 0; j < K; ++j) {
        const int p = m.parent[j];
        th[j] = (p == -1 ? qr[2] : th[p]) + qr[3 + j];
        ss_sincos(th[j], &st[j], &ct[j]);
    }
    for (int j = 0; j < K; ++j) {
        const int p = m.parent[j];
        double sn = sp, c = cp, px = qr[0], pz = qr[1];
        if (p != -1) {
            sn = st[p];
            c = ct[p];
            px = ax[p];
            pz = az[p];
        }
        const double ox = m.attach_x[j], oz = m.attach_z[j];
        ax[j] = px + (c * ox - sn * oz);
        az[j] = pz + (sn * ox + c * oz);
        const int64_t o = (int64_t)w * K + j;
        if (thetas) thetas[o] = th[j];
        if (attach) {
            attach[2 * o] = ax[j];
            attach[2 * o + 1] = az[j];
        }
        if (tips) {
            tips[2 * o] = ax[j] + m.link_len[j] * st[j];
            tips[2 * o + 1] = az[j] - m.link_len[j] * ct[j];
        }
    }
}

extern "C" int ss_fk(const ss_env_desc* desc, const double* q, double* thetas, double* attach, double* tips,
                     int32_t n, void* stream) {
    if (n <= 0) return 0;
    fk_kernel<<<(n + kAuxBlock - 1) / kAuxBlock, kAuxBlock, 0, (cudaStream_t)stream>>>(desc->model, q, thetas,
                                                                                        attach, tips, n);
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? 0 : aux_fail("ss_fk", e);
}

// ---------------------------------------------------------------------------
// heightfield queries (always the interpolating lookup, like Heightfield.heights)

__global__ void heights_kernel(const __grid_constant__ ss_terrain t, const double* x, double* out, int64_t n) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    ss_terrain tt = t;
    tt.flat = 0;
    out[i] = terrain_height(tt, x[i]);
}

extern "C" int ss_heights(const ss_terrain* terrain, const double* x, double* out, int64_t n, void* stream) {
    if (n <= 0) return 0;
    heights_kernel<<<(unsigned)((n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(*terrain, x, out, n);
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? 0 : aux_fail("ss_heights", e);
}

// ---------------------------------------------------------------------------
// randomize_field for explicit world ids (startup events, direct calls)

__global__ void __launch_bounds__(kAuxBlock) randomize_kernel(const __grid_constant__ ss_env_desc d, int field,
                                                              int dist, double r0, double r1, int op, int slot,
                                                              const int64_t* sel, int n_sel) {
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= n_sel) return;
    const int w = sel ? (int)sel[r] : r;
    const ss_field& f = d.field[field];
    const int N = d.n_worlds;
    const uint64_t key = stream_key(d.rng.base[slot], (uint64_t)(d.rng.world_id_offset + w));
    const uint64_t c = d.rng.counter[slot][w];
    for (int k = 0; k < f.size; ++k) {
        double draw;
        if (dist == SS_DIST_UNIFORM) draw = uniform_from_word(stream_word(key, c, k), r0, r1);
        else draw = r0 + normal_from_words(stream_word(key, c, k), stream_word(key, c, f.size + k), r1);
        double v = draw;
        if (op == SS_OP_SCALE) v = f.base[k] * draw;
        else if (op == SS_OP_ADD) v = f.base[k] + draw;
        f.ptr[(int64_t)k * N + w] = v;
    }
    d.rng.counter[slot][w] = c + (uint64_t)(dist == SS_DIST_UNIFORM ? f.size : 2 * f.size);
}

extern "C" int ss_randomize(const ss_env_desc* desc, int32_t field, int32_t distribution, double r0, double r1,
                            int32_t operation, int32_t slot, const int64_t* sel, int32_t n_sel, void* stream) {
    if (n_sel <= 0) return 0;
    if (!desc->field[field].expanded) {
        ss_set_error("ss_randomize", "field must be expanded before randomization");
        return -5;
    }
    randomize_kernel<<<(n_sel + kAuxBlock - 1) / kAuxBlock, kAuxBlock, 0, (cudaStream_t)stream>>>(
        *desc, field, distribution, r0, r1, operation, slot, sel, n_sel);
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? 0 : aux_fail("ss_randomize", e);
}

// ---------------------------------------------------------------------------
// pure torque laws, elementwise (kp/kd per element)

__global__ void actuator_eval_kernel(int kind, const double* kp, const double* kd, double effort, double sat,
                                     double vlim, const double* q_des, const double* q, const double* qd,
                                     double* out, int64_t n) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    double tau = kp[i] * (q_des[i] - q[i]) + kd[i] * (0.0 - qd[i]);
    if (kind == SS_ACT_PD) {
        tau = np_clip(tau, -effort, effort);
    } else {
        const double hi = np_clip(sat * (1.0 - qd[i] / vlim), 0.0, effort);
        const double lo = np_clip(sat * (-1.0 - qd[i] / vlim), -effort, 0.0);
        tau = np_clip(tau, lo, hi);
    }
    out[i] = tau;
}

extern "C" int ss_actuator_eval(int32_t kind, const double* kp, const double* kd, double effort, double saturation,
                                double vel_limit, const double* q_des, const double* q, const double* qd,
                                double* out, int64_t n, void* stream) {
    if (n <= 0) return 0;
    actuator_eval_kernel<<<(unsigned)((n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
        kind, kp, kd, effort, saturation, vel_limit, q_des, q, qd, out, n);
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? 0 : aux_fail("ss_actuator_eval", e);
}

// ---------------------------------------------------------------------------
// metrics.build_record's reductions (metrics.py:31-45) for one rank, packed
// into one vector for the single per-log-interval all-reduce.
// Value layout inside a block: [reward, ep_sums[0..T), nonfinite, hist[0..R)];
// the integer trigger counts are copied by the last block.

constexpr int kStatsBlock = 256;

__global__ void __launch_bounds__(kStatsBlock) stats_pack_kernel(const __grid_constant__ ss_stats_args a) {
    const int N = a.n_worlds, T = a.n_rewards, R = a.n_rows;
    const int V = 2 + T + R;  // float-summed values per block
    __shared__ double red[kStatsBlock / 32][SS_STATS_MAXV];
    __shared__ bool last;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int v = 0; v < V; ++v) {
        // each thread sums its strided worlds in index order, then a fixed
        // shuffle tree per warp and a fixed warp order per block
        double acc = 0.0;
        for (int w = blockIdx.x * blockDim.x + threadIdx.x; w < N; w += gridDim.x * blockDim.x) {
            double x;
            if (v == 0) x = a.reward[w];
            else if (v <= T) x = a.ep_sums[(int64_t)(v - 1) * N + w];
            else if (v == T + 1) x = a.nonfinite[w] ? 1.0 : 0.0;
            else x = (a.terrain_rows[w] == (int64_t)(v - T - 2)) ? 1.0 : 0.0;
            acc += x;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) acc += __shfl_down_sync(0xffffffffu, acc, o);
        if (lane == 0) red[warp][v] = acc;
    }
    __syncthreads();
    for (int v = threadIdx.x; v < V; v += blockDim.x) {
        double acc = 0.0;
        for (int k = 0; k < kStatsBlock / 32; ++k) acc += red[k][v];
        a.partials[(int64_t)blockIdx.x * SS_STATS_MAXV + v] = acc;
    }
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) last = atomicInc(a.ticket, gridDim.x - 1) == gridDim.x - 1;  // wraps to 0
    __syncthreads();
    if (!last) return;
    __threadfence();
    const int C = a.n_counts;
    for (int v = threadIdx.x; v < V; v += blockDim.x) {
        double acc = 0.0;
        for (int b = 0; b < (int)gridDim.x; ++b) acc += ((volatile double*)a.partials)[(int64_t)b * SS_STATS_MAXV + v];
        int o;
        if (v == 0) o = 1;                    // sum(reward)
        else if (v <= T) o = 1 + v;           // sum(ep_sums[v-1])
        else if (v == T + 1) o = 2 + T + C + R;  // sum(nonfinite)
        else o = 2 + T + C + (v - T - 2);     // histogram bin
        a.out[o] = acc;
    }
    for (int c = threadIdx.x; c < C; c += blockDim.x) a.out[2 + T + c] = (double)a.trigger_counts[c];
    if (threadIdx.x == 0) a.out[0] = (double)N;
}

extern "C" int ss_stats_pack(const ss_stats_args* a, void* stream) {
    if (!a || a->n_worlds <= 0) return 0;
    if (2 + a->n_rewards + a->n_rows > SS_STATS_MAXV) {
        ss_set_error("ss_stats_pack", "too many statistics for SS_STATS_MAXV");
        return -5;
    }
    int grid = (a->n_worlds + kStatsBlock - 1) / kStatsBlock;
    if (grid > SS_STATS_GRID) grid = SS_STATS_GRID;
    stats_pack_kernel<<<grid, kStatsBlock, 0, (cudaStream_t)stream>>>(*a);
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? 0 : aux_fail("ss_stats_pack", e);
}
