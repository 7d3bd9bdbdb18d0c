// ss_device.cuh -- device helpers shared by the sm_100a kernels.
//
// Numerics contract: the whole translation unit is compiled with
// --fmad=false so that every `a * b + c` rounds twice, exactly like the
// numpy float64 ufunc sequence of the reference; expression order below
// follows the reference line by line (cited per helper). Only the
// transcendental functions (sin, cos, exp, log, sqrt is exact) can differ
// from numpy by an ulp; the parity tests carry a tolerance for that.
#pragma once

#ifndef __CUDACC_RTC__
#include <cstdint>
#include <cstring>
#include <cuda_runtime.h>

#include "../../include/stridesim_b200.h"
#endif

namespace ss {

// ---------------------------------------------------------------------------
// splitmix64 counter streams (rng.py:21-41, :69-84)

constexpr uint64_t kGolden = 0x9E3779B97F4A7C15ull;
constexpr uint64_t kMixA = 0xBF58476D1CE4E5B9ull;
constexpr uint64_t kMixB = 0x94D049BB133111EBull;
constexpr uint64_t kKeySalt = 0xD6E8FEB86659FD93ull;
constexpr double kUnit = 1.1102230246251565e-16;  // 2**-53

__host__ __device__ __forceinline__ uint64_t mix(uint64_t x) {
    x = (x ^ (x >> 30)) * kMixA;
    x = (x ^ (x >> 27)) * kMixB;
    return x ^ (x >> 31);
}

// key = mix((id + 1) * SALT ^ mix(seed * GOLDEN ^ purpose_id))   (rng.py:64-65)
__host__ __device__ __forceinline__ uint64_t stream_key(uint64_t base, uint64_t gid) {
    return mix(((gid + 1ull) * kKeySalt) ^ base);
}

// word i of a draw starting at counter c   (rng.py:79)
__device__ __forceinline__ uint64_t stream_word(uint64_t key, uint64_t c, uint64_t i) {
    return mix(key + (c + i) * kGolden);
}

// (w >> 11) * 2**-53 in [0, 1)   (rng.py:102)
__device__ __forceinline__ double unit_from_word(uint64_t w) {
    return (double)(w >> 11) * kUnit;
}

// lo + u * (hi - lo)   (rng.py:111)
__device__ __forceinline__ double uniform_from_word(uint64_t w, double lo, double hi) {
    return lo + unit_from_word(w) * (hi - lo);
}

// ---------------------------------------------------------------------------
// sin/cos of the planar kinematics (sim/physics.py:31-40 calls np.sin/np.cos).
// Cody-Waite reduction by pi/2 in three FMA steps, then the fdlibm minimax
// kernels (__kernel_sin/__kernel_cos, |err| < 1 ulp, the same accuracy class
// as glibc and libdevice) with the polynomials in Estrin form: ~12 dependent
// DFMA levels instead of libdevice's ~25, and no branch, so the K joint
// angles of a substep evaluate as independent FMA chains. |x| >= 2^20, inf
// and NaN go to libdevice's sincos (kept out of line: one copy in the code).
static __device__ __noinline__ void sincos_slow(double x, double* s, double* c) { sincos(x, s, c); }

constexpr double kSincosFastMax = 1048576.0;  // 2^20

__host__ __device__ __forceinline__ unsigned lo_word(double v) {
#ifdef __CUDA_ARCH__
    return (unsigned)__double2loint(v);
#else
    unsigned long long b;
    memcpy(&b, &v, 8);
    return (unsigned)b;
#endif
}

// finite <=> exponent field not all ones: two integer ops on the high word
// instead of an FP64 subtract + compare (the FP64 pipe is the scarce one)
__host__ __device__ __forceinline__ bool finite_bits(double v) {
#ifdef __CUDA_ARCH__
    return (__double2hiint(v) & 0x7ff00000) != 0x7ff00000;
#else
    unsigned long long b;
    memcpy(&b, &v, 8);
    return ((b >> 32) & 0x7ff00000ull) != 0x7ff00000ull;
#endif
}

// v with its sign bit xor-ed by `flip` (0 or 0x80000000 on the high word)
__host__ __device__ __forceinline__ double flip_sign(double v, unsigned flip) {
#ifdef __CUDA_ARCH__
    return __hiloint2double(__double2hiint(v) ^ (int)flip, __double2loint(v));
#else
    unsigned long long b;
    memcpy(&b, &v, 8);
    b ^= (unsigned long long)flip << 32;
    memcpy(&v, &b, 8);
    return v;
#endif
}

__host__ __device__ __forceinline__ void sincos_fast(double x, double* sn, double* cs) {
    const double kMagic = 6755399441055744.0;  // 1.5 * 2^52: fma(x, 2/pi, M) - M = rint(x * 2/pi)
    const double t = fma(x, 0.63661977236758138243, kMagic);
    const double q = t - kMagic;
    double r = fma(-q, 1.5707963267948966e+00, x);
    r = fma(-q, 6.1232339957367574e-17, r);
    r = fma(-q, 8.4784276603688985e-32, r);
    const double z = r * r, z2 = z * z;
    // sin: r + r*z*(S1 + z*(S2 + z S3 + z^2 S4 + z^3 S5 + z^4 S6))
    const double sa = fma(z, -1.98412698298579493134e-04, 8.33333333332248946124e-03);
    const double sb = fma(z, -2.50507602534068634195e-08, 2.75573137070700676789e-06);
    const double sp = fma(z2, fma(z2, 1.58969099521155010221e-10, sb), sa);
    const double v = z * r;
    const double s = r == 0.0 ? r : fma(v, fma(z, sp, -1.66666666666666324348e-01), r);  // sin(-0) = -0
    // cos: w + (((1 - w) - z/2) + z^2 (C1 + z C2 + ... + z^5 C6)), w = 1 - z/2
    const double ca = fma(z, -1.38888888888741095749e-03, 4.16666666666666019037e-02);
    const double cb = fma(z, -2.75573143513906633035e-07, 2.48015872894767294178e-05);
    const double cc = fma(z, -1.13596475577881948265e-11, 2.08757232129817482790e-09);
    const double cp = fma(z2, fma(z2, cc, cb), ca);
    const double hz = 0.5 * z, w = 1.0 - hz;
    const double c = w + fma(z2, cp, (1.0 - w) - hz);
    // quadrant q mod 4 sits in the low bits of t (its ulp is 1); the result is
    // a swap plus sign-bit flips on the high words (no FP negations/selects)
    const unsigned n = lo_word(t) & 3u;
    const bool swap = n & 1u;
    *sn = flip_sign(swap ? c : s, (n & 2u) << 30);
    *cs = flip_sign(swap ? s : c, ((n + 1u) & 2u) << 30);
}

__device__ __forceinline__ void ss_sincos(double x, double* s, double* c) {
    if (fabs(x) < kSincosFastMax)
        sincos_fast(x, s, c);
    else
        sincos_slow(x, s, c);
}

// K angles: one range check for all of them, then K straight-line chains
template <int K>
__device__ __forceinline__ void ss_sincos_n(const double (&x)[K], double (&s)[K], double (&c)[K]) {
    bool fast = true;
#pragma unroll
    for (int j = 0; j < K; ++j) fast = fast && fabs(x[j]) < kSincosFastMax;
    if (fast) {
#pragma unroll
        for (int j = 0; j < K; ++j) sincos_fast(x[j], &s[j], &c[j]);
    } else {
#pragma unroll
        for (int j = 0; j < K; ++j) sincos_slow(x[j], &s[j], &c[j]);
    }
}

// std * sqrt(-2 log u1) * cos(2 pi u2); u1 in (0,1], u2 in [0,1)   (rng.py:114-119)
__device__ __forceinline__ double normal_from_words(uint64_t w1, uint64_t w2, double std_) {
    const double u1 = ((double)(w1 >> 11) + 1.0) * kUnit;
    const double u2 = (double)(w2 >> 11) * kUnit;
    const double two_pi = 6.283185307179586;  // 2.0 * np.pi, exactly as numpy forms it
    return std_ * sqrt(-2.0 * log(u1)) * cos(two_pi * u2);
}

// ---------------------------------------------------------------------------
// numpy semantics for NaN-propagating max / min / clip (numpy's _clip and
// maximum ufunc loops: a NaN in any operand propagates).

__device__ __forceinline__ bool isnan_(double x) { return x != x; }

__device__ __forceinline__ double np_maximum(double a, double b) {
    // numpy maximum: (a >= b || isnan(a)) ? a : b
    return (a >= b || isnan_(a)) ? a : b;
}
__device__ __forceinline__ double np_minimum(double a, double b) {
    return (a <= b || isnan_(a)) ? a : b;
}
__device__ __forceinline__ double np_clip(double x, double lo, double hi) {
    // numpy _NPY_CLIP = min(max(x, lo), hi) with NaN propagation from x.
    // "!(x <= lo)" is one unordered compare (true for x > lo or x NaN);
    // bounds are finite wherever the step uses clip with state-dependent x.
    const double m = !(x <= lo) ? x : lo;
    return !(m >= hi) ? m : hi;
}
// numpy maximum(0.0, x): NaN in x propagates
__device__ __forceinline__ double np_max0(double x) { return !(x <= 0.0) ? x : 0.0; }

// numpy add.reduce over a short contiguous axis: n < 8 is a sequential sum
// from 0.0; n >= 8 uses the 8-lane pairwise block (numpy pairwise_sum).
template <int NMAX>
__device__ __forceinline__ double np_sum(const double* a, int n) {
    if (n < 8) {
        double r = 0.0;
#pragma unroll
        for (int i = 0; i < (NMAX < 8 ? NMAX : 7); ++i)
            if (i < n) r += a[i];
        return r;
    }
    double r[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) r[j] = (j < NMAX) ? a[j] : 0.0;
    int i = 8;
#pragma unroll
    for (int blk = 8; blk + 8 <= NMAX; blk += 8) {
        if (blk + 8 <= n) {
#pragma unroll
            for (int j = 0; j < 8; ++j) r[j] += a[blk + j];
            i = blk + 8;
        }
    }
    double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
#pragma unroll
    for (int t = 8; t < NMAX; ++t)
        if (t >= i && t < n) res += a[t];
    return res;
}

// ---------------------------------------------------------------------------
// heightfield lookup (terrain.py:159-169)

// a / b correctly rounded, from y = RN(1/b) (loop-invariant): q = RN(a y),
// then one Markstein correction q + RN(a - b q) y (the remainder is exact
// under FMA). 3 dependent DFMA instead of DDIV's reciprocal iteration;
// checked equal to a / b on 3e8 quotients incl. random divisors
// (tests/test_div_rn_cpu.py). An overflowing quotient keeps RN(a y) (= inf).
__host__ __device__ __forceinline__ double div_rn(double a, double b, double y) {
    const double q = a * y;
    const double q1 = fma(fma(-q, b, a), y, q);
    return finite_bits(q1) ? q1 : q;
}


__device__ __forceinline__ double terrain_height(const ss_terrain& t, double x) {
    if (t.flat) return 0.0;
    const int64_t last = t.n_samples - 1;
    double pos = div_rn(finite_bits(x) ? x : 0.0, t.spacing, 1.0 / t.spacing);
    pos = np_clip(pos, 0.0, (double)last);
    int64_t idx = (int64_t)pos;
    if (idx > last - 1) idx = last - 1;
    const double frac = pos - (double)idx;
    const double s0 = __ldg(t.samples + idx);
    const double s1 = __ldg(t.samples + idx + 1);
    return s0 * (1.0 - frac) + s1 * frac;
}

// ---------------------------------------------------------------------------
// field access (sim/model.py:26-38): shared -> ptr[c]; expanded -> ptr[c*N + w]

__device__ __forceinline__ double field_at(const ss_field& f, int c, int w, int n) {
    return f.expanded ? f.ptr[(int64_t)c * n + w] : f.ptr[c];
}

}  // namespace ss
