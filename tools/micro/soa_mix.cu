// HBM ceiling of the fused step's access pattern: every thread (one world) reads R float64 components
// from R SoA streams (ptr[c * N + w]) and writes W components to W other streams, no compute; one
// 262,144-world launch, L2 flushed before each timed launch (as bench.py). Compared with a plain
// copy (the MEASURED_PEAKS.json figure) and read-only / write-only mixes.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/micro/soa_mix.cu -o /tmp/soa_mix && /tmp/soa_mix
#include <cstdio>
#include <cuda_runtime.h>

__global__ void mix_k(const double* __restrict__ in, double* __restrict__ out, int N, int R, int W, int block_loads) {
    const int w = blockIdx.x * blockDim.x + threadIdx.x;
    if (w >= N) return;
    double acc = 0.0;
    // the step's entry: every read issued up front (block_loads at a time), then the writes
    for (int c0 = 0; c0 < R; c0 += block_loads) {
        double v[16];
#pragma unroll
        for (int k = 0; k < 16; ++k) v[k] = (k < block_loads && c0 + k < R) ? in[(size_t)(c0 + k) * N + w] : 0.0;
#pragma unroll
        for (int k = 0; k < 16; ++k) acc += v[k];
    }
    for (int c = 0; c < W; ++c) out[(size_t)c * N + w] = acc + c;
}

__global__ void copy_k(const double* __restrict__ in, double* __restrict__ out, size_t n) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
        out[i] = in[i];
}

__global__ void flush_k(float* f, size_t n, float v) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) f[i] = v;
}

int main() {
    const int N = 262144;
    const int Rmax = 280, Wmax = 180;
    double *in, *out;
    float* fb;
    const size_t fn = 512ull * 1024 * 1024 / 4;
    cudaMalloc(&in, (size_t)Rmax * N * 8);
    cudaMalloc(&out, (size_t)Wmax * N * 8);
    cudaMalloc(&fb, fn * 4);
    cudaMemset(in, 0, (size_t)Rmax * N * 8);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    auto timeit = [&](auto launch, double bytes, const char* name) {
        float best = 1e9, sum = 0;
        const int reps = 10;
        for (int r = 0; r < reps + 2; ++r) {
            flush_k<<<1184, 256>>>(fb, fn, (float)r);
            cudaEventRecord(a);
            launch();
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            if (r >= 2) {
                sum += ms;
                best = ms < best ? ms : best;
            }
        }
        const float mean = sum / reps;
        printf("%-48s %8.1f us  %7.0f GB/s (best %7.0f)\n", name, mean * 1e3, bytes / (mean * 1e-3) / 1e9,
               bytes / (best * 1e-3) / 1e9);
    };
    // a copy of the same volume as the step's (2197 B per world)
    const size_t cn = (size_t)N * 2197 / 16;
    timeit([&] { copy_k<<<1184, 256>>>(in, out, cn); }, 2.0 * cn * 8, "copy (read + write, 50/50)");
    struct Mix { int r, w; const char* name; };
    const Mix mixes[] = {{100, 175, "step mix: 100 reads + 175 writes per world"},
                         {137, 137, "same bytes, 50/50"},
                         {275, 0, "275 reads"},
                         {0, 175, "175 writes"},
                         {100, 0, "100 reads"}};
    for (const Mix& m : mixes) {
        if (m.r > Rmax || m.w > Wmax) continue;
        for (int bl : {4, 16}) {
            char name[128];
            snprintf(name, sizeof name, "%s (loads in flight %d)", m.name, bl);
            timeit([&] { mix_k<<<(N + 63) / 64, 64>>>(in, out, N, m.r, m.w, bl); }, (double)N * 8 * (m.r + m.w), name);
        }
    }
    cudaError_t e = cudaGetLastError();
    printf("%s\n", cudaGetErrorString(e));
    return 0;
}
