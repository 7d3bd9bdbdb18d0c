// Launch cost vs kernel-parameter size, warm and after an L2 flush.
//   nvcc -O2 -gencode arch=compute_100a,code=sm_100a tools/micro/launch_param.cu -o /tmp/lp && /tmp/lp
#include <chrono>
#include <cstdio>
#include <cuda_runtime.h>

template <int S>
struct P {
    double v[S / 8];
};

template <int S>
__global__ void k_param(const __grid_constant__ P<S> p, double* out) {
    if (threadIdx.x == 0) out[blockIdx.x] = p.v[(blockIdx.x * 7) % (S / 8)];
}

__constant__ double c_bank[13312 / 8];

__global__ void k_const(int idx, double* out) {
    if (threadIdx.x == 0) out[blockIdx.x] = c_bank[(blockIdx.x * 7 + idx) % (13312 / 8)];
}

__global__ void flush_k(float* f, size_t n, float v) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) f[i] = v;
}

template <class L>
float time_it(L launch, bool flush, float* fbuf, size_t fn) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    float tot = 0;
    const int K = 200;
    for (int i = 0; i < K + 10; ++i) {
        if (flush) flush_k<<<1184, 512>>>(fbuf, fn, (float)i);
        cudaEventRecord(a);
        launch();
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        if (i >= 10) tot += ms;
    }
    return 1e3f * tot / K;
}

int main() {
    double* out;
    cudaMalloc(&out, 1 << 20);
    float* fbuf;
    const size_t fn = 512ull * 1024 * 1024 / 4;
    cudaMalloc(&fbuf, fn * 4);
    P<16> p16{};
    P<1024> p1k{};
    P<4096> p4k{};
    P<13312> p13k{};
    P<32000> p32k{};
    // host-side cost of one launch (queue depth kept low by periodic syncs)
    auto host_cost = [&](auto launch) {
        cudaDeviceSynchronize();
        double tot = 0;
        for (int r = 0; r < 20; ++r) {
            auto t0 = std::chrono::steady_clock::now();
            for (int i = 0; i < 100; ++i) launch();
            auto t1 = std::chrono::steady_clock::now();
            cudaDeviceSynchronize();
            tot += std::chrono::duration<double, std::micro>(t1 - t0).count();
        }
        return tot / 2000;
    };
    printf("host launch cost: 16 B %.2f us, 1 KB %.2f us, 4 KB %.2f us, 13 KB %.2f us, 32 KB %.2f us\n",
           host_cost([&] { k_param<16><<<64, 64>>>(p16, out); }), host_cost([&] { k_param<1024><<<64, 64>>>(p1k, out); }),
           host_cost([&] { k_param<4096><<<64, 64>>>(p4k, out); }), host_cost([&] { k_param<13312><<<64, 64>>>(p13k, out); }),
           host_cost([&] { k_param<32000><<<64, 64>>>(p32k, out); }));
    for (int fl = 0; fl < 2; ++fl) {
        printf("%s\n", fl ? "after L2 flush:" : "warm:");
        printf("  param 16 B   : %6.2f us\n", time_it([&] { k_param<16><<<64, 64>>>(p16, out); }, fl, fbuf, fn));
        printf("  param 1 KB   : %6.2f us\n", time_it([&] { k_param<1024><<<64, 64>>>(p1k, out); }, fl, fbuf, fn));
        printf("  param 4 KB   : %6.2f us\n", time_it([&] { k_param<4096><<<64, 64>>>(p4k, out); }, fl, fbuf, fn));
        printf("  param 13 KB  : %6.2f us\n", time_it([&] { k_param<13312><<<64, 64>>>(p13k, out); }, fl, fbuf, fn));
        printf("  param 32 KB  : %6.2f us\n", time_it([&] { k_param<32000><<<64, 64>>>(p32k, out); }, fl, fbuf, fn));
        printf("  __constant__ : %6.2f us\n", time_it([&] { k_const<<<64, 64>>>(1, out); }, fl, fbuf, fn));
    }
    return 0;
}
