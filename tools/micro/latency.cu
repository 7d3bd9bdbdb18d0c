// Dependent-chain latency probes on B200 (one warp): DADD, DFMA, FFMA, sincos(double), IMAD.WIDE
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k_dadd(double* out, double a, int n, long long* cyc) {
    double x = a; long long t0 = clock64();
    for (int i = 0; i < n; ++i) { x = x + a; x = x + a; x = x + a; x = x + a; }
    long long t1 = clock64(); out[threadIdx.x] = x; if (threadIdx.x == 0) *cyc = t1 - t0;
}
__global__ void k_dfma(double* out, double a, int n, long long* cyc) {
    double x = a; long long t0 = clock64();
    for (int i = 0; i < n; ++i) { x = fma(x, a, a); x = fma(x, a, a); x = fma(x, a, a); x = fma(x, a, a); }
    long long t1 = clock64(); out[threadIdx.x] = x; if (threadIdx.x == 0) *cyc = t1 - t0;
}
__global__ void k_ffma(float* out, float a, int n, long long* cyc) {
    float x = a; long long t0 = clock64();
    for (int i = 0; i < n; ++i) { x = fmaf(x, a, a); x = fmaf(x, a, a); x = fmaf(x, a, a); x = fmaf(x, a, a); }
    long long t1 = clock64(); out[threadIdx.x] = x; if (threadIdx.x == 0) *cyc = t1 - t0;
}
__global__ void k_sincos(double* out, double a, int n, long long* cyc) {
    double x = a; long long t0 = clock64();
    for (int i = 0; i < n; ++i) { double s, c; sincos(x, &s, &c); x = s + c * 1e-3; }
    long long t1 = clock64(); out[threadIdx.x] = x; if (threadIdx.x == 0) *cyc = t1 - t0;
}
__global__ void k_mix(unsigned long long* out, unsigned long long a, int n, long long* cyc) {
    unsigned long long x = a; long long t0 = clock64();
    for (int i = 0; i < n; ++i) { x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull; x = (x ^ (x >> 27)) * 0x94D049BB133111EBull; }
    long long t1 = clock64(); out[threadIdx.x] = x; if (threadIdx.x == 0) *cyc = t1 - t0;
}
int main() {
    double* d; float* f; unsigned long long* u; long long* c; long long h;
    cudaMalloc(&d, 4096); cudaMalloc(&f, 4096); cudaMalloc(&u, 4096); cudaMalloc(&c, 8);
    const int n = 4096;
    k_dadd<<<1, 32>>>(d, 1e-9, n, c); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost); k_dadd<<<1, 32>>>(d, 1e-9, n, c); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("DADD dependent latency: %.2f cycles\n", h / (4.0 * n));
    k_dfma<<<1, 32>>>(d, 0.5, n, c); k_dfma<<<1, 32>>>(d, 0.5, n, c); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("DFMA dependent latency: %.2f cycles\n", h / (4.0 * n));
    k_ffma<<<1, 32>>>(f, 0.5f, n, c); k_ffma<<<1, 32>>>(f, 0.5f, n, c); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("FFMA dependent latency: %.2f cycles\n", h / (4.0 * n));
    k_sincos<<<1, 32>>>(d, 0.3, n, c); k_sincos<<<1, 32>>>(d, 0.3, n, c); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("sincos(double)+dadd+dmul chain: %.1f cycles\n", h / (1.0 * n));
    k_mix<<<1, 32>>>(u, 12345, n, c); k_mix<<<1, 32>>>(u, 12345, n, c); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("splitmix round (2 xorshift-mul64): %.1f cycles\n", h / (1.0 * n));
    return 0;
}
