// GPU-side cost of launching a kernel with a large __grid_constant__ parameter block.
#include <cstdio>
#include <cuda_runtime.h>
template <int BYTES> struct Blob { unsigned char b[BYTES]; };
template <int BYTES>
__global__ void k(const __grid_constant__ Blob<BYTES> p, int* out) { if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = p.b[BYTES - 1]; }
template <int BYTES>
float run(int* out, int grid) {
    Blob<BYTES> p = {};
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    for (int i = 0; i < 100; ++i) k<BYTES><<<grid, 64>>>(p, out);
    cudaEventRecord(a);
    for (int i = 0; i < 2000; ++i) k<BYTES><<<grid, 64>>>(p, out);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b); return ms * 1000.f / 2000;
}
int main() {
    int* out; cudaMalloc(&out, 64);
    printf("64 B params:    %.2f us/launch (grid 64)\n", run<64>(out, 64));
    printf("4 KB params:    %.2f us/launch\n", run<4096>(out, 64));
    printf("14 KB params:   %.2f us/launch\n", run<14336>(out, 64));
    printf("14 KB, grid 1024: %.2f us/launch\n", run<14336>(out, 1024));
    return 0;
}
