// Launch latency seen between two CUDA events around one tiny kernel, after a 512 MiB L2 flush (the
// bench's protocol): a direct launch vs a one-node CUDA graph (with and without per-launch parameter
// updates), with a 16 B and a 4 KB parameter block.
//   nvcc -O2 -gencode arch=compute_100a,code=sm_100a tools/micro/launch_graph.cu -o /tmp/lg && /tmp/lg
#include <cstdio>
#include <cuda_runtime.h>

template <int S>
struct P {
    double v[S / 8];
};

template <int S>
__global__ void k(const __grid_constant__ P<S> p, double* out) {
    if (threadIdx.x == 0) out[blockIdx.x] = p.v[blockIdx.x % (S / 8)];
}

__global__ void flush_k(float* f, size_t n, float v) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) f[i] = v;
}

template <int S>
void run(float* fb, size_t fn, double* out, cudaStream_t st) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    P<S> p{};
    auto measure = [&](const char* name, auto launch) {
        float sum = 0, best = 1e9;
        const int reps = 30;
        for (int r = 0; r < reps + 3; ++r) {
            flush_k<<<1184, 256, 0, st>>>(fb, fn, (float)r);
            cudaEventRecord(a, st);
            launch(r);
            cudaEventRecord(b, st);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            if (r >= 3) {
                sum += ms;
                best = ms < best ? ms : best;
            }
        }
        printf("params %5d B  %-34s mean %6.2f us  best %6.2f us\n", S, name, sum / reps * 1e3, best * 1e3);
    };
    measure("direct launch", [&](int r) {
        p.v[0] = r;
        k<S><<<64, 64, 0, st>>>(p, out);
    });
    // one-node graph
    cudaGraph_t g;
    cudaGraphExec_t ge;
    cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal);
    k<S><<<64, 64, 0, st>>>(p, out);
    cudaStreamEndCapture(st, &g);
    cudaGraphInstantiate(&ge, g, 0);
    measure("graph launch", [&](int r) { cudaGraphLaunch(ge, st); });
    size_t nn = 1;
    cudaGraphNode_t node;
    cudaGraphGetNodes(g, &node, &nn);
    cudaKernelNodeParams kp;
    cudaGraphKernelNodeGetParams(node, &kp);
    measure("graph launch + param update", [&](int r) {
        p.v[0] = r;
        void* args[2] = {&p, &out};
        kp.kernelParams = args;
        cudaGraphExecKernelNodeSetParams(ge, node, &kp);
        cudaGraphLaunch(ge, st);
    });
    cudaGraphExecDestroy(ge);
    cudaGraphDestroy(g);
}

int main() {
    const size_t fn = 512ull * 1024 * 1024 / 4;
    float* fb;
    double* out;
    cudaMalloc(&fb, fn * 4);
    cudaMalloc(&out, 1 << 20);
    cudaStream_t st;
    cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
    run<16>(fb, fn, out, st);
    run<4096>(fb, fn, out, st);
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
