// ss_step.cu -- host side of the fused step: the ahead-of-time generic
// instantiation (RuntimeCfg) plus the per-env NVRTC specialization.
//
// The generic kernel is instantiated for three joint/foot bounds and reads
// every term table from the descriptor. ss_jit_compile/ss_jit_load build
// and load a kernel whose tables are compile-time constants (see
// ss_cfg.cuh); ss_env_step_jit launches it. Both execute the same source,
// ss_kernel.cuh, so their results are bitwise identical.
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include <cuda_runtime.h>
#include <nvrtc.h>

#include "../../include/stridesim_b200.h"
#include "ss_kernel.cuh"

namespace ss {

template <int KM, int FM>
__global__ void __launch_bounds__(kBlock) step_kernel(const __grid_constant__ ss_env_desc d,
                                                      const __grid_constant__ ss_uniforms u) {
    step_body<RuntimeCfg, KM, FM>(d, u);
}

static thread_local char g_err[4096] = "";

}  // namespace ss

using namespace ss;

void ss_set_error(const char* what, const char* msg) { snprintf(g_err, sizeof(g_err), "%s: %s", what, msg); }

extern "C" const char* ss_last_error(void) { return g_err; }

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
        case 3: return sizeof(ss_rt_state);
        case 4: return sizeof(ss_launch);
        case 5: return sizeof(ss_stats_args);
        default: return 0;
    }
}

static int check_desc(const ss_env_desc* desc, const ss_uniforms* u, const char* who) {
    if (!desc || !u) {
        snprintf(g_err, sizeof(g_err), "%s: null descriptor", who);
        return -2;
    }
    if (desc->abi_version != SS_ABI_VERSION) {
        snprintf(g_err, sizeof(g_err), "%s: abi version %d != %d", who, desc->abi_version, SS_ABI_VERSION);
        return -3;
    }
    if (desc->model.n_joints > SS_MAX_JOINTS || desc->model.n_feet > SS_MAX_FEET || desc->hist_len > SS_MAX_HIST ||
        desc->action_dim > SS_MAX_ACTION || desc->n_terms > 31) {
        snprintf(g_err, sizeof(g_err), "%s: model exceeds compiled limits", who);
        return -4;
    }
    if ((u->stages & SS_ST_ACTION) && u->policy_slot < 0 && !u->actions) {
        snprintf(g_err, sizeof(g_err), "%s: ACTION stage without actions or a policy stream", who);
        return -5;
    }
    if (u->policy_slot >= SS_MAX_SLOTS || ((u->stages & SS_ST_ACTION) && u->policy_slot >= 0 &&
                                           !desc->rng.counter[u->policy_slot])) {
        snprintf(g_err, sizeof(g_err), "%s: policy stream slot %d not allocated", who, u->policy_slot);
        return -6;
    }
    return 0;
}

extern "C" int ss_env_step(const ss_env_desc* desc, const ss_uniforms* u, void* stream) {
    if (int rc = check_desc(desc, u, "ss_env_step")) return rc;
    if (desc->n_worlds <= 0) return 0;
    const int K = desc->model.n_joints, F = desc->model.n_feet;
    cudaStream_t s = (cudaStream_t)stream;
    cudaError_t e;
    if (K <= 4 && F <= 2) e = launch_step<4, 2>(*desc, *u, s);
    else if (K <= 12 && F <= 4) e = launch_step<12, 4>(*desc, *u, s);
    else e = launch_step<16, 8>(*desc, *u, s);
    if (e != cudaSuccess) return ss_fail("ss_env_step launch", e);
    return 0;
}

// ---------------------------------------------------------------------------
// per-env specialization (NVRTC)

struct JitModule {
    cudaLibrary_t lib;
    cudaKernel_t kernel;
    int block;
    int min_grid;  // experiment knob (SS_MIN_GRID): pad the grid with empty blocks
    int64_t desc_bytes;  // size of the kernel's descriptor parameter (packed when < sizeof(ss_env_desc))
    int smem = 0;        // dynamic shared memory per block (staging buffers beyond the 48 KB static limit)
};

// Compile `src` (with named headers) for sm_100a. Returns the cubin through
// a two-call protocol: with out == NULL, *size receives the byte count.
extern "C" int ss_jit_compile(const char* src, const char* name, int n_headers, const char* const* header_src,
                              const char* const* header_names, int n_opts, const char* const* opts, void* out,
                              size_t* size, char* log, size_t log_size) {
    nvrtcProgram prog;
    nvrtcResult r = nvrtcCreateProgram(&prog, src, name ? name : "ss_step_jit.cu", n_headers, header_src,
                                       header_names);
    if (r != NVRTC_SUCCESS) {
        ss_set_error("nvrtcCreateProgram", nvrtcGetErrorString(r));
        return -10;
    }
    r = nvrtcCompileProgram(prog, n_opts, opts);
    size_t lsz = 0;
    nvrtcGetProgramLogSize(prog, &lsz);
    if (log && log_size) {
        std::vector<char> buf(lsz + 1, 0);
        nvrtcGetProgramLog(prog, buf.data());
        snprintf(log, log_size, "%s", buf.data());
    }
    if (r != NVRTC_SUCCESS) {
        ss_set_error("nvrtcCompileProgram", nvrtcGetErrorString(r));
        nvrtcDestroyProgram(&prog);
        return -11;
    }
    size_t n = 0;
    nvrtcGetCUBINSize(prog, &n);
    if (out && *size >= n) nvrtcGetCUBIN(prog, (char*)out);
    *size = n;
    nvrtcDestroyProgram(&prog);
    return 0;
}

extern "C" int ss_jit_load(const void* cubin, size_t size, const char* kernel_name, int block, void** handle) {
    (void)size;
    JitModule* m = new JitModule();
    m->block = block > 0 ? block : kBlock;
    m->desc_bytes = (int64_t)sizeof(ss_env_desc);
    const char* mg = getenv("SS_MIN_GRID");
    m->min_grid = mg ? atoi(mg) : 0;
    cudaError_t e = cudaLibraryLoadData(&m->lib, cubin, nullptr, nullptr, 0, nullptr, nullptr, 0);
    if (e != cudaSuccess) {
        delete m;
        return ss_fail("cudaLibraryLoadData", e);
    }
    e = cudaLibraryGetKernel(&m->kernel, m->lib, kernel_name);
    if (e != cudaSuccess) {
        cudaLibraryUnload(m->lib);
        delete m;
        return ss_fail("cudaLibraryGetKernel", e);
    }
    *handle = m;
    return 0;
}

extern "C" int ss_jit_unload(void* handle) {
    JitModule* m = (JitModule*)handle;
    if (!m) return 0;
    cudaLibraryUnload(m->lib);
    delete m;
    return 0;
}

static int jit_launch(JitModule* m, const ss_env_desc* desc, const void* param, const ss_uniforms* u, void* stream) {
    void* args[2] = {(void*)param, (void*)u};
    int blocks = (desc->n_worlds + m->block - 1) / m->block;
    if (blocks < m->min_grid) blocks = m->min_grid;
    const dim3 grid(blocks);
    cudaError_t e = cudaLaunchKernel((const void*)m->kernel, grid, dim3(m->block), args, (size_t)m->smem,
                                     (cudaStream_t)stream);
    if (e != cudaSuccess) return ss_fail("ss_env_step_jit launch", e);
    return 0;
}

extern "C" int ss_env_step_jit(void* handle, const ss_env_desc* desc, const ss_uniforms* u, void* stream) {
    if (int rc = check_desc(desc, u, "ss_env_step_jit")) return rc;
    if (desc->n_worlds <= 0) return 0;
    JitModule* m = (JitModule*)handle;
    if (m->desc_bytes != (int64_t)sizeof(ss_env_desc)) {
        ss_set_error("ss_env_step_jit", "module takes a packed descriptor: use ss_env_step_jit_packed");
        return -13;
    }
    return jit_launch(m, desc, desc, u, stream);
}

extern "C" int ss_jit_set_desc_bytes(void* handle, int64_t bytes) {
    JitModule* m = (JitModule*)handle;
    if (!m || bytes <= 0 || bytes > (int64_t)sizeof(ss_env_desc)) {
        ss_set_error("ss_jit_set_desc_bytes", "bad handle or size");
        return -14;
    }
    m->desc_bytes = bytes;
    return 0;
}

extern "C" int ss_jit_set_smem(void* handle, int32_t bytes) {
    JitModule* m = (JitModule*)handle;
    if (!m || bytes < 0) {
        ss_set_error("ss_jit_set_smem", "bad handle or size");
        return -14;
    }
    if (bytes > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute((const void*)m->kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
        if (e != cudaSuccess) return ss_fail("ss_jit_set_smem", e);
    }
    m->smem = bytes;
    return 0;
}

extern "C" int ss_env_step_jit_packed(void* handle, const ss_env_desc* desc, const void* packed, int64_t packed_bytes,
                                      const ss_uniforms* u, void* stream) {
    if (int rc = check_desc(desc, u, "ss_env_step_jit_packed")) return rc;
    if (desc->n_worlds <= 0) return 0;
    JitModule* m = (JitModule*)handle;
    if (!packed || packed_bytes != m->desc_bytes) {
        ss_set_error("ss_env_step_jit_packed", "packed descriptor size does not match the module");
        return -15;
    }
    return jit_launch(m, desc, packed, u, stream);
}
