// ss_runtime.cu -- native per-step bookkeeping of ManagerBasedRlEnv.step.
//
// Everything the fused kernel needs besides the descriptor is a pure
// function of counters the host owns (env.py:219-259): global_step,
// sim_step, the capture-ring cursor (capture.py:53-59), the contact sensor's
// once-per-sim_step guard (sensors.py:92-94), actuator delay-ring heads
// (actuators.py:208-211), observation delay/history heads
// (managers/observation.py:115-129) and the reward weights. ss_rt_launch
// derives the ss_uniforms block from them, launches, and advances them, so
// a control step costs the host one C call and no device round trip.
// Nonfinite detection (env.py:240-241) is deferred: each TERM launch gets a
// slot with a zero-copy flag in pinned host memory and a CUDA event;
// ss_rt_poll retires completed slots and reports the flagged ones.
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include <cuda_runtime.h>

#include "../../include/stridesim_b200.h"

void ss_set_error(const char* what, const char* msg);  // ss_step.cu

extern "C" int ss_rt_poll(ss_rt_state* st, int32_t keep, int32_t* out_slots, int32_t max_out);

extern "C" int ss_rt_launch(const ss_env_desc* d, ss_rt_state* st, const ss_launch* l, void* jit, void* stream) {
    st->nf_ready_n = 0;
    if ((l->stages & SS_ST_TERM) && l->poll_keep >= 0) {
        const int n = ss_rt_poll(st, l->poll_keep, st->nf_ready, SS_RT_SLOTS);
        if (n < 0) return n;
        st->nf_ready_n = n;
    }
    ss_uniforms u;
    memset(&u, 0, sizeof(u));
    const uint32_t stages = l->stages;
    const int nsub = l->nsub;
    u.stages = stages;
    u.nsub = nsub;
    u.flags = l->flags;
    u.global_step = st->global_step;
    u.sim_step = st->sim_step;
    if (stages & SS_ST_PUSH) {
        u.capture_slot0 = (int32_t)(st->cap_pushes % st->cap_phys);
        for (int i = 0; i < nsub; ++i) st->cap_sim_steps[(st->cap_pushes + i) % st->cap_phys] = st->sim_step + i;
        st->cap_pushes += nsub;
        st->cap_count = st->cap_count + nsub < st->cap_capacity ? st->cap_count + nsub : st->cap_capacity;
    }
    if (stages & SS_ST_SENSOR) {
        uint32_t mask = 0;
        const int phys = (stages & SS_ST_PHYS) ? 1 : 0;
        for (int s = 0; s < nsub; ++s) {
            const int64_t step = st->sim_step + s + phys;
            if (step != st->sensor_last_update) {
                mask |= 1u << s;
                st->sensor_last_update = step;
            }
        }
        u.sensor_mask = mask;
    }
    if (stages & SS_ST_APPLY) {
        for (int a = 0; a < st->n_act; ++a) {
            u.act_head0[a] = st->act_head[a];
            if (st->act_cap[a] > 0) st->act_head[a] = (st->act_head[a] + nsub) % st->act_cap[a];
        }
    }
    u.groups_mask = l->groups_mask;
    u.any_pending = st->any_pending;
    if (stages & SS_ST_OBS) {
        for (int t = 0; t < st->n_obs; ++t) {
            if ((l->groups_mask >> st->obs_group[t]) & 1u) {
                st->obs_delay_head[t] = (st->obs_delay_head[t] + 1) % st->obs_delay_len[t];
                st->obs_hist_head[t] = (st->obs_hist_head[t] + 1) % st->obs_hist_len[t];
            }
            u.obs_delay_head[t] = st->obs_delay_head[t];
            u.obs_hist_head[t] = st->obs_hist_head[t];
        }
    }
    for (int r = 0; r < st->n_rewards; ++r) u.weight[r] = st->weight[r];
    u.actions = l->actions;
    u.reset_mask = l->reset_mask;
    u.policy_slot = l->policy_slot;
    u.policy_pad = 0;
    u.policy_lo = l->policy_lo;
    u.policy_hi = l->policy_hi;
    u.stats_out = l->stats_out;
    u.stats_partials = l->stats_partials;
    u.stats_ticket = l->stats_ticket;
    u.stats_rows = l->stats_rows;
    u.stats_pad = 0;
    int slot = -1;
    if (stages & SS_ST_TERM) {
        if (st->nf_pending >= st->nf_slots) {
            ss_set_error("ss_rt_launch", "nonfinite lag ring full: call ss_rt_poll");
            return -20;
        }
        slot = st->nf_slot;
        u.nf_slot = slot;
        st->nf_flags[slot] = 0;
    }
    const int rc = !jit ? ss_env_step(d, &u, stream)
                   : l->jit_desc ? ss_env_step_jit_packed(jit, d, l->jit_desc, l->jit_desc_bytes, &u, stream)
                                 : ss_env_step_jit(jit, d, &u, stream);
    if (rc != 0) return rc;
    st->launches += 1;
    if ((stages & SS_ST_PHYS) && nsub > 0) st->sim_step += nsub;
    if ((stages & SS_ST_OBS) && l->groups_mask + 1 == (1u << st->n_groups)) st->any_pending = 0;
    if ((stages & (SS_ST_RESET | SS_ST_RESET_ALL)) && !(stages & SS_ST_OBS)) st->any_pending = 1;
    if (slot >= 0) {
        cudaEvent_t ev = (cudaEvent_t)st->nf_event[slot];
        if (!ev) {
            cudaError_t e = cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
            if (e != cudaSuccess) {
                ss_set_error("cudaEventCreate", cudaGetErrorString(e));
                return -21;
            }
            st->nf_event[slot] = (uint64_t)ev;
        }
        cudaEventRecord(ev, (cudaStream_t)stream);
        st->nf_pushes[slot] = st->cap_pushes;
        st->nf_count[slot] = st->cap_count;
        st->nf_sim_step[slot] = st->sim_step;
        st->nf_pending += 1;
        st->nf_slot = (slot + 1) % st->nf_slots;
    }
    return 0;
}

extern "C" int ss_rt_poll(ss_rt_state* st, int32_t keep, int32_t* out_slots, int32_t max_out) {
    int found = 0;
    while (st->nf_pending > 0) {
        const int slot = st->nf_head;
        cudaEvent_t ev = (cudaEvent_t)st->nf_event[slot];
        if (st->nf_pending > keep) {
            cudaError_t e = cudaEventSynchronize(ev);
            if (e != cudaSuccess) {
                ss_set_error("cudaEventSynchronize", cudaGetErrorString(e));
                return -22;
            }
        } else if (cudaEventQuery(ev) != cudaSuccess) {
            break;
        }
        st->nf_head = (slot + 1) % st->nf_slots;
        st->nf_pending -= 1;
        if (((volatile uint32_t*)st->nf_flags)[slot] && found < max_out) out_slots[found++] = slot;
    }
    return found;
}

extern "C" int ss_rt_release(ss_rt_state* st) {
    for (int i = 0; i < SS_RT_SLOTS; ++i) {
        if (st->nf_event[i]) cudaEventDestroy((cudaEvent_t)st->nf_event[i]);
        st->nf_event[i] = 0;
    }
    return 0;
}

// ---------------------------------------------------------------------------------------------
// Pipelined host I/O (env.step_async / env.step_wait): every control step's actions come from
// pinned host memory and its output arena goes back to pinned host memory, with the transfers on
// two copy-engine streams so the PCIe traffic of one step overlaps the kernel of the next:
//   in stream : H2D actions(i) -> event in_done[k]
//   main      : wait in_done[k]; step kernel(i); wait out_done[k] (slot k's previous D2H);
//               snapshot kernel arena -> stage[k] (SM copy, not a copy engine); event snap[k]
//   out stream: wait snap[k]; D2H stage[k] -> host[i mod nhost]; event out_done[k]
// S slots (k = i mod S, 2 <= S <= 8; several in flight let the host enqueue the next steps while earlier
// ones run, which hides the host's per-step cost; consecutive steps' copies are grouped, ss_pipe_post).
// The step kernel reads device actions, so no mapped PCIe reads compete with the bulk D2H writes.

namespace {

__global__ void arena_copy_kernel(const int4* __restrict__ src, int4* __restrict__ dst, int64_t n16, int tail) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n16; i += (int64_t)gridDim.x * blockDim.x)
        dst[i] = __ldg(src + i);
    if (blockIdx.x == 0 && threadIdx.x < tail)
        reinterpret_cast<uint8_t*>(dst + n16)[threadIdx.x] = reinterpret_cast<const uint8_t*>(src + n16)[threadIdx.x];
}

struct Pipe {
    cudaStream_t in = nullptr, out = nullptr;
    cudaEvent_t in_done[8] = {}, snap[8] = {}, out_done[8] = {};
    bool used[8] = {};
    int nslot = 2, nhost = 3;
    int64_t submitted = 0, waited = 0;
    int group = 2;           // steps whose arenas cross PCIe as one copy (SS_PIPE_GROUP; 1 = one copy per step)
    int64_t dstart = -1;     // first step of the group being collected (D2H deferred, see ss_pipe_post)
    int dcount = 0;          // steps collected so far
    void* dev_actions[8] = {};
    void* stage[8] = {};
    void* host[16] = {};  // nhost > nslot pinned blocks: a view step_wait returned survives the next step_async
    int64_t action_bytes = 0, arena_bytes = 0;
};

// slots and host blocks of steps i .. i + group - 1 contiguous (one copy can move their arenas)
bool group_contiguous(const Pipe* p, int64_t i) {
    const int k = (int)(i % p->nslot), hk = (int)(i % p->nhost);
    if (k + p->group > p->nslot || hk + p->group > p->nhost) return false;
    for (int c = 1; c < p->group; ++c) {
        if ((char*)p->stage[k] + (int64_t)c * p->arena_bytes != (char*)p->stage[k + c]) return false;
        if ((char*)p->host[hk] + (int64_t)c * p->arena_bytes != (char*)p->host[hk + c]) return false;
    }
    return true;
}

// D2H of `count` consecutive steps' arenas starting at step i (slots and host blocks contiguous)
cudaError_t pipe_copy(Pipe* p, int64_t i, int count) {
    const int k = (int)(i % p->nslot), hk = (int)(i % p->nhost);
    const int klast = (int)((i + count - 1) % p->nslot);
    cudaError_t e = cudaStreamWaitEvent(p->out, p->snap[klast], 0);  // the main stream snapshots in order
    if (e == cudaSuccess)
        e = cudaMemcpyAsync(p->host[hk], p->stage[k], (size_t)p->arena_bytes * count, cudaMemcpyDeviceToHost, p->out);
    for (int c = 0; c < count && e == cudaSuccess; ++c) e = cudaEventRecord(p->out_done[(k + c) % p->nslot], p->out);
    return e;
}

int pipe_err(cudaError_t e, const char* what) {
    ss_set_error(what, cudaGetErrorString(e));
    return -2;
}

}  // namespace

extern "C" int ss_pipe_create(int32_t nslot, int32_t nhost, void* const* dev_actions, void* const* stage,
                              void* const* host, int64_t action_bytes, int64_t arena_bytes, void** out) {
    if (!dev_actions || !stage || !host || !out || arena_bytes <= 0 || action_bytes < 0 || nslot < 2 || nslot > 8 ||
        nhost <= nslot || nhost > 16) {
        ss_set_error("ss_pipe_create", "null buffer, empty arena, nslot outside [2, 8] or nhost outside (nslot, 16]");
        return -1;
    }
    Pipe* p = new Pipe();
    p->nslot = nslot;
    p->nhost = nhost;
    cudaError_t e = cudaStreamCreateWithFlags(&p->in, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&p->out, cudaStreamNonBlocking);
    for (int k = 0; k < nslot && e == cudaSuccess; ++k) {
        e = cudaEventCreateWithFlags(&p->in_done[k], cudaEventDisableTiming);
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&p->snap[k], cudaEventDisableTiming);
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&p->out_done[k], cudaEventDisableTiming);
        p->dev_actions[k] = dev_actions[k];
        p->stage[k] = stage[k];
    }
    for (int k = 0; k < nhost; ++k) p->host[k] = host[k];
    if (e != cudaSuccess) {
        delete p;
        return pipe_err(e, "ss_pipe_create");
    }
    p->action_bytes = action_bytes;
    p->arena_bytes = arena_bytes;
    const char* pe = getenv("SS_PIPE_PAIR");  // 0: one copy per step (A/B)
    const char* ge = getenv("SS_PIPE_GROUP");
    p->group = (pe && pe[0] == '0') ? 1 : (ge ? atoi(ge) : 2);
    if (p->group < 1 || p->group > nslot) p->group = 1;  // a collected group must fit the slots
    *out = p;
    return 0;
}

extern "C" int ss_pipe_destroy(void* h) {
    Pipe* p = static_cast<Pipe*>(h);
    if (!p) return 0;
    cudaStreamSynchronize(p->in);
    cudaStreamSynchronize(p->out);
    for (int k = 0; k < p->nslot; ++k) {
        cudaEventDestroy(p->in_done[k]);
        cudaEventDestroy(p->snap[k]);
        cudaEventDestroy(p->out_done[k]);
    }
    cudaStreamDestroy(p->in);
    cudaStreamDestroy(p->out);
    delete p;
    return 0;
}

// Before the step launch: H2D of this step's actions into slot k's device buffer; the main stream
// waits for it. Returns the slot (its device action buffer is what the step must read).
extern "C" int ss_pipe_pre(void* h, const void* host_actions, void* main_stream) {
    Pipe* p = static_cast<Pipe*>(h);
    if (p->submitted - p->waited >= p->nslot) {
        ss_set_error("ss_pipe_pre", "every slot pending: call step_wait first");
        return -1;
    }
    const int k = (int)(p->submitted % p->nslot);
    cudaStream_t main = static_cast<cudaStream_t>(main_stream);
    cudaError_t e = cudaSuccess;
    if (p->action_bytes) {
        // slot k's action buffer was last read by step i-S's kernel: order the copy after it
        if (p->used[k]) e = cudaStreamWaitEvent(p->in, p->snap[k], 0);
        if (e == cudaSuccess)
            e = cudaMemcpyAsync(p->dev_actions[k], host_actions, (size_t)p->action_bytes, cudaMemcpyHostToDevice, p->in);
        if (e == cudaSuccess) e = cudaEventRecord(p->in_done[k], p->in);
        if (e == cudaSuccess) e = cudaStreamWaitEvent(main, p->in_done[k], 0);
    }
    if (e != cudaSuccess) return pipe_err(e, "ss_pipe_pre");
    return k;
}

// After the step launch: snapshot the arena into slot k's staging buffer once the D2H that last
// read it is done, then D2H it on the out stream.
extern "C" int ss_pipe_post(void* h, const void* arena, void* main_stream) {
    Pipe* p = static_cast<Pipe*>(h);
    if (p->submitted - p->waited >= p->nslot) {
        ss_set_error("ss_pipe_post", "every slot pending: call step_wait first");
        return -1;
    }
    const int k = (int)(p->submitted % p->nslot);
    cudaStream_t main = static_cast<cudaStream_t>(main_stream);
    cudaError_t e = cudaSuccess;
    if (p->used[k]) e = cudaStreamWaitEvent(main, p->out_done[k], 0);
    if (e == cudaSuccess) {
        const int64_t n16 = p->arena_bytes / 16;
        const int grid = (int)((n16 + 255) / 256 < 296 ? (n16 + 255) / 256 : 296);
        arena_copy_kernel<<<grid > 0 ? grid : 1, 256, 0, main>>>(static_cast<const int4*>(arena),
                                                                  static_cast<int4*>(p->stage[k]), n16,
                                                                  (int)(p->arena_bytes & 15));
        e = cudaGetLastError();
    }
    if (e == cudaSuccess) e = cudaEventRecord(p->snap[k], main);
    // (one stream: splitting the D2H over two copy-engine streams measured no faster, 36.4 vs 34.0 us/step)
    // Host blocks rotate over nhost > nslot: the block of step i is rewritten by step i + nhost, which cannot be
    // submitted before step i + 1 has been waited for.
    // Grouping: back-to-back copies of one 1.58 MB arena each sustain ~31.3 us, of two arenas ~29.4 us per
    // arena, of four ~28.7 (tools/e2e_host.py), so when the slots and host blocks of `group` consecutive
    // steps (the first a multiple of `group`) are contiguous, their D2H copies are deferred and issued as one
    // once the last is submitted -- or, for the steps collected so far, by ss_pipe_wait if the caller waits
    // for one of them first (results are never held back behind a step not yet submitted). The deferred
    // steps are the latest submitted, fewer than group <= nslot, so a slot is never reused before its copy
    // was issued.
    const int64_t i = p->submitted;
    if (e == cudaSuccess) {
        if (p->dcount > 0) {  // i continues the group being collected
            if (++p->dcount == p->group) {
                e = pipe_copy(p, p->dstart, p->dcount);
                p->dcount = 0;
            }
        } else if (p->group > 1 && i % p->group == 0 && group_contiguous(p, i)) {
            p->dstart = i;
            p->dcount = 1;
        } else {
            e = pipe_copy(p, i, 1);
        }
    }
    if (e != cudaSuccess) return pipe_err(e, "ss_pipe_post");
    p->used[k] = true;
    p->submitted += 1;
    return k;
}

// Block until the oldest pending step's results are in host memory; returns its host block index
// (0..nslot; the block stays untouched until step_wait is called again).
extern "C" int ss_pipe_wait(void* h) {
    Pipe* p = static_cast<Pipe*>(h);
    if (p->waited >= p->submitted) {
        ss_set_error("ss_pipe_wait", "no pending step");
        return -1;
    }
    const int k = (int)(p->waited % p->nslot);
    const int hk = (int)(p->waited % p->nhost);
    cudaError_t e = cudaSuccess;
    if (p->dcount > 0 && p->waited >= p->dstart) {  // its group is incomplete: copy the steps collected so far
        e = pipe_copy(p, p->dstart, p->dcount);
        p->dcount = 0;
    }
    if (e == cudaSuccess) e = cudaEventSynchronize(p->out_done[k]);
    if (e != cudaSuccess) return pipe_err(e, "ss_pipe_wait");
    p->waited += 1;
    return hk;
}
