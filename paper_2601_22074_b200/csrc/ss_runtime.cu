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
