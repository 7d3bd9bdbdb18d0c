// ss_cfg.cuh -- every configuration value the step kernel reads, as one list.
//
// The kernel body (ss_kernel.cuh) is a template over a config type C and
// reads each value as C::name(d[, i[, j]]). Two config types exist:
//
//  * RuntimeCfg (below): reads the value from the ss_env_desc kernel
//    parameter -- the generic ahead-of-time build, valid for any env.
//  * the JIT config generated per env by paper_2601_22074_b200/jit.py:
//    every value is a constexpr, so the NVRTC-compiled kernel has all term
//    tables, topology and constants folded in and every loop unrolled. This
//    is the B200 analog of the reference's StepPipeline._rebuild
//    (sim/physics.py:158-237): re-specialize the step to the current model
//    layout; it is recompiled whenever the layout (generation) changes.
//
// jit.py parses these X-lists and evaluates each expression (valid Python
// over the ctypes desc) to emit the constexpr values, so the two can never
// drift apart. Format: X(type, name, expression) / XA(type, name, bound,
// expression using i) / XB(type, name, bound_t, bound_i, expression using t, i).
#pragma once

// clang-format off
#define SS_CFG_SCALARS(X) \
    X(int, NW, d.n_worlds) \
    X(int, cap_phys, d.capture_phys) \
    X(int, mirror_on, (d.out_mirror != 0)) \
    X(int, K, d.model.n_joints) \
    X(int, F, d.model.n_feet) \
    X(double, gravity, d.model.gravity) \
    X(double, dt, d.model.dt) \
    X(double, k_n, d.model.k_n) \
    X(double, c_n, d.model.c_n) \
    X(double, k_t, d.model.k_t) \
    X(int, f_base_mass, d.model.f_base_mass) \
    X(int, f_base_inertia, d.model.f_base_inertia) \
    X(int, f_link_mass, d.model.f_link_mass) \
    X(int, f_rotor, d.model.f_rotor_inertia) \
    X(int, f_damping, d.model.f_damping) \
    X(int, f_friction, d.model.f_friction) \
    X(int, flat, d.terrain.flat) \
    X(int, decimation, d.decimation) \
    X(int, max_episode_steps, d.max_episode_steps) \
    X(double, dt_control, d.dt_control) \
    X(double, spawn_offset, d.spawn_offset) \
    X(int, n_action_terms, d.n_action_terms) \
    X(int, A, d.action_dim) \
    X(int, n_act, d.n_actuators) \
    X(int, hist_len, d.hist_len) \
    X(int, n_rays, d.n_rays) \
    X(int, n_terms, d.n_terms) \
    X(int, n_rewards, d.n_rewards) \
    X(int, n_cmd, d.n_cmd) \
    X(int, period_steps, d.period_steps) \
    X(int, cmd_slot, d.cmd_slot) \
    X(double, cap_scale, d.cap_scale) \
    X(int, n_events, d.n_events) \
    X(int, n_curr, d.n_curriculum) \
    X(int, n_groups, d.n_groups) \
    X(int, n_obs, d.n_obs_terms)

#define SS_CFG_ARRAYS(XA) \
    XA(int, parent, SS_MAX_JOINTS, d.model.parent[i]) \
    XA(int, foot, SS_MAX_FEET, d.model.foot_joint[i]) \
    XA(unsigned, chain, SS_MAX_FEET, d.model.chain_mask[i]) \
    XA(double, attach_x, SS_MAX_JOINTS, d.model.attach_x[i]) \
    XA(double, attach_z, SS_MAX_JOINTS, d.model.attach_z[i]) \
    XA(double, link_len, SS_MAX_JOINTS, d.model.link_len[i]) \
    XA(double, half_len, SS_MAX_JOINTS, d.model.half_len[i]) \
    XA(double, pos_lo, SS_MAX_JOINTS, d.model.pos_lo[i]) \
    XA(double, pos_hi, SS_MAX_JOINTS, d.model.pos_hi[i]) \
    XA(double, soft_frac, SS_MAX_JOINTS, d.model.soft_frac[i]) \
    XA(int, fexp, SS_MAX_FIELDS, d.field[i].expanded) \
    XA(int, fsize, SS_MAX_FIELDS, d.field[i].size) \
    XA(double, base_pose, 3, d.base_pose[i]) \
    XA(double, base_vel, 3, d.base_vel[i]) \
    XA(double, joint_pos, SS_MAX_JOINTS, d.joint_pos[i]) \
    XA(double, joint_vel, SS_MAX_JOINTS, d.joint_vel[i]) \
    XA(int, at_dim, SS_MAX_ACTION_TERMS, d.action_term[i].dim) \
    XA(int, at_start, SS_MAX_ACTION_TERMS, d.action_term[i].start) \
    XA(int, at_has_clip, SS_MAX_ACTION_TERMS, d.action_term[i].has_clip) \
    XA(double, at_scale, SS_MAX_ACTION_TERMS, d.action_term[i].scale) \
    XA(double, at_clip_lo, SS_MAX_ACTION_TERMS, d.action_term[i].clip_lo) \
    XA(double, at_clip_hi, SS_MAX_ACTION_TERMS, d.action_term[i].clip_hi) \
    XA(int, act_kind, SS_MAX_ACTUATORS, d.actuator[i].kind) \
    XA(int, act_delayed, SS_MAX_ACTUATORS, d.actuator[i].delayed) \
    XA(int, act_dim, SS_MAX_ACTUATORS, d.actuator[i].dim) \
    XA(int, act_f_kp, SS_MAX_ACTUATORS, d.actuator[i].f_kp) \
    XA(int, act_f_kd, SS_MAX_ACTUATORS, d.actuator[i].f_kd) \
    XA(int, act_cap, SS_MAX_ACTUATORS, d.actuator[i].cap) \
    XA(int, act_lat_slot, SS_MAX_ACTUATORS, d.actuator[i].lat_slot) \
    XA(int, act_lat_const, SS_MAX_ACTUATORS, d.actuator[i].lat_const) \
    XA(int, act_resample, SS_MAX_ACTUATORS, d.actuator[i].resample_on_reset) \
    XA(double, act_effort, SS_MAX_ACTUATORS, d.actuator[i].effort) \
    XA(double, act_sat, SS_MAX_ACTUATORS, d.actuator[i].saturation) \
    XA(double, act_vlim, SS_MAX_ACTUATORS, d.actuator[i].vel_limit) \
    XA(double, act_lat_lo, SS_MAX_ACTUATORS, d.actuator[i].lat_lo) \
    XA(double, act_lat_hi, SS_MAX_ACTUATORS, d.actuator[i].lat_hi) \
    XA(double, ray_offset, SS_MAX_RAYS, d.ray_offset[i]) \
    XA(int, term_func, SS_MAX_TERMINATIONS, d.term[i].func) \
    XA(int, term_time_out, SS_MAX_TERMINATIONS, d.term[i].time_out) \
    XA(double, term_p0, SS_MAX_TERMINATIONS, d.term[i].p0) \
    XA(int, rew_func, SS_MAX_REWARDS, d.reward[i].func) \
    XA(double, rew_p0, SS_MAX_REWARDS, d.reward[i].p0) \
    XA(double, init_lo, SS_MAX_CMD, d.init_lo[i]) \
    XA(double, init_hi, SS_MAX_CMD, d.init_hi[i]) \
    XA(int, ev_func, SS_MAX_EVENTS, d.event[i].func) \
    XA(int, ev_mode, SS_MAX_EVENTS, d.event[i].mode) \
    XA(int, ev_iv_slot, SS_MAX_EVENTS, d.event[i].iv_slot) \
    XA(int, ev_field, SS_MAX_EVENTS, d.event[i].field) \
    XA(int, ev_dist, SS_MAX_EVENTS, d.event[i].distribution) \
    XA(int, ev_op, SS_MAX_EVENTS, d.event[i].operation) \
    XA(int, ev_slot_a, SS_MAX_EVENTS, d.event[i].slot_a) \
    XA(int, ev_slot_b, SS_MAX_EVENTS, d.event[i].slot_b) \
    XA(double, ev_iv_lo, SS_MAX_EVENTS, d.event[i].iv_lo) \
    XA(double, ev_iv_hi, SS_MAX_EVENTS, d.event[i].iv_hi) \
    XA(double, ev_iv_lo_q, SS_MAX_EVENTS, d.event[i].iv_lo_q) \
    XA(double, ev_iv_hi_q, SS_MAX_EVENTS, d.event[i].iv_hi_q) \
    XA(double, ev_r0, SS_MAX_EVENTS, d.event[i].r0) \
    XA(double, ev_r1, SS_MAX_EVENTS, d.event[i].r1) \
    XA(double, ev_r2, SS_MAX_EVENTS, d.event[i].r2) \
    XA(double, ev_r3, SS_MAX_EVENTS, d.event[i].r3) \
    XA(int, cur_func, SS_MAX_CURRICULUM, d.curriculum[i].func) \
    XA(int, cur_term, SS_MAX_CURRICULUM, d.curriculum[i].term) \
    XA(double, cur_p0, SS_MAX_CURRICULUM, d.curriculum[i].p0) \
    XA(double, cur_p1, SS_MAX_CURRICULUM, d.curriculum[i].p1) \
    XA(int, g_dim, SS_MAX_GROUPS, d.group[i].dim) \
    XA(int, g_first, SS_MAX_GROUPS, d.group[i].first_term) \
    XA(int, g_n, SS_MAX_GROUPS, d.group[i].n_terms) \
    XA(int, obs_func, SS_MAX_OBS_TERMS, d.obs[i].func) \
    XA(int, obs_dim, SS_MAX_OBS_TERMS, d.obs[i].dim) \
    XA(int, obs_col, SS_MAX_OBS_TERMS, d.obs[i].col) \
    XA(int, obs_has_clip, SS_MAX_OBS_TERMS, d.obs[i].has_clip) \
    XA(int, obs_has_scale, SS_MAX_OBS_TERMS, d.obs[i].has_scale) \
    XA(int, obs_noise, SS_MAX_OBS_TERMS, d.obs[i].noise) \
    XA(int, obs_noise_slot, SS_MAX_OBS_TERMS, d.obs[i].noise_slot) \
    XA(int, obs_delay, SS_MAX_OBS_TERMS, d.obs[i].delay) \
    XA(int, obs_history, SS_MAX_OBS_TERMS, d.obs[i].history) \
    XA(double, obs_clip_lo, SS_MAX_OBS_TERMS, d.obs[i].clip_lo) \
    XA(double, obs_clip_hi, SS_MAX_OBS_TERMS, d.obs[i].clip_hi) \
    XA(double, obs_scale, SS_MAX_OBS_TERMS, d.obs[i].scale) \
    XA(double, obs_noise_scale, SS_MAX_OBS_TERMS, d.obs[i].noise_scale)

#define SS_CFG_ARRAYS2(XB) \
    XB(int, at_joint, SS_MAX_ACTION_TERMS, SS_MAX_JOINTS, d.action_term[t].joint[i]) \
    XB(double, at_offset, SS_MAX_ACTION_TERMS, SS_MAX_JOINTS, d.action_term[t].offset[i]) \
    XB(int, act_joint, SS_MAX_ACTUATORS, SS_MAX_JOINTS, d.actuator[t].joint[i]) \
    XB(double, fbase, SS_MAX_FIELDS, SS_MAX_JOINTS, d.field[t].base[i])
// clang-format on

namespace ss {

// Generic (ahead-of-time) configuration: every value from the descriptor.
struct RuntimeCfg {
    static constexpr bool kJit = false;
    static constexpr int kUnroll = 1;  // term-table loops stay loops in the generic build
    static constexpr int kCapAct = SS_MAX_ACTUATORS, kCapActTerms = SS_MAX_ACTION_TERMS;
    static constexpr int kCapTerms = SS_MAX_TERMINATIONS, kCapRewards = SS_MAX_REWARDS;
    static constexpr int kCapEvents = SS_MAX_EVENTS, kCapGroups = SS_MAX_GROUPS, kCapObs = SS_MAX_OBS_TERMS;
    static constexpr int kBlock = 128, kStageObs = 0, kObsTotal = 0, kRays = SS_MAX_RAYS;
    static constexpr int kParamSmemAlone = 0;
    static constexpr int kParamSmem = 0, kActSmem = 0, kDynSmem = 0, kDynObs = 0, kDynParam = 0, kDynAct = 0;
    static __device__ __forceinline__ int g_soff(const ss_env_desc&, int) { return 0; }
#define SS_RT_X(T, name, expr) \
    static __device__ __forceinline__ T name(const ss_env_desc& d) { return (T)(expr); }
#define SS_RT_XA(T, name, bound, expr) \
    static __device__ __forceinline__ T name(const ss_env_desc& d, int i) { return (T)(expr); }
#define SS_RT_XB(T, name, bt, bi, expr) \
    static __device__ __forceinline__ T name(const ss_env_desc& d, int t, int i) { return (T)(expr); }
    SS_CFG_SCALARS(SS_RT_X)
    SS_CFG_ARRAYS(SS_RT_XA)
    SS_CFG_ARRAYS2(SS_RT_XB)
#undef SS_RT_X
#undef SS_RT_XA
#undef SS_RT_XB
};

}  // namespace ss
