#define SS_DCAP_JOINTS 4
#define SS_DCAP_FEET 2
#define SS_DCAP_ACTION_TERMS 1
#define SS_DCAP_ACTUATORS 1
#define SS_DCAP_CMD 2
#define SS_DCAP_RAYS 5
#define SS_DCAP_GROUPS 2
#define SS_DCAP_OBS_TERMS 16
#define SS_DCAP_REWARDS 7
#define SS_DCAP_TERMINATIONS 3
#define SS_DCAP_EVENTS 3
#define SS_DCAP_CURRICULUM 2
#define SS_DCAP_FIELDS 8
#define SS_DCAP_SLOTS 16
#define SS_DCAP_MLP_LAYERS 1
#include "stridesim_b200.h"
static_assert(sizeof(ss_env_desc) == 4208, "packed descriptor layout differs from the host packing");
#include "ss_kernel.cuh"
struct JitCfg {
  static constexpr bool kJit = true;
  static constexpr int kUnroll = 64;
  static constexpr int kCapAct = 1;
  static constexpr int kCapActTerms = 1;
  static constexpr int kCapTerms = 3;
  static constexpr int kCapRewards = 7;
  static constexpr int kCapEvents = 3;
  static constexpr int kCapGroups = 2;
  static constexpr int kCapObs = 16;
  static constexpr int kBlock = 64, kStageObs = 1, kObsTotal = 47, kRays = 5;
  static __device__ __forceinline__ int g_soff(const ss_env_desc&, int g) { constexpr int a[4] = {0, 19, 0, 0}; return a[g]; }
  static __device__ __forceinline__ int NW(const ss_env_desc&) { return 4096; }
  static __device__ __forceinline__ int cap_phys(const ss_env_desc&) { return 220; }
  static __device__ __forceinline__ int mirror_on(const ss_env_desc&) { return 0; }
  static __device__ __forceinline__ int K(const ss_env_desc&) { return 4; }
  static __device__ __forceinline__ int F(const ss_env_desc&) { return 2; }
  static __device__ __forceinline__ double gravity(const ss_env_desc& d) { return d.model.gravity; }
  static __device__ __forceinline__ double dt(const ss_env_desc& d) { return d.model.dt; }
  static __device__ __forceinline__ double k_n(const ss_env_desc& d) { return d.model.k_n; }
  static __device__ __forceinline__ double c_n(const ss_env_desc& d) { return d.model.c_n; }
  static __device__ __forceinline__ double k_t(const ss_env_desc& d) { return d.model.k_t; }
  static __device__ __forceinline__ int f_base_mass(const ss_env_desc&) { return 0; }
  static __device__ __forceinline__ int f_base_inertia(const ss_env_desc&) { return 1; }
  static __device__ __forceinline__ int f_link_mass(const ss_env_desc&) { return 2; }
  static __device__ __forceinline__ int f_rotor(const ss_env_desc&) { return 3; }
  static __device__ __forceinline__ int f_damping(const ss_env_desc&) { return 4; }
  static __device__ __forceinline__ int f_friction(const ss_env_desc&) { return 5; }
  static __device__ __forceinline__ int flat(const ss_env_desc&) { return 0; }
  static __device__ __forceinline__ int decimation(const ss_env_desc&) { return 4; }
  static __device__ __forceinline__ int max_episode_steps(const ss_env_desc&) { return 1000; }
  static __device__ __forceinline__ double dt_control(const ss_env_desc& d) { return d.dt_control; }
  static __device__ __forceinline__ double spawn_offset(const ss_env_desc& d) { return d.spawn_offset; }
  static __device__ __forceinline__ int n_action_terms(const ss_env_desc&) { return 1; }
  static __device__ __forceinline__ int A(const ss_env_desc&) { return 4; }
  static __device__ __forceinline__ int n_act(const ss_env_desc&) { return 1; }
  static __device__ __forceinline__ int hist_len(const ss_env_desc&) { return 3; }
  static __device__ __forceinline__ int n_rays(const ss_env_desc&) { return 5; }
  static __device__ __forceinline__ int n_terms(const ss_env_desc&) { return 3; }
  static __device__ __forceinline__ int n_rewards(const ss_env_desc&) { return 7; }
  static __device__ __forceinline__ int n_cmd(const ss_env_desc&) { return 2; }
  static __device__ __forceinline__ int period_steps(const ss_env_desc&) { return 500; }
  static __device__ __forceinline__ int cmd_slot(const ss_env_desc&) { return 2; }
  static __device__ __forceinline__ double cap_scale(const ss_env_desc& d) { return d.cap_scale; }
  static __device__ __forceinline__ int n_events(const ss_env_desc&) { return 3; }
  static __device__ __forceinline__ int n_curr(const ss_env_desc&) { return 2; }
  static __device__ __forceinline__ int n_groups(const ss_env_desc&) { return 2; }
  static __device__ __forceinline__ int n_obs(const ss_env_desc&) { return 16; }
  static __device__ __forceinline__ int parent(const ss_env_desc&, int i) { constexpr int a[16] = {-1, 0, -1, 2, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0}; return a[i]; }
  static __device__ __forceinline__ int foot(const ss_env_desc&, int i) { constexpr int a[8] = {1, 3, 0, 0, 0, 0, 0, 0}; return a[i]; }
  static __device__ __forceinline__ unsigned chain(const ss_env_desc&, int i) { constexpr unsigned a[8] = {3u, 12u, 0u, 0u, 0u, 0u, 0u, 0u}; return a[i]; }
  static __device__ __forceinline__ double attach_x(const ss_env_desc& d, int i) { return d.model.attach_x[i]; }
  static __device__ __forceinline__ double attach_z(const ss_env_desc& d, int i) { return d.model.attach_z[i]; }
  static __device__ __forceinline__ double link_len(const ss_env_desc& d, int i) { return d.model.link_len[i]; }
  static __device__ __forceinline__ double half_len(const ss_env_desc& d, int i) { return d.model.half_len[i]; }
  static __device__ __forceinline__ double pos_lo(const ss_env_desc& d, int i) { return d.model.pos_lo[i]; }
  static __device__ __forceinline__ double pos_hi(const ss_env_desc& d, int i) { return d.model.pos_hi[i]; }
  static __device__ __forceinline__ double soft_frac(const ss_env_desc& d, int i) { return d.model.soft_frac[i]; }
  static __device__ __forceinline__ int fexp(const ss_env_desc&, int i) { constexpr int a[24] = {1, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0}; return a[i]; }
  static __device__ __forceinline__ int fsize(const ss_env_desc&, int i) { constexpr int a[24] = {1, 1, 4, 4, 4, 1, 4, 4, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0}; return a[i]; }
  static __device__ __forceinline__ double base_pose(const ss_env_desc& d, int i) { return d.base_pose[i]; }
  static __device__ __forceinline__ double base_vel(const ss_env_desc& d, int i) { return d.base_vel[i]; }
  static __device__ __forceinline__ double joint_pos(const ss_env_desc& d, int i) { return d.joint_pos[i]; }
  static __device__ __forceinline__ double joint_vel(const ss_env_desc& d, int i) { return d.joint_vel[i]; }
  static __device__ __forceinline__ int at_dim(const ss_env_desc&, int i) { constexpr int a[4] = {4, 0, 0, 0}; return a[i]; }
  static __device__ __forceinline__ int at_start(const ss_env_desc&, int i) { constexpr int a[4] = {0, 0, 0, 0}; return a[i]; }
  static __device__ __forceinline__ int at_has_clip(const ss_env_desc&, int i) { constexpr int a[4] = {1, 0, 0, 0}; return a[i]; }
  static __device__ __forceinline__ double at_scale(const ss_env_desc& d, int i) { return d.action_term[i].scale; }
  static __device__ __forceinline__ double at_clip_lo(const ss_env_desc& d, int i) { return d.action_term[i].clip_lo; }
  static __device__ __forceinline__ double at_clip_hi(const ss_env_desc& d, int i) { return d.action_term[i].clip_hi; }
  static __device__ __forceinline__ int act_kind(const ss_env_desc&, int i) { constexpr int a[4] = {0, 0, 0, 0}; return a[i]; }
  static __device__ __forceinline__ int act_delayed(const ss_env_desc&, int i) { constexpr int a[4] = {0, 0, 0, 0}; return a[i]; }
  static __device__ __forceinline__ int act_dim(const ss_env_desc&, int i) { constexpr int a[4] = {4, 0, 0, 0}; return a[i]; }
  static __device__ __forceinline__ int act_f_kp(const ss_env_desc&, int i) { constexpr int a[4] = {6, 0, 0, 0}; return a[i]; }
  static __device__ __forceinline__ int act_f_kd(const ss_env_desc&, int i) { constexpr int a[4] = {7, 0, 0, 0}; return a[i]; }
  static __device__ __forceinline__ int act_cap(const ss_env_desc&, int i) { constexpr int a[4] = {0, 0, 0, 0}; return a[i]; }
  static __device__ __forceinline__ int act_lat_slot(const ss_env_desc&, int i) { constexpr int a[4] = {0, 0, 0, 0}; return a[i]; }
  static __device__ __forceinline__ int act_lat_const(const ss_env_desc&, int i) { constexpr int a[4] = {0, 0, 0, 0}; return a[i]; }
  static __device__ __forceinline__ int act_resample(const ss_env_desc&, int i) { constexpr int a[4] = {0, 0, 0, 0}; return a[i]; }
  static __device__ __forceinline__ double act_effort(const ss_env_desc& d, int i) { return d.actuator[i].effort; }
  static __device__ __forceinline__ double act_sat(const ss_env_desc& d, int i) { return d.actuator[i].saturation; }
  static __device__ __forceinline__ double act_vlim(const ss_env_desc& d, int i) { return d.actuator[i].vel_limit; }
  static __device__ __forceinline__ double act_lat_lo(const ss_env_desc& d, int i) { return d.actuator[i].lat_lo; }
  static __device__ __forceinline__ double act_lat_hi(const ss_env_desc& d, int i) { return d.actuator[i].lat_hi; }
  static __device__ __forceinline__ double ray_offset(const ss_env_desc& d, int i) { return d.ray_offset[i]; }
  static __device__ __forceinline__ int term_func(const ss_env_desc&, int i) { constexpr int a[8] = {1, 2, 3, 0, 0, 0, 0, 0}; return a[i]; }
  static __device__ __forceinline__ int term_time_out(const ss_env_desc&, int i) { constexpr int a[8] = {0, 0, 1, 0, 0, 0, 0, 0}; return a[i]; }
  static __device__ __forceinline__ double term_p0(const ss_env_desc& d, int i) { return d.term[i].p0; }
  static __device__ __forceinline__ int rew_func(const ss_env_desc&, int i) { constexpr int a[16] = {3, 4, 5, 6, 7, 8, 9, 0, 0, 0, 0, 0, 0, 0, 0, 0}; return a[i]; }
  static __device__ __forceinline__ double rew_p0(const ss_env_desc& d, int i) { return d.reward[i].p0; }
  static __device__ __forceinline__ double init_lo(const ss_env_desc& d, int i) { return d.init_lo[i]; }
  static __device__ __forceinline__ double init_hi(const ss_env_desc& d, int i) { return d.init_hi[i]; }
  static __device__ __forceinline__ int ev_func(const ss_env_desc&, int i) { constexpr int a[8] = {1, 3, 2, 0, 0, 0, 0, 0}; return a[i]; }
  static __device__ __forceinline__ int ev_mode(const ss_env_desc&, int i) { constexpr int a[8] = {0, 1, 2, 0, 0, 0, 0, 0}; return a[i]; }
  static __device__ __forceinline__ int ev_iv_slot(const ss_env_desc&, int i) { constexpr int a[8] = {0, 0, 0, 0, 0, 0, 0, 0}; return a[i]; }
  static __device__ __forceinline__ int ev_field(const ss_env_desc&, int i) { constexpr int a[8] = {0, 0, 0, 0, 0, 0, 0, 0}; return a[i]; }
  static __device__ __forceinline__ int ev_dist(const ss_env_desc&, int i) { constexpr int a[8] = {0, 0, 0, 0, 0, 0, 0, 0}; return a[i]; }
  static __device__ __forceinline__ int ev_op(const ss_env_desc&, int i) { constexpr int a[8] = {1, 0, 0, 0, 0, 0, 0, 0}; return a[i]; }
  static __device__ __forceinline__ int ev_slot_a(const ss_env_desc&, int i) { constexpr int a[8] = {1, 3, 4, 0, 0, 0, 0, 0}; return a[i]; }
  static __device__ __forceinline__ int ev_slot_b(const ss_env_desc&, int i) { constexpr int a[8] = {0, 0, 5, 0, 0, 0, 0, 0}; return a[i]; }
  static __device__ __forceinline__ double ev_iv_lo(const ss_env_desc& d, int i) { return d.event[i].iv_lo; }
  static __device__ __forceinline__ double ev_iv_hi(const ss_env_desc& d, int i) { return d.event[i].iv_hi; }
  static __device__ __forceinline__ double ev_iv_lo_q(const ss_env_desc& d, int i) { return d.event[i].iv_lo_q; }
  static __device__ __forceinline__ double ev_iv_hi_q(const ss_env_desc& d, int i) { return d.event[i].iv_hi_q; }
  static __device__ __forceinline__ double ev_r0(const ss_env_desc& d, int i) { return d.event[i].r0; }
  static __device__ __forceinline__ double ev_r1(const ss_env_desc& d, int i) { return d.event[i].r1; }
  static __device__ __forceinline__ double ev_r2(const ss_env_desc& d, int i) { return d.event[i].r2; }
  static __device__ __forceinline__ double ev_r3(const ss_env_desc& d, int i) { return d.event[i].r3; }
  static __device__ __forceinline__ int cur_func(const ss_env_desc&, int i) { constexpr int a[4] = {2, 1, 0, 0}; return a[i]; }
  static __device__ __forceinline__ int cur_term(const ss_env_desc&, int i) { constexpr int a[4] = {0, 0, 0, 0}; return a[i]; }
  static __device__ __forceinline__ double cur_p0(const ss_env_desc& d, int i) { return d.curriculum[i].p0; }
  static __device__ __forceinline__ double cur_p1(const ss_env_desc& d, int i) { return d.curriculum[i].p1; }
  static __device__ __forceinline__ int g_dim(const ss_env_desc&, int i) { constexpr int a[4] = {19, 28, 0, 0}; return a[i]; }
  static __device__ __forceinline__ int g_first(const ss_env_desc&, int i) { constexpr int a[4] = {0, 7, 0, 0}; return a[i]; }
  static __device__ __forceinline__ int g_n(const ss_env_desc&, int i) { constexpr int a[4] = {7, 9, 0, 0}; return a[i]; }
  static __device__ __forceinline__ int obs_func(const ss_env_desc&, int i) { constexpr int a[32] = {1, 2, 4, 5, 6, 7, 8, 1, 2, 4, 5, 6, 7, 8, 12, 11, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0}; return a[i]; }
  static __device__ __forceinline__ int obs_dim(const ss_env_desc&, int i) { constexpr int a[32] = {2, 1, 2, 4, 4, 4, 2, 2, 1, 2, 4, 4, 4, 2, 4, 5, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0}; return a[i]; }
  static __device__ __forceinline__ int obs_col(const ss_env_desc&, int i) { constexpr int a[32] = {0, 2, 3, 5, 9, 13, 17, 0, 2, 3, 5, 9, 13, 17, 19, 23, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0}; return a[i]; }
  static __device__ __forceinline__ int obs_has_clip(const ss_env_desc&, int i) { constexpr int a[32] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 1, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0}; return a[i]; }
  static __device__ __forceinline__ int obs_has_scale(const ss_env_desc&, int i) { constexpr int a[32] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 1, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0}; return a[i]; }
  static __device__ __forceinline__ int obs_noise(const ss_env_desc&, int i) { constexpr int a[32] = {1, 1, 1, 1, 1, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0}; return a[i]; }
  static __device__ __forceinline__ int obs_noise_slot(const ss_env_desc&, int i) { constexpr int a[32] = {6, 7, 8, 9, 10, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0}; return a[i]; }
  static __device__ __forceinline__ int obs_delay(const ss_env_desc&, int i) { constexpr int a[32] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0}; return a[i]; }
  static __device__ __forceinline__ int obs_history(const ss_env_desc&, int i) { constexpr int a[32] = {1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0}; return a[i]; }
  static __device__ __forceinline__ double obs_clip_lo(const ss_env_desc& d, int i) { return d.obs[i].clip_lo; }
  static __device__ __forceinline__ double obs_clip_hi(const ss_env_desc& d, int i) { return d.obs[i].clip_hi; }
  static __device__ __forceinline__ double obs_scale(const ss_env_desc& d, int i) { return d.obs[i].scale; }
  static __device__ __forceinline__ double obs_noise_scale(const ss_env_desc& d, int i) { return d.obs[i].noise_scale; }
  static __device__ __forceinline__ int at_joint(const ss_env_desc&, int t, int i) { constexpr int a[4][16] = {{0, 1, 2, 3, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0}, {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0}, {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0}, {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0}}; return a[t][i]; }
  static __device__ __forceinline__ double at_offset(const ss_env_desc& d, int t, int i) { return d.action_term[t].offset[i]; }
  static __device__ __forceinline__ int act_joint(const ss_env_desc&, int t, int i) { constexpr int a[4][16] = {{0, 1, 2, 3, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0}, {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0}, {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0}, {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0}}; return a[t][i]; }
  static __device__ __forceinline__ double fbase(const ss_env_desc& d, int t, int i) { return d.field[t].base[i]; }
};
extern "C" __global__ void __launch_bounds__(64) ss_step_jit(
    const __grid_constant__ ss_env_desc d, const __grid_constant__ ss_uniforms u) {
  ss::step_body<JitCfg, 4, 2>(d, u);
}
