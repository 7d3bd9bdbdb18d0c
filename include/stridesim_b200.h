/*
 * stridesim_b200.h -- C-ABI of the B200 (sm_100a) batched ManagerBasedRlEnv.step.
 *
 * This is the drop-in boundary of the hot path. The reference is pure Python
 * (`stridesim`, /root/reference/pkg/src/stridesim); its "FFI" for this path is
 * the Python call surface below, which the host package binds with ctypes
 * (see INTEGRATION.md). Every entry point takes plain pointers / sizes, never
 * torch types, is asynchronous on the given CUDA stream, allocation-free, and
 * returns 0 on success or a negative status (message via ss_last_error()).
 *
 * Reference interfaces each entry point replaces:
 *   ss_env_step      ManagerBasedRlEnv.step / reset stages      env.py:202-259
 *                    (ActionManager.process/apply     managers/action.py:68-97,
 *                     StepPipeline.substep            sim/physics.py:239-249,
 *                     EntityData.refresh              entity.py:145-165,
 *                     ContactSensor.update/reset      sensors.py:81-115,
 *                     CaptureRing.push                capture.py:53-59,
 *                     TerminationManager.compute      managers/termination.py:24-41,
 *                     RewardManager.compute/reset     managers/reward.py:36-62,
 *                     CurriculumManager.update        managers/curriculum.py:21-23,
 *                     _reset_worlds                   env.py:182-200,
 *                     CommandManager.update/resample  managers/command.py:33-50,
 *                     EventManager.apply_reset/interval managers/event.py:92-114,
 *                     ObservationManager.compute      managers/observation.py:99-141)
 *   ss_rng_draw      StreamPack.uniform / normal        rng.py:86-119
 *   ss_fk            fk_batch_trig                      sim/physics.py:22-57
 *   ss_heights       Heightfield.heights                terrain.py:159-169
 *   ss_randomize     randomize_field (startup/explicit) managers/event.py:19-52
 *   ss_actuator_eval pd_torque / dc_motor_torque        actuators.py:104-117
 *   ss_stats_pack    metrics.build_record reductions    metrics.py:31-45
 *   ss_rt_*          ManagerBasedRlEnv.step bookkeeping (env.py:219-259)
 *   ss_jit_*         StepPipeline._rebuild (re-specialize to the layout) sim/physics.py:158-237
 *
 * Layout: every per-world array is structure-of-arrays, component-major,
 * i.e. element (world w, component c) of an (N, C) logical array lives at
 * ptr[c * N + w]. Observation group outputs are the exception: they are
 * row-major (N, D) because that is what a policy consumes.
 *
 * The struct definitions below are parsed by the Python host package
 * (paper_2601_22074_b200/native.py) to build matching ctypes layouts, so keep
 * to the restricted style: one field per line, `type name;` or
 * `type name[DIM];` / `type name[DIM][DIM];`.
 */
#ifndef STRIDESIM_B200_H
#define STRIDESIM_B200_H

#ifdef __CUDACC_RTC__
/* NVRTC (the per-env JIT specialization of the step) has no libc headers */
typedef signed char int8_t;
typedef unsigned char uint8_t;
typedef int int32_t;
typedef unsigned int uint32_t;
typedef long long int64_t;
typedef unsigned long long uint64_t;
#else
#include <stddef.h>
#include <stdint.h>
#endif

#ifdef __cplusplus
extern "C" {
#endif

#define SS_ABI_VERSION 5

#define SS_MAX_JOINTS 16
#define SS_MAX_FEET 8
#define SS_MAX_ACTION 16
#define SS_MAX_ACTION_TERMS 4
#define SS_MAX_ACTUATORS 4
#define SS_MAX_CMD 4
#define SS_MAX_RAYS 16
#define SS_MAX_GROUPS 4
#define SS_MAX_OBS_TERMS 32
#define SS_MAX_REWARDS 16
#define SS_MAX_TERMINATIONS 8
#define SS_MAX_EVENTS 8
#define SS_MAX_CURRICULUM 4
#define SS_MAX_FIELDS 24
#define SS_MAX_SLOTS 48
#define SS_MAX_MLP_LAYERS 4
#define SS_MAX_HIST 8

/* Array bounds of the descriptor structs. The ABI (this header as compiled
 * by the library and parsed by the Python binding) uses the SS_MAX_* caps;
 * a per-env specialized kernel (jit.py) defines them to the env's actual
 * counts before including this header, so its descriptor parameter block
 * holds only the entries that exist (ss_launch.jit_desc carries that packed
 * copy). */
#ifndef SS_DCAP_JOINTS
#define SS_DCAP_JOINTS SS_MAX_JOINTS
#endif
#ifndef SS_DCAP_FEET
#define SS_DCAP_FEET SS_MAX_FEET
#endif
#ifndef SS_DCAP_ACTION_TERMS
#define SS_DCAP_ACTION_TERMS SS_MAX_ACTION_TERMS
#endif
#ifndef SS_DCAP_ACTUATORS
#define SS_DCAP_ACTUATORS SS_MAX_ACTUATORS
#endif
#ifndef SS_DCAP_CMD
#define SS_DCAP_CMD SS_MAX_CMD
#endif
#ifndef SS_DCAP_RAYS
#define SS_DCAP_RAYS SS_MAX_RAYS
#endif
#ifndef SS_DCAP_GROUPS
#define SS_DCAP_GROUPS SS_MAX_GROUPS
#endif
#ifndef SS_DCAP_OBS_TERMS
#define SS_DCAP_OBS_TERMS SS_MAX_OBS_TERMS
#endif
#ifndef SS_DCAP_REWARDS
#define SS_DCAP_REWARDS SS_MAX_REWARDS
#endif
#ifndef SS_DCAP_TERMINATIONS
#define SS_DCAP_TERMINATIONS SS_MAX_TERMINATIONS
#endif
#ifndef SS_DCAP_EVENTS
#define SS_DCAP_EVENTS SS_MAX_EVENTS
#endif
#ifndef SS_DCAP_CURRICULUM
#define SS_DCAP_CURRICULUM SS_MAX_CURRICULUM
#endif
#ifndef SS_DCAP_FIELDS
#define SS_DCAP_FIELDS SS_MAX_FIELDS
#endif
#ifndef SS_DCAP_SLOTS
#define SS_DCAP_SLOTS SS_MAX_SLOTS
#endif
#ifndef SS_DCAP_MLP_LAYERS
#define SS_DCAP_MLP_LAYERS SS_MAX_MLP_LAYERS
#endif

/* stage bits for ss_uniforms.stages (reference order: env.py:219-259) */
#define SS_ST_ACTION 1u        /* ActionManager.process                      */
#define SS_ST_APPLY 2u         /* per substep: ActionManager.apply            */
#define SS_ST_PUSH 4u          /* per substep: CaptureRing.push               */
#define SS_ST_PHYS 8u          /* per substep: StepPipeline.substep (+refresh)*/
#define SS_ST_SENSOR 16u       /* per substep: ContactSensor.update           */
#define SS_ST_TERM 32u         /* episode bookkeeping + TerminationManager    */
#define SS_ST_REWARD 64u       /* RewardManager.compute                       */
#define SS_ST_CURRICULUM 128u  /* CurriculumManager.update on reset worlds    */
#define SS_ST_RESET 256u       /* _reset_worlds(terminated | truncated)       */
#define SS_ST_RESET_ALL 512u   /* _reset_worlds(all)  (env.reset)             */
#define SS_ST_COMMAND 1024u    /* CommandManager.update                       */
#define SS_ST_EVENTS 2048u     /* EventManager.apply_interval                 */
#define SS_ST_OBS 4096u        /* ObservationManager.compute for groups_mask  */
#define SS_ST_PREV_AFTER 8192u /* prev_lin_vel_b <- root_lin_vel_b after obs  */
#define SS_ST_PREV_BEFORE 16384u /* ... before obs (env.reset order)          */
#define SS_ST_RESET_EXT 32768u /* reset mask read from uniforms.reset_mask    */
#define SS_ST_STEP_ALL 0x3DFFu /* ACTION..PREV_AFTER, without RESET_ALL      */

/* ss_uniforms.flags */
#define SS_FLAG_NO_EPISODE 1u  /* TERM without the env.py:235-238 bookkeeping  */

/* observation term function ids (mdp.py:26-89) */
#define SS_OBS_BASE_LIN_VEL 1
#define SS_OBS_BASE_ANG_VEL 2
#define SS_OBS_BASE_LIN_ACC 3
#define SS_OBS_PROJECTED_GRAVITY 4
#define SS_OBS_JOINT_POS_REL 5
#define SS_OBS_JOINT_VEL 6
#define SS_OBS_LAST_ACTION 7
#define SS_OBS_COMMAND 8
#define SS_OBS_BASE_HEIGHT 9
#define SS_OBS_SIM_TIME 10
#define SS_OBS_HEIGHT_SCAN 11
#define SS_OBS_FOOT_CONTACT_FORCES 12
#define SS_OBS_EXTERNAL 99

/* reward term function ids (mdp.py:96-160) */
#define SS_REW_CONSTANT 1
#define SS_REW_BASE_HEIGHT 2
#define SS_REW_TRACK_VX_EXP 3
#define SS_REW_PITCH_RATE 4
#define SS_REW_ANG_MOMENTUM 5
#define SS_REW_ACTION_RATE 6
#define SS_REW_JOINT_LIMIT 7
#define SS_REW_FOOT_SLIP 8
#define SS_REW_FEET_AIR_TIME 9
#define SS_REW_EXTERNAL 99

/* termination term function ids (mdp.py:167-179) */
#define SS_TERM_BASE_HEIGHT_BELOW 1
#define SS_TERM_PITCH_BEYOND 2
#define SS_TERM_TIME_OUT 3
#define SS_TERM_EXTERNAL 99

/* event term function ids (mdp.py:186-220) and modes (managers/event.py) */
#define SS_EVT_RANDOMIZE_FIELD 1
#define SS_EVT_PUSH_BASE 2
#define SS_EVT_JOINT_JITTER 3
#define SS_EVT_EXTERNAL 99
#define SS_MODE_STARTUP 0
#define SS_MODE_RESET 1
#define SS_MODE_INTERVAL 2
#define SS_DIST_UNIFORM 0
#define SS_DIST_GAUSSIAN 1
#define SS_OP_SET 0
#define SS_OP_SCALE 1
#define SS_OP_ADD 2

/* curriculum term function ids (mdp.py:227-275); schedule terms run on host */
#define SS_CUR_TERRAIN_LEVELS 1
#define SS_CUR_COMMAND_WIDEN 2

/* actuator kinds (actuators.py:37-117) */
#define SS_ACT_PD 0
#define SS_ACT_DC 1
#define SS_ACT_MLP 2
#define SS_MLP_IDENTITY 0
#define SS_MLP_RELU 1
#define SS_MLP_TANH 2

/* noise kinds (managers/base.py:95-98) */
#define SS_NOISE_NONE 0
#define SS_NOISE_UNIFORM 1
#define SS_NOISE_GAUSSIAN 2

/* A randomizable model field (sim/model.py:26-38): shared -> `size` values
 * read by every world; expanded -> SoA (size, N). */
typedef struct ss_field {
    double* ptr;
    int32_t expanded;
    int32_t size;
    double base[SS_DCAP_JOINTS];
} ss_field;

/* Compiled chain structure (sim/model.py:43-92) + contact constants. */
typedef struct ss_model {
    int32_t n_joints;
    int32_t n_feet;
    int32_t parent[SS_DCAP_JOINTS];
    int32_t foot_joint[SS_DCAP_FEET];
    uint32_t chain_mask[SS_DCAP_FEET];
    double attach_x[SS_DCAP_JOINTS];
    double attach_z[SS_DCAP_JOINTS];
    double link_len[SS_DCAP_JOINTS];
    double half_len[SS_DCAP_JOINTS];
    double pos_lo[SS_DCAP_JOINTS];
    double pos_hi[SS_DCAP_JOINTS];
    double soft_frac[SS_DCAP_JOINTS];
    double gravity;
    double dt;
    double k_n;
    double c_n;
    double k_t;
    int32_t f_base_mass;
    int32_t f_base_inertia;
    int32_t f_link_mass;
    int32_t f_rotor_inertia;
    int32_t f_damping;
    int32_t f_friction;
} ss_model;

/* Stitched 1-D heightfield (terrain.py:121-169). */
typedef struct ss_terrain {
    const double* samples;
    int64_t n_samples;
    double spacing;
    int32_t flat;
    int32_t rows;
    int32_t cols;
    int32_t pad0;
    double patch_length;
} ss_terrain;

/* BatchState + ContactCache (sim/state.py:10-38). */
typedef struct ss_state {
    double* q;
    double* qd;
    double* ctrl;
    double* ext_force;
    double* time;
    double* c_normal;
    double* c_tangent;
    double* c_foot_pos;
    double* c_foot_vel;
    uint8_t* c_in_contact;
} ss_state;

/* Counter-based splitmix streams (rng.py:44-84): key(world) is recomputed
 * on device from base[slot] and the global world id; counters are (N,). */
typedef struct ss_rng {
    int64_t world_id_offset;
    uint64_t base[SS_DCAP_SLOTS];
    uint64_t* counter[SS_DCAP_SLOTS];
} ss_rng;

typedef struct ss_action_term {
    int32_t dim;
    int32_t start;
    int32_t has_clip;
    int32_t pad0;
    int32_t joint[SS_DCAP_JOINTS];
    double offset[SS_DCAP_JOINTS];
    double scale;
    double clip_lo;
    double clip_hi;
} ss_action_term;

typedef struct ss_mlp_layer {
    const double* w;
    const double* b;
    int32_t in_dim;
    int32_t out_dim;
    int32_t act;
    int32_t pad0;
} ss_mlp_layer;

typedef struct ss_actuator {
    int32_t kind;
    int32_t delayed;
    int32_t dim;
    int32_t f_kp;
    int32_t f_kd;
    int32_t cap;
    int32_t lat_slot;
    int32_t lat_const;
    int32_t resample_on_reset;
    int32_t n_layers;
    int32_t err_hist;
    int32_t vel_hist;
    int32_t joint[SS_DCAP_JOINTS];
    double effort;
    double saturation;
    double vel_limit;
    double lat_lo;
    double lat_hi;
    double* ring;
    int64_t* delay_steps;
    double* err_buf;
    double* vel_buf;
    ss_mlp_layer layer[SS_DCAP_MLP_LAYERS];
} ss_actuator;

typedef struct ss_obs_term {
    int32_t func;
    int32_t dim;
    int32_t group;
    int32_t col;
    int32_t has_clip;
    int32_t has_scale;
    int32_t noise;
    int32_t noise_slot;
    int32_t delay;
    int32_t history;
    double clip_lo;
    double clip_hi;
    double scale;
    double noise_scale;
    double* delay_ring;
    double* hist_ring;
    const double* ext;
} ss_obs_term;

typedef struct ss_obs_group {
    double* out;
    uint8_t* pending;
    int32_t dim;
    int32_t first_term;
    int32_t n_terms;
    int32_t enable_noise;
} ss_obs_group;

typedef struct ss_reward_term {
    int32_t func;
    int32_t pad0;
    double p0;
    const double* ext;
} ss_reward_term;

typedef struct ss_term_term {
    int32_t func;
    int32_t time_out;
    double p0;
    const uint8_t* ext;
} ss_term_term;

typedef struct ss_event_term {
    int32_t func;
    int32_t mode;
    int32_t iv_slot;
    int32_t field;
    int32_t distribution;
    int32_t operation;
    int32_t slot_a;
    int32_t slot_b;
    double iv_lo;
    double iv_hi;
    double iv_lo_q;
    double iv_hi_q;
    double r0;
    double r1;
    double r2;
    double r3;
    double* elapsed;
    double* target;
    uint8_t* fired;
} ss_event_term;

typedef struct ss_curriculum_term {
    int32_t func;
    int32_t term;
    double p0;
    double p1;
} ss_curriculum_term;

/* Everything the fused step needs: passed BY VALUE as the kernel parameter
 * (a __grid_constant__ struct, read through the constant bank). */
typedef struct ss_env_desc {
    int32_t abi_version;
    int32_t n_worlds;
    int32_t decimation;
    int32_t max_episode_steps;
    double dt_control;
    ss_model model;
    ss_terrain terrain;
    ss_state state;
    ss_field field[SS_DCAP_FIELDS];
    ss_rng rng;
    /* default state (entity.py:91-105, env.py:121-135) and spawn */
    double base_pose[3];
    double base_vel[3];
    double joint_pos[SS_DCAP_JOINTS];
    double joint_vel[SS_DCAP_JOINTS];
    double spawn_offset;
    /* actions */
    int32_t n_action_terms;
    int32_t action_dim;
    ss_action_term action_term[SS_DCAP_ACTION_TERMS];
    double* action;
    double* prev_action;
    double* targets;
    int32_t n_actuators;
    int32_t pad1;
    ss_actuator actuator[SS_DCAP_ACTUATORS];
    /* capture ring (capture.py:41-59), physical capacity capture_phys */
    int32_t capture_phys;
    int32_t pad2;
    double* cap_q;
    double* cap_qd;
    double* cap_ctrl;
    /* contact sensor (sensors.py:55-118) */
    int32_t hist_len;
    int32_t pad3;
    uint8_t* s_in_contact;
    double* s_normal;
    double* s_tangent;
    double* s_force_hist;
    double* s_cur_air;
    double* s_last_air;
    double* s_cur_contact;
    int64_t* s_last_td;
    /* ray scanner (sensors.py:20-46) */
    int32_t n_rays;
    int32_t pad4;
    double ray_offset[SS_DCAP_RAYS];
    /* terminations (managers/termination.py) */
    int32_t n_terms;
    int32_t pad5;
    ss_term_term term[SS_DCAP_TERMINATIONS];
    uint8_t* terminated;
    uint8_t* truncated;
    uint8_t* nonfinite;
    int64_t* trigger_counts;
    uint32_t* nf_flags;
    /* rewards (managers/reward.py) */
    int32_t n_rewards;
    int32_t pad6;
    ss_reward_term reward[SS_DCAP_REWARDS];
    double* reward_out;
    double* ep_sums;
    double* ep_raw;
    double* last_values;
    double* finalized;
    /* commands (managers/command.py) */
    int32_t n_cmd;
    int32_t period_steps;
    int32_t cmd_slot;
    int32_t pad7;
    double cap_scale;
    double init_lo[SS_DCAP_CMD];
    double init_hi[SS_DCAP_CMD];
    double* command;
    double* ranges;
    int64_t* countdown;
    /* events + curriculum */
    int32_t n_events;
    int32_t n_curriculum;
    ss_event_term event[SS_DCAP_EVENTS];
    ss_curriculum_term curriculum[SS_DCAP_CURRICULUM];
    /* episode bookkeeping (env.py:146-151) */
    int64_t* episode_steps;
    double* episode_start_x;
    double* commanded_distance;
    int64_t* terrain_rows;
    int64_t* terrain_cols;
    double* prev_lin_vel_b;
    /* observations */
    int32_t n_groups;
    int32_t n_obs_terms;
    ss_obs_group group[SS_DCAP_GROUPS];
    ss_obs_term obs[SS_DCAP_OBS_TERMS];
    uint32_t* obs_bad;
    /* optional clock64() phase probes of world 0 (JIT builds with -DSS_PROBES) */
    int64_t* probe;
    /* host mirror of the output arena (obs groups, reward, terminated,
     * truncated): when nonzero, every output store is repeated at
     * address + out_mirror, a mapped pinned host buffer, so the step's results
     * cross PCIe from the kernel itself (no separate device->host copy) */
    int64_t out_mirror;
} ss_env_desc;

/* Per-launch uniform values, all host-tracked (no device round trip). */
typedef struct ss_uniforms {
    uint32_t stages;
    int32_t nsub;
    uint32_t flags;
    int32_t nf_slot;
    int64_t global_step;
    int64_t sim_step;
    int32_t capture_slot0;
    uint32_t sensor_mask;
    uint32_t groups_mask;
    int32_t any_pending;
    int32_t act_head0[SS_MAX_ACTUATORS];
    int32_t obs_delay_head[SS_MAX_OBS_TERMS];
    int32_t obs_hist_head[SS_MAX_OBS_TERMS];
    double weight[SS_MAX_REWARDS];
    const double* actions;
    const uint8_t* reset_mask;
    /* fused random policy (policies.py:14-16): policy_slot >= 0 makes the
     * ACTION stage draw U[policy_lo, policy_hi) from that stream slot instead
     * of reading `actions` */
    int32_t policy_slot;
    int32_t policy_pad;
    double policy_lo;
    double policy_hi;
    /* non-NULL: this launch also reduces the job statistics of metrics.build_record
     * (metrics.py:31-45) over its worlds, fused into the step's tail, into stats_out
     * (the ss_stats_pack layout); stats_partials holds gridDim x SS_STATS_MAXV doubles,
     * stats_ticket one zeroed uint32 the kernel resets */
    double* stats_out;
    double* stats_partials;
    uint32_t* stats_ticket;
    int32_t stats_rows;
    int32_t stats_pad;
} ss_uniforms;

/* Host-side runtime state of one env: every per-launch uniform (step
 * counters, ring heads, reward weights) is derived and advanced here by
 * ss_rt_launch, so a control step costs the host one C call. The struct is
 * shared memory between Python (ctypes) and C: Python reads the counters
 * directly, C advances them. */
#define SS_RT_SLOTS 8
typedef struct ss_rt_state {
    int64_t global_step;
    int64_t sim_step;
    int64_t cap_pushes;
    int64_t* cap_sim_steps;
    int32_t cap_count;
    int32_t cap_capacity;
    int32_t cap_phys;
    int32_t n_act;
    int64_t sensor_last_update;
    int32_t act_head[SS_MAX_ACTUATORS];
    int32_t act_cap[SS_MAX_ACTUATORS];
    int32_t n_obs;
    int32_t n_groups;
    int32_t obs_group[SS_MAX_OBS_TERMS];
    int32_t obs_delay_head[SS_MAX_OBS_TERMS];
    int32_t obs_delay_len[SS_MAX_OBS_TERMS];
    int32_t obs_hist_head[SS_MAX_OBS_TERMS];
    int32_t obs_hist_len[SS_MAX_OBS_TERMS];
    int32_t any_pending;
    int32_t n_rewards;
    double weight[SS_MAX_REWARDS];
    uint32_t* nf_flags;
    int32_t nf_slots;
    int32_t nf_slot;
    int32_t nf_head;
    int32_t nf_pending;
    int64_t nf_pushes[SS_RT_SLOTS];
    int64_t nf_sim_step[SS_RT_SLOTS];
    int32_t nf_count[SS_RT_SLOTS];
    uint64_t nf_event[SS_RT_SLOTS];
    int64_t launches;
    /* slots retired by the poll folded into the last ss_rt_launch that were
     * flagged nonfinite (ss_launch.poll_keep >= 0) */
    int32_t nf_ready_n;
    int32_t nf_ready[SS_RT_SLOTS];
} ss_rt_state;

/* One launch request for ss_rt_launch. */
typedef struct ss_launch {
    uint32_t stages;
    int32_t nsub;
    uint32_t flags;
    uint32_t groups_mask;
    const double* actions;
    const uint8_t* reset_mask;
    int32_t policy_slot;
    /* >= 0: retire nonfinite slots first (ss_rt_poll with this keep), results
     * in ss_rt_state.nf_ready -- one host call per step instead of two */
    int32_t poll_keep;
    double policy_lo;
    double policy_hi;
    /* the descriptor packed with the specialized kernel's SS_DCAP_* bounds
     * (NULL: the kernel takes the full ss_env_desc); its size in bytes */
    const void* jit_desc;
    int64_t jit_desc_bytes;
    /* fused statistics of this step (see ss_uniforms.stats_out); NULL: none */
    double* stats_out;
    double* stats_partials;
    uint32_t* stats_ticket;
    int32_t stats_rows;
    int32_t stats_pad;
} ss_launch;

/* One draw call of StreamPack.uniform/normal (rng.py:69-119). sel == NULL
 * means all N streams; otherwise n_sel world indices (int64). lo/hi are
 * broadcast per `lohi_mode`: 0 scalar, 1 per selected row (n_sel), 2 per
 * (row, dim) element. out is row-major (n_sel, dim). */
typedef struct ss_rng_draw_args {
    int32_t kind;
    int32_t dim;
    int32_t lohi_mode;
    int32_t n_sel;
    uint64_t base;
    int64_t world_id_offset;
    uint64_t* counter;
    const int64_t* sel;
    double lo;
    double hi;
    const double* lo_arr;
    const double* hi_arr;
    double* out;
} ss_rng_draw_args;

/* One log interval's statistics of this rank packed into ONE float64 vector
 * (metrics.build_record, metrics.py:31-45), ready for a single all-reduce:
 *   out = [n_worlds, sum(reward), sum(ep_sums[t]) for t < n_rewards,
 *          trigger_counts[c] for c < n_counts, histogram(terrain_rows)[r] for r < n_rows,
 *          sum(nonfinite)]            (length 3 + n_rewards + n_counts + n_rows)
 * One launch: every block reduces a fixed stride of worlds in a fixed order
 * into `partials` (grid x SS_STATS_MAXV doubles), the last block to finish
 * (ticket) sums the partials in block order -- deterministic for a given N.
 * `ticket` is one zero-initialised uint32 the kernel resets itself. */
#define SS_STATS_MAXV 64
#define SS_STATS_GRID 148
typedef struct ss_stats_args {
    int32_t n_worlds;
    int32_t n_rewards;
    int32_t n_counts;
    int32_t n_rows;
    const double* reward;
    const double* ep_sums;
    const int64_t* trigger_counts;
    const int64_t* terrain_rows;
    const uint8_t* nonfinite;
    double* partials;
    uint32_t* ticket;
    double* out;
} ss_stats_args;

#ifndef __CUDACC_RTC__ /* host entry points (not part of the JIT translation unit) */
int ss_abi_version(void);
size_t ss_sizeof(int which); /* 0 env_desc, 1 uniforms, 2 rng_draw_args, 3 rt_state, 4 launch, 5 stats_args */
const char* ss_last_error(void);

int ss_env_step(const ss_env_desc* desc, const ss_uniforms* u, void* stream);
int ss_rng_draw(const ss_rng_draw_args* args, void* stream);
int ss_fk(const ss_env_desc* desc, const double* q, double* thetas, double* attach,
          double* tips, int32_t n, void* stream);
int ss_heights(const ss_terrain* terrain, const double* x, double* out, int64_t n,
               void* stream);
int ss_randomize(const ss_env_desc* desc, int32_t field, int32_t distribution,
                 double r0, double r1, int32_t operation, int32_t slot,
                 const int64_t* sel, int32_t n_sel, void* stream);
/* Per-env specialization: NVRTC-compile the step body with the env's term
 * tables as compile-time constants (csrc/ss_cfg.cuh), load it, launch it.
 * Same semantics and results as ss_env_step. */
int ss_jit_compile(const char* src, const char* name, int n_headers, const char* const* header_src,
                   const char* const* header_names, int n_opts, const char* const* opts,
                   void* out, size_t* size, char* log, size_t log_size);
int ss_jit_load(const void* cubin, size_t size, const char* kernel_name, int block, void** handle);
int ss_jit_unload(void* handle);
int ss_env_step_jit(void* handle, const ss_env_desc* desc, const ss_uniforms* u, void* stream);
/* A module compiled with SS_DCAP_* bounds takes the packed descriptor:
 * declare its size once, then launch with the full descriptor (validated)
 * plus the packed copy that becomes the kernel parameter block. */
int ss_jit_set_desc_bytes(void* handle, int64_t bytes);
/* Dynamic shared memory per block of a module whose staging buffers exceed the static 48 KB. */
int ss_jit_set_smem(void* handle, int32_t bytes);
int ss_env_step_jit_packed(void* handle, const ss_env_desc* desc, const void* packed, int64_t packed_bytes,
                           const ss_uniforms* u, void* stream);
/* Runtime: derive the uniforms from *st, launch (JIT module when jit != NULL,
 * else the generic kernel), advance *st. ss_rt_poll retires completed TERM
 * launches (blocking on the oldest while more than `keep` are pending) and
 * returns the slots whose nonfinite flag was raised; ss_rt_release frees the
 * runtime's CUDA events. */
int ss_rt_launch(const ss_env_desc* desc, ss_rt_state* st, const ss_launch* l, void* jit, void* stream);
int ss_rt_poll(ss_rt_state* st, int32_t keep, int32_t* out_slots, int32_t max_out);
int ss_rt_release(ss_rt_state* st);

/* Pipelined host I/O for env.step_async / env.step_wait (gym VectorEnv style), nslot in [2, 8] slots:
 * ss_pipe_pre copies a step's actions from pinned host memory into the slot's device buffer on a
 * copy stream (the launching stream waits for it) and returns the slot; ss_pipe_post snapshots the
 * output arena into the slot's staging buffer (SM copy kernel) and copies it to a pinned host block
 * on a second copy stream, so the PCIe transfers of one step overlap the kernel of the next;
 * ss_pipe_wait blocks until the oldest pending step's results are in host memory and returns the
 * index of its host block. `host` holds nhost (nslot < nhost <= 10) blocks used round-robin: the block
 * step_wait returned is not written again before the following ss_pipe_wait call. When the staging
 * buffers and host blocks of an even step and the next are contiguous, the two results cross PCIe as
 * one copy (issued by the next step's ss_pipe_post, or by ss_pipe_wait alone if it comes first).
 * Buffers are owned by the caller (16-byte aligned). */
int ss_pipe_create(int32_t nslot, int32_t nhost, void* const* dev_actions, void* const* stage, void* const* host,
                   int64_t action_bytes, int64_t arena_bytes, void** out);
int ss_pipe_destroy(void* pipe);
int ss_pipe_pre(void* pipe, const void* host_actions, void* main_stream);
int ss_pipe_post(void* pipe, const void* arena, void* main_stream);
int ss_pipe_wait(void* pipe);
int ss_stats_pack(const ss_stats_args* args, void* stream);
int ss_actuator_eval(int32_t kind, const double* kp, const double* kd, double effort,
                     double saturation, double vel_limit, const double* q_des,
                     const double* q, const double* qd, double* out, int64_t n,
                     void* stream);
#endif /* __CUDACC_RTC__ */

#ifdef __cplusplus
}
#endif

#endif /* STRIDESIM_B200_H */
