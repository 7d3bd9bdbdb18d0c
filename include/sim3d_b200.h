/* sim3d_b200.h -- C-ABI of the 3-D articulated-body path.
 *
 * The reference (stridesim) is planar and has no 3-D engine; in
 * mjlab this path is MuJoCo Warp's mjwarp.step over an MjModel/MjData pair
 * (PAPER.md:111-118, 171-177). These entry points are what a host binding of
 * that step would call: plain pointers and sizes, everything asynchronous on
 * the given CUDA stream, no allocation inside. Arrays are device pointers,
 * row-major with the world index outermost ((N, nq) qpos, (N, nv) qvel ...),
 * in the element type selected by `dtype` (S3_F64 or S3_F32); the model
 * tables are packed by the host in the same element type.
 *
 * Style: one field per line (paper_2601_22074_b200/sim3d/native.py parses
 * the structs into ctypes; s3_sizeof cross-checks them).
 */
#ifndef SIM3D_B200_H
#define SIM3D_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define S3_ABI_VERSION 21
#define S3_F64 0
#define S3_F32 1

#define S3_MAX_NV 64
#define S3_MAX_NBODY 64
#define S3_MAX_CHAIN 32
#define S3_MAX_CON 16
#define S3_MAX_LIM 32
#define S3_MAX_ROWS 96
#define S3_MAX_RAYS 128
#define S3_MAX_TREE 4
#define S3_MAX_TRACK 16 /* tracked bodies of the motion task (besides the anchor) */
#define S3_MAX_SENSOR 4 /* contact sensors */
#define S3_MAX_KERNEL 8 /* adaptive-sampling smoothing kernel length */
#define S3_BODY_STATE 13 /* pos[3] quat[4] linvel[3] angvel[3] (world frame; linvel of the body origin) */

#define S3_OK 0
#define S3_ERR_ARG 1
#define S3_ERR_CUDA 2
#define S3_ERR_BOUNDS 3

/* Model tables (device pointers). Float tables hold `dtype` elements. */
typedef struct s3_model {
    int32_t dtype;
    int32_t nbody;
    int32_t njnt;
    int32_t nq;
    int32_t nv;
    int32_t ngeom;
    int32_t npair;
    int32_t nu;
    int32_t nlimjnt;
    int32_t nlevel;
    int32_t chain_stride;
    int32_t terrain_hfield;
    int32_t hf_nrow;
    int32_t hf_ncol;
    int32_t iterations;
    int32_t ls_iterations;
    int32_t nldl_norm;
    int32_t ntree;
    int32_t flags; /* bit 0: refactor every dof in each Newton iteration (A/B of the partial refactorization);
                      bit 1: tree-level schedule of the factorization / solves from CSR tables (measured
                      slower; kept for A/B); bit 2: tree-level schedule driven by per-lane dof bit masks;
                      bit 3: block barrier at the start of each substep; bit 4: before the Newton solve;
                      bit 5: after it (bits 3-5: full blocks only); bit 6: balance warps per block over
                      the waves of a launch (the Python layer sets 40, plus 64 for models with nv >= 24);
                      bit 7: conjugate-gradient solver instead of Newton (Opt.solver = "cg"; plan the layout
                      with it set: the solver keeps two extra vectors per world) */
    int32_t nhlev;
    int32_t ndlev;
    int32_t nkintree; /* kinematic trees (robot, free objects) */
    int32_t ncon_max; /* contact capacity per world (<= S3_MAX_CON); later contacts are dropped and counted */
    int32_t pad4;
    uint64_t nonroot_mask; /* dofs with a parent dof */
    uint64_t nonleaf_mask; /* dofs with a child dof */
    double timestep;
    double gravity[3];
    double tolerance;
    double ls_tolerance;
    double solref[2];
    double solimp[5];
    double scale;
    double total_mass;
    double hf_spacing;
    double hf_origin[2];
    double hf_max;
    /* bodies */
    const int32_t* body_parentid;
    const int32_t* body_jntadr;
    const int32_t* body_jntnum;
    const int32_t* body_dofadr;
    const int32_t* body_dofnum;
    const uint64_t* body_dofmask;
    const int32_t* level_ptr;
    const int32_t* level_body;
    const int32_t* child_ptr;
    const int32_t* child_idx;
    const void* body_pos;
    const void* body_quat;
    const void* body_ipos;
    const void* body_ilmat;
    const void* body_mass;
    const void* body_inertia;
    const void* body_invweight0;
    const int32_t* body_treeid; /* kinematic tree of each body (each tree's subtree com is its c-frame) */
    const void* tree_mass;
    /* joints */
    const int32_t* jnt_type;
    const int32_t* jnt_qposadr;
    const int32_t* jnt_dofadr;
    const void* jnt_pos;
    const void* jnt_axis;
    const void* qpos0;
    /* dofs */
    const int32_t* dof_bodyid;
    const int32_t* dof_parentid;
    const uint64_t* dof_descmask;
    const uint8_t* dof_chain;
    const int32_t* dof_chainlen;
    const void* dof_damping;
    const void* dof_armature;
    const void* dof_invweight0;
    /* limited joints */
    const int32_t* lim_qposadr;
    const int32_t* lim_dofadr;
    const void* lim_range;
    /* geoms */
    const int32_t* geom_type;
    const int32_t* geom_bodyid;
    const void* geom_pos;
    const void* geom_lmat;
    const void* geom_size;
    const void* geom_friction;
    const void* geom_rbound;
    /* collision pairs */
    const int32_t* pair_geom;
    const uint8_t* pair_chain;
    const int32_t* pair_chainlen;
    const uint8_t* pair_condim; /* 1: frictionless (mu = 0, its 4 pyramid rows at 1/4 the normal stiffness each,
                                   i.e. MuJoCo's single normal row), 3: pyramidal sliding friction */
    /* actuators */
    const int32_t* act_dofadr;
    const int32_t* act_qposadr;
    const int32_t* act_kind;
    const void* act_gain;
    /* derived tables: per-dof (i, j) update lists of the tree-sparse factorization (ldl_ptr[nv+1],
     * ldl_pair = i << 8 | j), Jacobian class per pair (pairs with identical column lists), 1 when a
     * pair's J^T J keeps the tree sparsity pattern, and the (a, b) decode of packed-lower index t */
    const int32_t* ldl_ptr;
    const uint16_t* ldl_pair;
    const uint16_t* ldl_norm;
    const uint16_t* tree_ent;
    const uint64_t* dof_chainmask;
    const uint64_t* pair_dofmask;
    /* level schedules: per height level the factorization's (i, j) entries (fl_ent = i << 8 | j) with
     * the eliminated dofs k contributing to each (fl_k, CSR by fl_kptr), and the leaf-to-root solve's
     * target ancestors (bl_ent) with their contributing dofs (bl_i, CSR by bl_iptr); per depth level
     * the dofs of the root-to-leaf solve (fw_dof, CSR by fw_ptr) */
    const int32_t* fl_ptr;
    const uint16_t* fl_ent;
    const int32_t* fl_kptr;
    const uint8_t* fl_k;
    const int32_t* bl_ptr;
    const uint8_t* bl_ent;
    const int32_t* bl_iptr;
    const uint8_t* bl_i;
    const int32_t* fw_ptr;
    const uint8_t* fw_dof;
    const uint64_t* hlev_mask; /* dof bit mask of each height level */
    const uint64_t* dlev_mask; /* dof bit mask of each depth level */
    const int32_t* pair_class;
    const int32_t* pair_tree;
    const uint16_t* tri_tab;
    /* heightfield samples (hf_nrow, hf_ncol) */
    const void* hfield;
} s3_model;

/* Per-world state and optional per-substep outputs (NULL = not written). */
typedef struct s3_data {
    int64_t nworld;
    void* qpos;
    void* qvel;
    void* ctrl;
    void* qacc_warmstart;
    void* qfrc_applied;
    void* time;
    void* friction_scale; /* (N,) per-world friction multiplier (domain randomisation), NULL = 1 */
    void* mass_scale;     /* (N,) per-world scale of body 1's mass and inertia, NULL = 1 */
    /* outputs of the LAST substep of a launch (for parity tests / sensors) */
    void* xpos;
    void* xquat;
    void* com; /* (N, S3_MAX_TREE, 3) subtree com per kinematic tree */
    void* cdof;
    void* qM;
    void* qLD;
    void* qfrc_bias;
    void* qfrc_smooth;
    void* qacc_smooth;
    void* qacc;
    void* qfrc_constraint;
    void* geom_xpos;
    void* geom_xmat;
    int32_t* ncon;
    int32_t* ndropped;
    int32_t* nefc;
    int32_t* con_pair;
    void* con_dist;
    void* con_pos;
    void* con_frame;
    void* efc_force;
    int32_t* solver_niter;
} s3_data;

/* Workspace layout: offsets (in elements) inside one world's shared-memory block. */
typedef struct s3_layout {
    int32_t warps_per_block;
    int32_t elems_per_world;
    int32_t bytes_per_block;
    int32_t off[40];
} s3_layout;

/* Fused velocity-tracking task (paper_2601_22074_b200/sim3d/task.py): configuration + per-world
 * task state (device pointers, `dtype` elements unless noted). */
typedef struct s3_task {
    int32_t kind; /* 0 velocity tracking, 1 motion imitation (reference-motion command), 2 cube lift */
    int32_t decimation;
    int32_t episode_steps;
    int32_t cmd_resample_steps;
    int32_t obs_dim;
    int32_t nscan;
    int32_t nframes;
    int32_t pad0;
    uint64_t seed;
    int64_t world_offset;
    double action_scale;
    double action_clip;
    double track_sigma;
    double min_height;
    double max_tilt_cos;
    double reset_joint_jitter;
    double spawn_half_extent;
    double cmd_lo[3];
    double cmd_hi[3];
    double reward_weights[10];
    double noise[7];
    double scan_xy[256];
    double scan_offset;
    double scan_noise;
    double frame_dt;
    double motion_sigmas[8];
    double max_height_error;
    double max_ori_error;
    double motion_start_frac;
    /* motion kind, BeyondMimic's relative body terms: the anchor body and the tracked bodies; the clip's
     * body states (S3_BODY_STATE per body, anchor first) come from s3_motion_bodies */
    int32_t anchor_body;
    int32_t ntrack;
    int32_t track_body[S3_MAX_TRACK];
    /* contact sensors (every kind): bit s of pair_sensor[p] makes the contacts of collision pair p count
     * toward sensor s; sensor[w * nsensor + s] = the most such contacts any substep of the control step saw */
    int32_t nsensor;
    int32_t nfeet; /* velocity kind: sensors 0..nfeet-1 are the feet's ground contacts (foot-slip term) */
    int32_t foot_body[S3_MAX_SENSOR];
    const uint8_t* pair_sensor; /* (npair,) */
    void* sensor;               /* (N, nsensor) */
    const void* motion_body;    /* (nframes, 1 + ntrack, S3_BODY_STATE) */
    /* motion kind, BeyondMimic's adaptive sampling of the start time (nbins = 0: uniform over the first
     * motion_start_frac of the clip): each termination counts in the clip bin of its motion time
     * (bin_fail_now, uint32 atomics); the last block of the launch folds the counts into an exponential
     * average bin_failed = alpha now + (1 - alpha) bin_failed, adds uniform_ratio / nbins, smooths
     * forward with the kernel weights (q_b = sum_i w_i p_min(b + i, nbins - 1)) and writes the cumulative
     * sums bin_cum that the NEXT launch's resets sample a bin from (a uniform time inside it) */
    int32_t nbins;
    int32_t nkernel;
    double adaptive_alpha;
    double adaptive_uniform;
    double adaptive_kernel[S3_MAX_KERNEL];
    void* bin_failed;       /* (nbins,) */
    void* bin_cum;          /* (nbins,) */
    uint32_t* bin_fail_now; /* (nbins,) */
    uint32_t* bin_ticket;   /* (1,) */
    int32_t cube_qposadr;
    int32_t tip_geom[2];
    int32_t pad2;
    double cube_half;
    double reach_std;
    double goal_std;
    double lift_height;
    double min_cube_z;
    double cube_x[2];
    double cube_y[2];
    int32_t events; /* velocity kind: 1 = startup friction randomisation + interval pushes */
    int32_t pad3;
    double friction_range[2];
    double base_mass_range[2];
    double push_interval[2];
    double push_velocity;
    void* event_timer; /* (N,) time to the next push */
    int32_t curriculum; /* velocity kind: 1 = terrain levels on a rows x cols patch grid */
    int32_t terrain_rows;
    int32_t terrain_cols;
    int32_t curriculum_max_init_level;
    double patch_size;
    double curriculum_promote;
    double curriculum_demote;
    int32_t* terrain_level; /* (N,) */
    void* spawn_xy;         /* (N, 2) */
    void* cmd_dist;         /* (N,) commanded distance of the running episode */
    const void* motion_qpos; /* (nframes, nq) */
    const void* motion_qvel; /* (nframes, nv) */
    const void* default_qpos;
    void* action;
    void* prev_action;
    void* command;
    int32_t* cmd_timer;
    int32_t* episode_step;
    void* episode_return;
    void* obs;
    void* reward;
    uint8_t* terminated;
    uint8_t* truncated;
    /* optional cost-ordered scheduling (both or neither): the step writes each world's solver cost (Newton
     * iterations summed over its substeps) to cost[N]; the next step first sorts the worlds by it (heaviest
     * first) into order[N] and block b's warps take worlds order[b * warps_per_block + i], so each block's
     * worlds need similar solver work and the block's barriers wait less. Results do not depend on it. */
    int32_t* cost;
    int32_t* order;
} s3_task;

int s3_abi_version(void);
size_t s3_sizeof(int which); /* 0 model, 1 data, 2 layout, 3 task */
const char* s3_last_error(void);

/* Fill the shared-memory layout for this model; warps_per_block = 0 picks the largest
 * count that fits the per-block shared-memory limit. */
int s3_plan(const s3_model* m, int32_t warps_per_block, s3_layout* out);

/* `nsub` physics substeps of every world (mj_step x nsub: kinematics, com, CRB + L^T D L,
 * RNE, actuation, collision, constraints, Newton, implicitfast), ctrl held fixed.
 * Replaces, for the 3-D path, StepPipeline.substep x decimation (sim/physics.py:239-249,
 * env.py:228-233 of the reference; mjwarp.step in mjlab).
 * s3_step and s3_env_step upload *m to the library's constant-memory model slot (one per device) on
 * `stream` before their kernel. The library serializes the slot itself: a launch from another stream than
 * the previous launch waits on the GPU for that launch's kernels before the slot changes, an identical
 * model on the same stream skips the upload, and concurrent host threads take a per-device lock, so
 * different models / dtypes / streams may be mixed freely (at the price of serializing their kernels). */
int s3_step(const s3_model* m, const s3_data* d, const s3_layout* l, int32_t nsub, void* stream);

/* One control step of the fused task (mode 0; kind velocity or motion): ActionManager.process -> decimation x
 * substep -> terminations -> rewards -> masked reset + command resample -> command countdown ->
 * observations, every world in ONE launch (env.py:219-259 of the reference, on the 3-D model).
 * mode 1 resets every world (counter 0 draws) and writes the first observation; actions unused. */
int s3_env_step(const s3_model* m, const s3_data* d, const s3_layout* l, const s3_task* t, const void* actions,
                int32_t mode, int64_t global_step, void* stream);

/* Body states of a motion clip (the per-frame body_pos_w / body_quat_w / body_lin_vel_w / body_ang_vel_w a
 * BeyondMimic motion file carries): for each of t->nframes frames of t->motion_qpos / t->motion_qvel, forward
 * kinematics + the dof motion vectors of that frame, then for the anchor body and each tracked body its
 * world position, orientation, origin linear velocity and angular velocity, written to
 * out[(f * (1 + ntrack) + k) * S3_BODY_STATE ...] (k = 0 the anchor). One warp per frame. The motion kind
 * of s3_env_step reads the table through t->motion_body. */
int s3_motion_bodies(const s3_model* m, const s3_layout* l, const s3_task* t, void* out, void* stream);

/* Ray casting against every geom of each world (frames from s3_step / s3_env_step geom outputs):
 * nearest hit distance along o + t d (|d| = 1, t <= max_dist), -1 and geom -1 on a miss; geoms on
 * `exclude_body` are skipped. Height scanners pass vertical rays; s3_depth builds pinhole rays of a
 * camera fixed to geom `cam_geom` (forward +x, right -y, up +z of the geom frame, vertical field of
 * view `fovy` radians) and writes an (N, height, width) range image. Replaces, for the 3-D path,
 * RayScanner.read (sensors.py:26-46 of the reference; mjlab's RayCastSensor / depth camera). */
int s3_raycast(const s3_model* m, const void* geom_xpos, const void* geom_xmat, int64_t nworld, int32_t nray,
               const void* origin, const void* dir, double max_dist, int32_t exclude_body, void* dist, int32_t* geom,
               void* stream);
int s3_depth(const s3_model* m, const void* geom_xpos, const void* geom_xmat, int64_t nworld, int32_t cam_geom,
             const double* offset, int32_t width, int32_t height, double fovy, double max_dist, int32_t exclude_body,
             void* dist, int32_t* geom, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* SIM3D_B200_H */
