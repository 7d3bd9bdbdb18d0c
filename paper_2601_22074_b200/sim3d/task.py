"""Velocity-tracking task on the 3-D path, fused into one kernel launch per control step.

The reference's manager pipeline (env.py:219-259) -- ActionManager.process ->
decimation x (actuators + physics substep) -> TerminationManager ->
RewardManager -> masked reset (+ CommandManager.resample) ->
CommandManager.update -> ObservationManager -- run for the 3-D model with
mjlab's velocity-tracking terms (§6.1): exp-kernel tracking of the
commanded planar velocity and yaw rate, vertical-velocity / roll-pitch-rate /
action-rate / flat-orientation penalties, fall and tilt terminations, a
time-out truncation, masked reset with joint jitter and random yaw, and
uniformly resampled (vx, vy, wz) commands. Every stochastic draw is a
counter-based splitmix64 word keyed by (seed, global world id, purpose), the
construction of the reference's rng.py, so worlds are partition-independent.

``VelocityEnv3D`` is the batched env: ``reset()`` and ``step(actions)``
return device tensors (obs (N, D), reward (N,), terminated (N,), truncated
(N,)); the whole control step is ONE launch of ``s3_env_step``.
"""

from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass, field

import numpy as np
import torch

from . import native as N
from .device import Data, DeviceModel
from .model import Model

PURPOSE_RESET, PURPOSE_COMMAND, PURPOSE_OBS = 1, 2, 3

# BeyondMimic's tracked bodies on the G1 (the anchor is the torso); models without these names track every
# body of the first kinematic tree (up to S3_MAX_TRACK) about its root
BEYONDMIMIC_ANCHOR = "torso_link"
BEYONDMIMIC_BODIES = ("pelvis", "left_hip_roll_link", "left_knee_link", "left_ankle_roll_link", "right_hip_roll_link",
                      "right_knee_link", "right_ankle_roll_link", "torso_link", "left_shoulder_roll_link",
                      "left_elbow_link", "left_wrist_yaw_link", "right_shoulder_roll_link", "right_elbow_link",
                      "right_wrist_yaw_link")


def robot_geoms(m: Model, tree: int = 0) -> tuple:
    """Geoms on the bodies of kinematic tree ``tree`` (not the terrain)."""
    return tuple(g for g in range(m.ngeom) if m.geom_bodyid[g] > 0 and m.body_treeid[m.geom_bodyid[g]] == tree)


def pair_sensor_bits(m: Model, sensors) -> np.ndarray:
    """s3_task.pair_sensor: bit s of entry p is set when collision pair p is a contact of sensor s, i.e. one
    geom of the pair is in the sensor's first set and the other in its second set (None: any geom)."""
    bits = np.zeros(max(m.npair, 1), dtype=np.uint8)
    for s, (_, a, b) in enumerate(sensors):
        a = set(a)
        b = None if b is None else set(b)
        for p, (g1, g2) in enumerate(m.pair_geom):
            if (g1 in a and (b is None or g2 in b)) or (g2 in a and (b is None or g1 in b)):
                bits[p] |= np.uint8(1 << s)
    return bits


def fold_bins(failed: np.ndarray, now: np.ndarray, cfg) -> tuple:
    """Adaptive sampling's fold (s3_kernel.cu adaptive_fold, in the same order): failed <- alpha now +
    (1 - alpha) failed; cumulative sums of q_b = sum_i w_i (failed_min(b + i, nb - 1) + uniform / nb)."""
    nb = len(failed)
    a = cfg.adaptive_alpha
    failed = np.array([a * float(now[b]) + (1.0 - a) * failed[b] for b in range(nb)])
    u = cfg.adaptive_uniform_ratio / nb
    w = cfg.kernel_weights()
    cum, acc = np.zeros(nb), 0.0
    for b in range(nb):
        q = 0.0
        for i in range(len(w)):
            q += w[i] * (failed[min(b + i, nb - 1)] + u)
        acc += q
        cum[b] = acc
    return failed, cum


def padded(v, n: int) -> tuple:
    """A reward-weight / sigma tuple padded with zeros to the struct's length."""
    v = tuple(v)
    if len(v) > n:
        raise ValueError(f"at most {n} values")
    return v + (0.0,) * (n - len(v))


@dataclass
class VelocityTaskCfg:
    default_qpos: np.ndarray
    decimation: int = 4
    action_scale: float = 0.25
    action_clip: float = 2.0
    episode_steps: int = 1000          # 20 s at 50 Hz
    command_resample_steps: int = 500  # 10 s
    command_ranges: tuple = ((-1.0, 1.0), (-0.5, 0.5), (-1.0, 1.0))
    track_sigma: float = 0.25
    # track_lin_vel_xy_exp, track_ang_vel_z_exp, lin_vel_z_l2, ang_vel_xy_l2, action_rate_l2, flat_orientation_l2,
    # angular_momentum_l2 (robot's centroidal angular momentum), joint_pos_limits (distance outside the ranges),
    # foot_slip (squared horizontal velocity of the feet in ground contact) -- PAPER.md §6.1's penalty set
    reward_weights: tuple = (1.0, 0.5, -2.0, -0.05, -0.01, -1.0, -0.02, -1.0, -0.1)
    min_height: float = 0.3
    max_tilt_cos: float = -0.5         # terminate when projected gravity z > -cos(60 deg)
    reset_joint_jitter: float = 0.1
    spawn_half_extent: float = 0.5
    noise: tuple = (0.1, 0.2, 0.05, 0.0, 0.01, 1.5, 0.0)  # lin vel, ang vel, gravity, command, qpos, qvel, action
    height_scan: bool = False
    scan_size: tuple = (1.6, 1.0)
    scan_resolution: float = 0.2
    scan_offset: float = 0.5
    scan_noise: float = 0.02
    # domain randomisation (EventManager analog): startup per-world friction scale; interval pushes that
    # add U(-v, v) to the base's planar velocity every U(push_interval) seconds. None disables pushes.
    friction_range: tuple = (0.6, 1.2)
    base_mass_range: tuple = (0.8, 1.2)  # startup scale of the base body's mass and inertia
    push_interval: tuple | None = (10.0, 15.0)
    push_velocity: float = 0.5
    # terrain curriculum (robots.curriculum_heightfield): None disables. Worlds spawn at the centre of their
    # (level row, world_id % cols) patch; at episode end a world walked farther than promote x its commanded
    # distance moves one row up, less than demote x down (the planar reference's terrain_levels rule).
    curriculum: tuple | None = None    # (rows, cols, patch metres)
    curriculum_max_init_level: int = 1
    curriculum_promote: float = 0.8
    curriculum_demote: float = 0.4
    # feet (body names; None: the *ankle_roll_link / *_calf bodies): each gets a ground-contact sensor (the
    # first sensors), read by the foot-slip term
    feet: tuple | None = None
    # contact sensors (ContactSensor analog): (name, geoms, other geoms or None for any), at most
    # S3_MAX_SENSOR with the feet's; env.sensor[w, s] = the most contacts of sensor s in one substep of the
    # control step
    contact_sensors: tuple = ()

    def foot_bodies(self, m: Model) -> tuple:
        if self.feet is not None:
            return tuple(m.body_names.index(b) if isinstance(b, str) else int(b) for b in self.feet)
        return tuple(b for b, nm in enumerate(m.body_names) if nm.endswith("ankle_roll_link") or nm.endswith("_calf"))

    def sensors(self, m: Model) -> tuple:
        feet = tuple((f"{m.body_names[b]}_ground", tuple(g for g in range(m.ngeom) if m.geom_bodyid[g] == b), (0,))
                     for b in self.foot_bodies(m))
        return feet + tuple(self.contact_sensors)

    def scan_points(self):
        nx = int(round(self.scan_size[0] / self.scan_resolution)) + 1
        ny = int(round(self.scan_size[1] / self.scan_resolution)) + 1
        xs = (np.arange(nx) - (nx - 1) / 2) * self.scan_resolution
        ys = (np.arange(ny) - (ny - 1) / 2) * self.scan_resolution
        return [(x, y) for y in ys for x in xs]

    def obs_dim(self, m: Model) -> int:
        return 12 + 3 * m.nu + (len(self.scan_points()) if self.height_scan else 0)

    def noise_vector(self, m: Model) -> np.ndarray:
        n = self.noise
        v = [n[0]] * 3 + [n[1]] * 3 + [n[2]] * 3 + [n[3]] * 3 + [n[4]] * m.nu + [n[5]] * m.nu + [n[6]] * m.nu
        if self.height_scan:
            v += [self.scan_noise] * len(self.scan_points())
        return np.array(v)


@dataclass
class MotionTrackingCfg:
    """BeyondMimic-style motion imitation (BASELINE configs[2]): a reference-motion command manager plays
    a clip (motion.py); each world tracks it from a random phase (reference state initialisation) at a
    random spawn anchor. Observations: [ref joint pos - default, ref joint vel, base lin vel, base ang vel,
    projected gravity, root pos error (base frame), root orientation error (rotation vector), joint pos -
    default, joint vel, last action]. Rewards: exp tracking kernels of joint pos / joint vel / root pos /
    root orientation, action rate, and BeyondMimic's body terms -- exp kernels of the tracked bodies'
    position / orientation error with the clip's body poses re-expressed about the robot's anchor body, and
    of their world linear / angular velocity error (the clip's body states come from s3_motion_bodies) --
    plus a self-collision cost (contact sensor 0: robot-robot contacts). Terminations: root height error,
    orientation error; truncation at the clip end or after episode_steps. ``command`` holds (motion time,
    anchor x, anchor y) per world."""
    default_qpos: np.ndarray
    motion_qpos: np.ndarray
    motion_qvel: np.ndarray
    motion_dt: float
    decimation: int = 4
    action_scale: float = 0.25
    action_clip: float = 2.0
    episode_steps: int = 500
    # track_joint_pos, track_joint_vel, track_root_pos, track_root_ori, action_rate_l2, body_pos, body_ori,
    # body_lin_vel, body_ang_vel, self_collisions
    reward_weights: tuple = (0.5, 0.1, 0.5, 0.5, -0.01, 1.0, 1.0, 1.0, 1.0, -0.1)
    # exp-kernel denominators of the same terms (BeyondMimic's std^2 for the body terms: 0.3, 0.4, 1, pi)
    motion_sigmas: tuple = (1.0, 50.0, 0.1, 0.5, 0.09, 0.16, 1.0, 9.8696)
    anchor_body: str | int | None = None      # None: BEYONDMIMIC_ANCHOR if the model has it, else body 1
    track_bodies: tuple | None = None         # None: BEYONDMIMIC_BODIES present in the model, else tree 0
    self_collision: bool = True               # contact sensor 0 = robot-robot contacts, costed by term 9
    contact_sensors: tuple = ()               # extra sensors after the self-collision one
    # BeyondMimic's adaptive sampling of the start time over clip bins (failures of the previous launches,
    # exponentially averaged, plus a uniform share, smoothed forward with lambda^i weights); False: uniform
    # over the first motion_start_frac of the clip
    adaptive_sampling: bool = True
    bin_seconds: float = 1.0
    adaptive_kernel_size: int = 3
    adaptive_lambda: float = 0.8
    adaptive_uniform_ratio: float = 0.1
    adaptive_alpha: float = 0.001
    # domain randomisation, as the velocity task's (None: off): startup friction / base-mass scales, pushes
    friction_range: tuple = (0.6, 1.2)
    base_mass_range: tuple = (0.8, 1.2)
    push_interval: tuple | None = None
    push_velocity: float = 0.5

    def n_bins(self) -> int:
        clip = (self.motion_qpos.shape[0] - 1) * self.motion_dt
        return int(clip / self.bin_seconds) + 1 if self.adaptive_sampling else 0

    def kernel_weights(self) -> np.ndarray:
        w = self.adaptive_lambda ** np.arange(self.adaptive_kernel_size, dtype=np.float64)
        return w / w.sum()

    def initial_bin_cum(self) -> np.ndarray:
        """Cumulative sampling weights before any failure (the fold of zero counts): uniform."""
        return fold_bins(np.zeros(self.n_bins()), np.zeros(self.n_bins()), self)[1]
    max_height_error: float = 0.25
    max_ori_error: float = 0.8
    spawn_half_extent: float = 0.5
    motion_start_frac: float = 0.9
    noise: tuple = (0.1, 0.2, 0.05, 0.0, 0.01, 1.5, 0.0)
    kind: int = 1

    def obs_dim(self, m: Model) -> int:
        return 15 + 5 * m.nu

    def tracked(self, m: Model) -> tuple[int, tuple]:
        """(anchor body id, tracked body ids)."""
        bid = lambda b: m.body_names.index(b) if isinstance(b, str) else int(b)  # noqa: E731
        if self.anchor_body is not None:
            anchor = bid(self.anchor_body)
        else:
            anchor = m.body_names.index(BEYONDMIMIC_ANCHOR) if BEYONDMIMIC_ANCHOR in m.body_names else 1
        if self.track_bodies is not None:
            bodies = tuple(bid(b) for b in self.track_bodies)
        else:
            bodies = tuple(m.body_names.index(b) for b in BEYONDMIMIC_BODIES if b in m.body_names)
            if not bodies:
                bodies = tuple(b for b in range(1, m.nbody) if m.body_treeid[b] == 0)[:N.S3_MAX_TRACK]
        if not 1 <= len(bodies) <= N.S3_MAX_TRACK:
            raise ValueError(f"1..{N.S3_MAX_TRACK} tracked bodies")
        return anchor, bodies

    def sensors(self, m: Model) -> tuple:
        own = (("self_collision", robot_geoms(m), robot_geoms(m)),) if self.self_collision else ()
        return own + tuple(self.contact_sensors)

    def noise_vector(self, m: Model) -> np.ndarray:
        n = self.noise
        return np.array([0.0] * (2 * m.nu) + [n[0]] * 3 + [n[1]] * 3 + [n[2]] * 3 + [0.0] * 6 +
                        [n[4]] * m.nu + [n[5]] * m.nu + [n[6]] * m.nu)


@dataclass
class LiftTaskCfg:
    """Cube lift (BASELINE configs[3], mjlab's manipulation example) on ``robots.arm_cube_like``: reach the
    cube with the claw (tanh kernel), lift it above ``lift_height``, carry it to a per-episode goal
    (tanh kernel gated by the lift); action-rate and joint-velocity penalties; termination when the cube
    falls off the table, truncation after ``episode_steps``. ``command`` holds the goal position.
    Observations: [joint pos - default, joint vel, cube pos, cube quat, claw (mean fingertip) pos, goal,
    last action]. Pair with sensors.DepthCamera on the palm for the depth stream."""
    default_qpos: np.ndarray
    cube_qposadr: int
    tip_geoms: tuple
    cube_half: float = 0.025
    decimation: int = 4
    action_scale: float = 0.5
    action_clip: float = 2.0
    episode_steps: int = 250
    # reach, lifted, goal tracking, action_rate_l2, joint_vel_l2, end-effector / ground contacts (sensor 1)
    reward_weights: tuple = (1.0, 15.0, 16.0, -1e-4, -1e-4, -0.1)
    reach_std: float = 0.1
    goal_std: float = 0.3
    lift_height: float = 0.04
    min_cube_z: float = -0.05
    reset_joint_jitter: float = 0.1
    cube_x: tuple = (0.45, 0.65)
    cube_y: tuple = (-0.15, 0.15)
    goal_ranges: tuple = ((0.45, 0.65), (-0.2, 0.2), (0.2, 0.4))
    noise: tuple = (0.0, 0.0, 0.0, 0.0, 0.01, 0.05, 0.0)
    kind: int = 2
    # contact sensors on the end effector (the claw: the hand and finger bodies) and the ground plane (PAPER.md
    # §6.3): 0 claw-cube, 1 claw-ground (costed by reward term 5), 2 cube-ground; set by for_model
    contact_sensors: tuple = ()

    @classmethod
    def for_model(cls, m: Model, default_qpos: np.ndarray, **kw) -> "LiftTaskCfg":
        cube = m.body_names.index("cube")
        j = [k for k in range(m.njnt) if m.jnt_bodyid[k] == cube][0]
        tips = tuple(g for g in range(m.ngeom) if m.geom_type[g] == 2 and m.geom_bodyid[g] != cube)
        fingers = {int(m.geom_bodyid[g]) for g in tips}
        claw = fingers | {int(m.body_parentid[b]) for b in fingers}
        ee = tuple(g for g in range(m.ngeom) if int(m.geom_bodyid[g]) in claw)
        cube_g = tuple(g for g in range(m.ngeom) if m.geom_bodyid[g] == cube)
        kw.setdefault("contact_sensors", (("ee_cube", ee, cube_g), ("ee_ground", ee, (0,)), ("cube_ground", cube_g, (0,))))
        return cls(default_qpos=default_qpos, cube_qposadr=int(m.jnt_qposadr[j]), tip_geoms=tips, **kw)

    def sensors(self, m: Model) -> tuple:
        return tuple(self.contact_sensors)

    def obs_dim(self, m: Model) -> int:
        return 13 + 3 * m.nu

    def noise_vector(self, m: Model) -> np.ndarray:
        n = self.noise
        return np.array([n[4]] * m.nu + [n[5]] * m.nu + [0.0] * 13 + [n[6]] * m.nu)


class VelocityEnv3D:
    """Batched fused 3-D env on the GPU (world index outermost): velocity tracking
    (``VelocityTaskCfg``) or motion imitation (``MotionTrackingCfg``)."""

    def __init__(self, model: Model, cfg: VelocityTaskCfg, num_envs: int, seed: int = 0, world_offset: int = 0,
                 dtype: str = "f64", device="cuda"):
        self.model, self.cfg, self.num_envs, self.seed = model, cfg, int(num_envs), int(seed)
        self.world_offset = int(world_offset)
        self.dm = DeviceModel(model, dtype, device)
        self.dm.set_const()
        self.data = Data(self.dm, num_envs)
        dev, dt = self.dm.device, self.dm.tdtype
        n, nu = self.num_envs, model.nu
        self.obs_dim = cfg.obs_dim(model)
        z = lambda *s: torch.zeros(*s, dtype=dt, device=dev)  # noqa: E731
        self.action = z(n, nu)
        self.prev_action = z(n, nu)
        self.command = z(n, 3)
        self.cmd_timer = torch.zeros(n, dtype=torch.int32, device=dev)
        self.episode_step = torch.zeros(n, dtype=torch.int32, device=dev)
        self.episode_return = z(n)
        self.obs = z(n, self.obs_dim)
        self.reward = z(n)
        self.terminated = torch.zeros(n, dtype=torch.uint8, device=dev)
        self.truncated = torch.zeros(n, dtype=torch.uint8, device=dev)
        self.global_step = 0
        t = N.TaskT()
        motion = isinstance(cfg, MotionTrackingCfg)
        lift = isinstance(cfg, LiftTaskCfg)
        t.kind = cfg.kind if (motion or lift) else 0
        t.decimation, t.episode_steps = cfg.decimation, cfg.episode_steps
        t.obs_dim = self.obs_dim
        t.seed = self.seed
        t.world_offset = self.world_offset
        t.action_scale, t.action_clip = cfg.action_scale, cfg.action_clip
        t.spawn_half_extent = getattr(cfg, "spawn_half_extent", 0.0)
        t.reward_weights[:] = padded(cfg.reward_weights, len(t.reward_weights))
        t.noise[:] = cfg.noise
        # contact sensors
        self.sensor_names = tuple(name for name, _, _ in cfg.sensors(model))
        if len(self.sensor_names) > N.S3_MAX_SENSOR:
            raise ValueError(f"at most {N.S3_MAX_SENSOR} contact sensors")
        self.sensor = z(n, len(self.sensor_names))
        if self.sensor_names:
            self._pair_sensor = torch.as_tensor(pair_sensor_bits(model, cfg.sensors(model)), device=dev)
            t.nsensor, t.pair_sensor, t.sensor = len(self.sensor_names), self._pair_sensor.data_ptr(), \
                self.sensor.data_ptr()
        self.motion_body = None
        if motion:
            self._motion_q = torch.as_tensor(cfg.motion_qpos, dtype=dt, device=dev).contiguous()
            self._motion_v = torch.as_tensor(cfg.motion_qvel, dtype=dt, device=dev).contiguous()
            t.nframes, t.frame_dt = cfg.motion_qpos.shape[0], cfg.motion_dt
            t.motion_qpos, t.motion_qvel = self._motion_q.data_ptr(), self._motion_v.data_ptr()
            t.motion_sigmas[:] = padded(cfg.motion_sigmas, len(t.motion_sigmas))
            if not cfg.self_collision:  # term 9 costs sensor 0, the self-collision sensor when there is one
                t.reward_weights[9] = 0.0
            nb = cfg.n_bins()
            if nb:
                if not 1 <= cfg.adaptive_kernel_size <= N.S3_MAX_KERNEL:
                    raise ValueError(f"adaptive_kernel_size in 1..{N.S3_MAX_KERNEL}")
                t.nbins, t.nkernel = nb, cfg.adaptive_kernel_size
                t.adaptive_alpha, t.adaptive_uniform = cfg.adaptive_alpha, cfg.adaptive_uniform_ratio
                t.adaptive_kernel[:cfg.adaptive_kernel_size] = tuple(cfg.kernel_weights())
                self.bin_failed = z(nb)
                self.bin_cum = torch.as_tensor(cfg.initial_bin_cum(), dtype=dt, device=dev)
                self._bin_now = torch.zeros(nb, dtype=torch.int32, device=dev)
                self._bin_ticket = torch.zeros(1, dtype=torch.int32, device=dev)
                t.bin_failed, t.bin_cum = self.bin_failed.data_ptr(), self.bin_cum.data_ptr()
                t.bin_fail_now, t.bin_ticket = self._bin_now.data_ptr(), self._bin_ticket.data_ptr()
            anchor, bodies = cfg.tracked(model)
            t.anchor_body, t.ntrack = anchor, len(bodies)
            t.track_body[:len(bodies)] = bodies
            # the clip's body states (BeyondMimic's body_pos_w / quat / lin_vel / ang_vel): one launch, here
            self.motion_body = z(t.nframes, 1 + len(bodies), N.S3_BODY_STATE)
            t.motion_body = self.motion_body.data_ptr()
            st = torch.cuda.current_stream(dev).cuda_stream
            N.call("s3_motion_bodies", ctypes.byref(self.dm.struct), ctypes.byref(self.dm.layout), ctypes.byref(t),
                   self.motion_body.data_ptr(), st, launch=True)
            t.max_height_error, t.max_ori_error = cfg.max_height_error, cfg.max_ori_error
            t.motion_start_frac = cfg.motion_start_frac
        elif lift:
            t.cube_qposadr = cfg.cube_qposadr
            t.tip_geom[0], t.tip_geom[1] = cfg.tip_geoms
            t.cube_half, t.reach_std, t.goal_std = cfg.cube_half, cfg.reach_std, cfg.goal_std
            t.lift_height, t.min_cube_z, t.reset_joint_jitter = cfg.lift_height, cfg.min_cube_z, cfg.reset_joint_jitter
            t.cube_x[:], t.cube_y[:] = cfg.cube_x, cfg.cube_y
            for i, (lo, hi) in enumerate(cfg.goal_ranges):
                t.cmd_lo[i], t.cmd_hi[i] = lo, hi
        else:
            feet = cfg.foot_bodies(model)
            if len(feet) > N.S3_MAX_SENSOR:
                raise ValueError(f"at most {N.S3_MAX_SENSOR} feet")
            t.nfeet = len(feet)
            t.foot_body[:len(feet)] = feet
            if cfg.curriculum is not None:
                rows, cols, patch = cfg.curriculum
                t.curriculum, t.terrain_rows, t.terrain_cols, t.patch_size = 1, rows, cols, patch
                t.curriculum_max_init_level = cfg.curriculum_max_init_level
                t.curriculum_promote, t.curriculum_demote = cfg.curriculum_promote, cfg.curriculum_demote
                self.terrain_level = torch.zeros(n, dtype=torch.int32, device=dev)
                self.spawn_xy = z(n, 2)
                self.cmd_dist = z(n)
                t.terrain_level = self.terrain_level.data_ptr()
                t.spawn_xy, t.cmd_dist = self.spawn_xy.data_ptr(), self.cmd_dist.data_ptr()
            t.cmd_resample_steps = cfg.command_resample_steps
            t.track_sigma = cfg.track_sigma
            t.min_height, t.max_tilt_cos, t.reset_joint_jitter = cfg.min_height, cfg.max_tilt_cos, \
                cfg.reset_joint_jitter
            for i, (lo, hi) in enumerate(cfg.command_ranges):
                t.cmd_lo[i], t.cmd_hi[i] = lo, hi
        if not lift and cfg.push_interval is not None:  # domain randomisation events (velocity, motion kinds)
            t.events = 1
            self.data.friction_scale = torch.ones(n, dtype=dt, device=dev)
            self.event_timer = z(n)
            t.event_timer = self.event_timer.data_ptr()
            t.friction_range[:] = cfg.friction_range
            t.base_mass_range[:] = cfg.base_mass_range
            self.data.mass_scale = torch.ones(n, dtype=dt, device=dev)
            t.push_interval[:] = cfg.push_interval
            t.push_velocity = cfg.push_velocity
        pts = cfg.scan_points() if getattr(cfg, "height_scan", False) else []
        if len(pts) > N.S3_MAX_RAYS:
            raise ValueError("height scan larger than S3_MAX_RAYS")
        t.nscan = len(pts)
        for i, (x, y) in enumerate(pts):
            t.scan_xy[2 * i], t.scan_xy[2 * i + 1] = x, y
        if pts:
            t.scan_offset, t.scan_noise = cfg.scan_offset, cfg.scan_noise
        self._default = torch.as_tensor(cfg.default_qpos, dtype=dt, device=dev).contiguous()
        t.default_qpos = self._default.data_ptr()
        for name in ("action", "prev_action", "command", "cmd_timer", "episode_step", "episode_return", "obs",
                     "reward", "terminated", "truncated"):
            setattr(t, name, getattr(self, name).data_ptr())
        # cost-ordered schedule (s3_task.cost / order): worlds sorted by their last solver cost before each step
        self.solver_cost = self.world_order = None
        if os.environ.get("S3_ORDER", "1") != "0":
            self.solver_cost = torch.zeros(n, dtype=torch.int32, device=dev)
            self.world_order = torch.zeros(n, dtype=torch.int32, device=dev)
            t.cost, t.order = self.solver_cost.data_ptr(), self.world_order.data_ptr()
        self.task = t
        self._actions_in = z(n, nu)

    def _launch(self, mode: int, actions=None):
        d = self.data.struct(False)
        ptr = None if actions is None else actions.data_ptr()
        st = torch.cuda.current_stream(self.dm.device).cuda_stream
        N.call("s3_env_step", ctypes.byref(self.dm.struct), ctypes.byref(d), ctypes.byref(self.dm.layout),
               ctypes.byref(self.task), ptr, int(mode), int(self.global_step), st, launch=True)
        if mode == 0 and self.world_order is not None:
            N.LAUNCHES["count"] += 1  # the cost sort (order_kernel) launched ahead of the step kernel

    def metrics_record(self, step: int, group=None, steps_per_sec=None):
        """Job-wide statistics of the last step (metrics.py record): reward mean, running episode return,
        terminated / truncated counts, terrain-level histogram -- packed into one float64 vector and
        all-reduced in ONE collective across ranks (NCCL between GPUs; no-op on one rank)."""
        from .. import metrics

        rows = self.cfg.curriculum[0] if getattr(self.cfg, "curriculum", None) else 1
        levels = getattr(self, "terrain_level", None)
        levels = (levels if levels is not None else torch.zeros_like(self.episode_step)).long()
        counts = torch.stack([self.terminated.sum(), self.truncated.sum()])
        vec = metrics.pack_stats(self.reward, [self.episode_return], counts, levels, rows,
                                 torch.zeros(1, device=self.reward.device))
        metrics.allreduce_stats(vec, group)
        return metrics.unpack_stats(vec, ["episode_return"], ["terminated", "truncated"], rows, step, steps_per_sec)

    def reset(self):
        """Reset every world (counter 0 draws) and return the observation tensor."""
        self.global_step = 0
        self._launch(1)
        return self.obs

    def step(self, actions: torch.Tensor):
        """One control step: (obs, reward, terminated, truncated) as device tensors (reused buffers)."""
        if actions.dtype != self.dm.tdtype or actions.device != self.dm.device or not actions.is_contiguous():
            self._actions_in.copy_(actions)
            actions = self._actions_in
        if tuple(actions.shape) != (self.num_envs, self.model.nu):
            raise ValueError(f"actions shape {tuple(actions.shape)} does not match ({self.num_envs}, {self.model.nu})")
        self.global_step += 1
        self._launch(0, actions)
        return self.obs, self.reward, self.terminated, self.truncated
