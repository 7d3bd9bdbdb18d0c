"""Reference motions for the 3-D motion-imitation task (BASELINE configs[2], BeyondMimic-style).

The reference has no motion tracking (SPEC.md:8 drops mjlab's §6.2); mjlab's
BeyondMimic task drives a ``MotionCommand`` that plays a retargeted human clip.
No clip can be downloaded here, so ``synthetic_walk_clip`` generates a
deterministic walking-like G1 clip (hip/knee/ankle/shoulder oscillations at a
1 Hz gait, forward root motion with a small vertical bob and yaw sway) with
qvel by central differences. A clip is (F, nq) qpos + (F, nv) qvel sampled at
``frame_dt``; the task interpolates it at each world's motion time.
"""

from __future__ import annotations

import numpy as np

from .model import JNT_FREE, Model


def _yaw_quat(yaw):
    return np.array([np.cos(0.5 * yaw), 0.0, 0.0, np.sin(0.5 * yaw)])


def synthetic_walk_clip(m: Model, default_qpos: np.ndarray, seconds: float = 10.0, fps: float = 50.0,
                        speed: float = 0.5, gait_hz: float = 1.0):
    F = int(round(seconds * fps)) + 1
    dt = 1.0 / fps
    t = np.arange(F) * dt
    w = 2.0 * np.pi * gait_hz
    Q = np.tile(default_qpos, (F, 1))
    for j, name in enumerate(m.jnt_names):
        if m.jnt_type[j] == JNT_FREE:
            continue
        a = m.jnt_qposadr[j]
        ph = 0.0 if name.startswith("left") else np.pi
        if "hip_pitch" in name:
            Q[:, a] += 0.35 * np.sin(w * t + ph)
        elif "knee" in name:
            Q[:, a] += 0.35 * 0.5 * (1.0 - np.cos(w * t + ph))
        elif "ankle_pitch" in name:
            Q[:, a] += -0.2 * np.sin(w * t + ph)
        elif "shoulder_pitch" in name:
            Q[:, a] += -0.3 * np.sin(w * t + ph)
        elif "elbow" in name:
            Q[:, a] += 0.15 * np.sin(w * t + ph)
        elif name == "waist_yaw_joint":
            Q[:, a] += 0.1 * np.sin(w * t)
    Q[:, 0] = speed * t
    Q[:, 1] = 0.0
    Q[:, 2] = default_qpos[2] + 0.02 * np.cos(2.0 * w * t)
    yaw = 0.1 * np.sin(w * t)
    Q[:, 3:7] = np.array([_yaw_quat(y) for y in yaw])
    V = np.zeros((F, m.nv))
    for j in range(m.njnt):
        a, d = m.jnt_qposadr[j], m.jnt_dofadr[j]
        if m.jnt_type[j] == JNT_FREE:
            V[:, d:d + 3] = np.gradient(Q[:, a:a + 3], dt, axis=0)
            V[:, d + 5] = np.gradient(yaw, dt)  # body-frame angular velocity of a pure yaw motion
        else:
            V[:, d] = np.gradient(Q[:, a], dt)
    return Q, V, dt


def _qconj_rotate(q, v):
    """R(q)^T v for a unit quaternion q = (w, x, y, z) (world -> body frame)."""
    w, x, y, z = q
    R = np.array([[1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y)],
                  [2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x)],
                  [2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)]])
    return R.T @ v


def load_motion_npz(path, m: Model, joint_names=None):
    """A BeyondMimic / mjlab motion file (``.npz``: ``fps``, ``joint_pos`` / ``joint_vel`` (F, J) in the
    robot's hinge-joint order or ``joint_names`` order, ``body_pos_w`` / ``body_quat_w`` (w, x, y, z) /
    ``body_lin_vel_w`` / ``body_ang_vel_w`` (F, B, .) with the root body first) -> the task's clip
    ``(qpos (F, nq), qvel (F, nv), frame_dt)``: the free joint from the root body's pose and velocity (its
    angular velocity rotated into the body frame, MuJoCo's free-joint convention), the hinges from the
    joint arrays. The clip's body states for the relative body terms are then rebuilt on the device from
    this qpos / qvel (``s3_motion_bodies``), so every tracked body follows the model's own kinematics."""
    data = np.load(path)
    fps = float(np.asarray(data["fps"]).reshape(-1)[0])
    jp, jv = np.asarray(data["joint_pos"], dtype=np.float64), np.asarray(data["joint_vel"], dtype=np.float64)
    F = jp.shape[0]
    hinges = [j for j in range(m.njnt) if m.jnt_type[j] != JNT_FREE]
    if joint_names is not None:
        order = [list(joint_names).index(m.jnt_names[j]) for j in hinges]
    else:
        if jp.shape[1] != len(hinges):
            raise ValueError(f"joint_pos has {jp.shape[1]} joints, the model {len(hinges)} hinges")
        order = list(range(len(hinges)))
    Q = np.tile(m.qpos0, (F, 1))
    V = np.zeros((F, m.nv))
    for col, j in zip(order, hinges):
        Q[:, m.jnt_qposadr[j]] = jp[:, col]
        V[:, m.jnt_dofadr[j]] = jv[:, col]
    free = [j for j in range(m.njnt) if m.jnt_type[j] == JNT_FREE]
    if free:
        a, d = m.jnt_qposadr[free[0]], m.jnt_dofadr[free[0]]
        pos, quat = np.asarray(data["body_pos_w"])[:, 0], np.asarray(data["body_quat_w"])[:, 0]
        quat = quat / np.linalg.norm(quat, axis=1, keepdims=True)
        Q[:, a:a + 3], Q[:, a + 3:a + 7] = pos, quat
        V[:, d:d + 3] = np.asarray(data["body_lin_vel_w"])[:, 0]
        ang = np.asarray(data["body_ang_vel_w"])[:, 0]
        V[:, d + 3:d + 6] = np.array([_qconj_rotate(quat[f], ang[f]) for f in range(F)])
    return Q, V, 1.0 / fps
