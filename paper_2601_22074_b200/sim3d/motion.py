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
