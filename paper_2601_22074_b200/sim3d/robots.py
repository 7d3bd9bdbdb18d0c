"""Robots for the 3-D path, built in code (no MJCF parser, no network for assets).

* ``g1_like`` -- a 29-dof humanoid with the Unitree G1's joint layout (6 per leg,
  3 waist, 7 per arm; one hinge per body, free-floating pelvis: nq = 36,
  nv = 35) and approximately its link lengths and masses (~35 kg). The
  dimensions are a surrogate: the real G1 MJCF is not available offline.
* ``go1_like`` -- a 12-dof quadruped with the Unitree Go1's layout (hip
  abduction, thigh, calf per leg; nq = 19, nv = 18).
* ``terrain`` -- a flat plane or a seeded rough heightfield.

Both robots use position actuators (implicit ``kv`` by default, the mjlab G1
velocity configuration's ``BuiltinPositionActuator``), joint armature and
range limits, sphere feet and capsule limbs.
"""

from __future__ import annotations

import numpy as np

from .model import (ACT_IMPLICIT, GEOM_BOX, GEOM_CAPSULE, GEOM_SPHERE, ModelBuilder, Opt)


def rough_heightfield(seed: int, size_m: float = 16.0, spacing: float = 0.1, amplitude: float = 0.06):
    """Seeded rough terrain: uniform noise smoothed by a 3x3 box filter, centred at the origin,
    with a flat 2 m pad at the centre (spawn area)."""
    n = int(round(size_m / spacing)) + 1
    rng = np.random.default_rng(seed)
    h = rng.uniform(-amplitude, amplitude, size=(n + 2, n + 2))
    h = sum(h[i:i + n, j:j + n] for i in range(3) for j in range(3)) / 9.0
    c = (np.arange(n) - (n - 1) / 2) * spacing
    pad = (np.abs(c)[:, None] < 1.0) & (np.abs(c)[None, :] < 1.0)
    h = np.where(pad, 0.0, h)
    return h, spacing, (-(n - 1) / 2 * spacing, -(n - 1) / 2 * spacing)


def curriculum_heightfield(seed: int, rows: int = 5, cols: int = 6, patch: float = 8.0, spacing: float = 0.1,
                           amplitude: tuple = (0.0, 0.12)):
    """Terrain-curriculum grid (mjlab's rough-terrain generator analog, planar reference terrain.py:293-328
    restated in 3-D): rows x cols patches of ``patch`` metres; row r carries smoothed uniform noise of
    amplitude lerp(amplitude, r / (rows - 1)); each patch has a flat 1 m spawn pad at its centre.
    Patch (row r, col c) spans x in [c P, (c+1) P), y in [r P, (r+1) P); origin (0, 0)."""
    nx, ny = int(round(cols * patch / spacing)) + 1, int(round(rows * patch / spacing)) + 1
    rng = np.random.default_rng(seed)
    h = rng.uniform(-1.0, 1.0, size=(ny + 2, nx + 2))
    h = sum(h[i:i + ny, j:j + nx] for i in range(3) for j in range(3)) / 9.0
    x = np.arange(nx) * spacing
    y = np.arange(ny) * spacing
    row = np.minimum((y / patch).astype(int), rows - 1)
    amp = amplitude[0] + (amplitude[1] - amplitude[0]) * row / max(rows - 1, 1)
    h = h * amp[:, None]
    px = np.abs((x % patch) - 0.5 * patch)
    py = np.abs((y % patch) - 0.5 * patch)
    pad = (py[:, None] < 0.5) & (px[None, :] < 0.5)
    return np.where(pad, 0.0, h), spacing, (0.0, 0.0)


def _terrain(b: ModelBuilder, rough, seed: int):
    if rough == "curriculum":
        data, sp, origin = curriculum_heightfield(seed)
        b.heightfield(data, sp, origin, friction=1.0)
    elif rough:
        data, sp, origin = rough_heightfield(seed)
        b.heightfield(data, sp, origin, friction=1.0)
    else:
        b.plane(friction=1.0)


def g1_like(rough: bool | str = False, seed: int = 0, actuator_kind: int = ACT_IMPLICIT, self_collision: bool = True,
            opt: Opt | None = None):
    """rough: False (plane), True (16 m seeded rough patch), "curriculum" (5 x 6 graded patches)."""
    # 12 contacts: 8 foot spheres standing plus knees/hands; a fallen humanoid (which terminates) may
    # exceed it, later contacts are dropped in pair order and counted (ndropped)
    b = ModelBuilder("g1_like", opt, ncon_max=12)
    _terrain(b, rough, seed)
    pelvis = b.body("pelvis", 0, pos=(0, 0, 0.793), mass=3.81, inertia=(0.010, 0.009, 0.008))
    b.free_joint(pelvis)
    b.geom(pelvis, GEOM_SPHERE, (0.07,), pos=(0, 0, -0.02))
    arm = 0.01
    leg_gains = dict(kp=100.0, kv=2.0)
    for side, sy in (("left", 1.0), ("right", -1.0)):
        hp = b.body(f"{side}_hip_pitch_link", pelvis, pos=(0, 0.064 * sy, -0.103), mass=1.35,
                    inertia=(0.002, 0.002, 0.002))
        b.hinge(hp, (0, 1, 0), name=f"{side}_hip_pitch_joint", range=(-2.53, 2.88), armature=arm)
        hr = b.body(f"{side}_hip_roll_link", hp, pos=(0, 0.052 * sy, -0.030), mass=1.52, inertia=(0.002, 0.002, 0.002))
        b.hinge(hr, (1, 0, 0), name=f"{side}_hip_roll_joint",
                range=(-0.52, 2.97) if sy > 0 else (-2.97, 0.52), armature=arm)
        hy = b.body(f"{side}_hip_yaw_link", hr, pos=(0.025, 0, -0.124), mass=1.70, inertia=(0.006, 0.006, 0.002),
                    ipos=(0, 0, -0.08))
        b.hinge(hy, (0, 0, 1), name=f"{side}_hip_yaw_joint", range=(-2.75, 2.75), armature=arm)
        b.geom(hy, GEOM_CAPSULE, (0.055,), fromto=(0, 0, -0.02, -0.05, 0, -0.16))
        kn = b.body(f"{side}_knee_link", hy, pos=(-0.078, 0.0, -0.177), mass=1.93, inertia=(0.012, 0.012, 0.002),
                    ipos=(0, 0, -0.13))
        b.hinge(kn, (0, 1, 0), name=f"{side}_knee_joint", range=(-0.087, 2.88), armature=arm)
        b.geom(kn, GEOM_CAPSULE, (0.045,), fromto=(0, 0, -0.03, 0, 0, -0.26))
        ap = b.body(f"{side}_ankle_pitch_link", kn, pos=(0, 0, -0.30), mass=0.074, inertia=(1e-4, 1e-4, 1e-4))
        b.hinge(ap, (0, 1, 0), name=f"{side}_ankle_pitch_joint", range=(-0.87, 0.52), armature=arm)
        ar = b.body(f"{side}_ankle_roll_link", ap, pos=(0, 0, -0.017), mass=0.61, inertia=(4e-4, 1.5e-3, 1.6e-3),
                    ipos=(0.03, 0, -0.02))
        b.hinge(ar, (1, 0, 0), name=f"{side}_ankle_roll_joint", range=(-0.26, 0.26), armature=arm)
        for fx in (-0.05, 0.12):
            for fy in (-0.025, 0.025):
                b.geom(ar, GEOM_SPHERE, (0.012,), pos=(fx, fy, -0.031), name=f"{side}_foot")
    # waist + torso
    wy = b.body("waist_yaw_link", pelvis, pos=(0, 0, 0), mass=0.21, inertia=(1e-4, 1e-4, 1e-4))
    b.hinge(wy, (0, 0, 1), name="waist_yaw_joint", range=(-2.62, 2.62), armature=arm)
    wr = b.body("waist_roll_link", wy, pos=(-0.004, 0, 0.035), mass=0.09, inertia=(1e-4, 1e-4, 1e-4))
    b.hinge(wr, (1, 0, 0), name="waist_roll_joint", range=(-0.52, 0.52), armature=arm)
    torso = b.body("torso_link", wr, pos=(0, 0, 0.019), mass=9.6, inertia=(0.11, 0.09, 0.04), ipos=(0, 0, 0.2))
    b.hinge(torso, (0, 1, 0), name="waist_pitch_joint", range=(-0.52, 0.52), armature=arm)
    b.geom(torso, GEOM_CAPSULE, (0.09,), fromto=(0, 0, 0.1, 0, 0, 0.3))
    b.geom(torso, GEOM_SPHERE, (0.07,), pos=(0, 0, 0.45), name="head")
    for side, sy in (("left", 1.0), ("right", -1.0)):
        sp = b.body(f"{side}_shoulder_pitch_link", torso, pos=(0, 0.10 * sy, 0.24), mass=0.72,
                    inertia=(5e-4, 5e-4, 5e-4))
        b.hinge(sp, (0, 1, 0), name=f"{side}_shoulder_pitch_joint", range=(-3.09, 2.67), armature=arm)
        sr = b.body(f"{side}_shoulder_roll_link", sp, pos=(0, 0.038 * sy, -0.014), mass=0.64,
                    inertia=(5e-4, 5e-4, 5e-4))
        b.hinge(sr, (1, 0, 0), name=f"{side}_shoulder_roll_joint",
                range=(-1.59, 2.25) if sy > 0 else (-2.25, 1.59), armature=arm)
        sw = b.body(f"{side}_shoulder_yaw_link", sr, pos=(0, 0.006 * sy, -0.1), mass=0.60, inertia=(1e-3, 1e-3, 3e-4),
                    ipos=(0, 0, -0.04))
        b.hinge(sw, (0, 0, 1), name=f"{side}_shoulder_yaw_joint", range=(-2.62, 2.62), armature=arm)
        b.geom(sw, GEOM_CAPSULE, (0.035,), fromto=(0, 0, 0.0, 0, 0, -0.08))
        el = b.body(f"{side}_elbow_link", sw, pos=(0.016, 0, -0.08), mass=0.60, inertia=(1e-3, 1e-3, 3e-4),
                    ipos=(0.05, 0, 0))
        b.hinge(el, (0, 1, 0), name=f"{side}_elbow_joint", range=(-1.05, 2.09), armature=arm)
        b.geom(el, GEOM_CAPSULE, (0.03,), fromto=(0.0, 0, 0, 0.1, 0, 0))
        wrl = b.body(f"{side}_wrist_roll_link", el, pos=(0.1, 0.002 * sy, -0.01), mass=0.085,
                     inertia=(5e-5, 5e-5, 5e-5))
        b.hinge(wrl, (1, 0, 0), name=f"{side}_wrist_roll_joint", range=(-1.97, 1.97), armature=arm)
        wp = b.body(f"{side}_wrist_pitch_link", wrl, pos=(0.038, 0, 0), mass=0.48, inertia=(3e-4, 3e-4, 3e-4))
        b.hinge(wp, (0, 1, 0), name=f"{side}_wrist_pitch_joint", range=(-1.61, 1.61), armature=arm)
        wyl = b.body(f"{side}_wrist_yaw_link", wp, pos=(0.046, 0, 0), mass=0.25, inertia=(2e-4, 2e-4, 2e-4))
        b.hinge(wyl, (0, 0, 1), name=f"{side}_wrist_yaw_joint", range=(-1.61, 1.61), armature=arm)
        b.geom(wyl, GEOM_SPHERE, (0.04,), pos=(0.05, 0, 0), name=f"{side}_hand")
    for j in list(b.joints):
        if j["type"] == 3:
            name = j["name"]
            if "hip" in name or "knee" in name:
                gains = dict(kp=leg_gains["kp"] * (1.5 if "knee" in name else 1.0), kv=leg_gains["kv"],
                             effort=139.0 if "knee" in name else 88.0)
            elif "ankle" in name:
                gains = dict(kp=40.0, kv=2.0, effort=50.0)
            elif "waist" in name:
                gains = dict(kp=200.0, kv=5.0, effort=88.0)
            else:
                gains = dict(kp=40.0, kv=1.0, effort=25.0)
            b.actuator(name, kind=actuator_kind, **gains)
    if not self_collision:
        _only_terrain(b)
    else:
        _limit_self_pairs(b)
    return b.compile()


def _only_terrain(b: ModelBuilder):
    for g in b.geoms[1:]:
        g["contype"], g["conaffinity"] = 2, 1  # robot geoms collide with terrain (contype 1) only
    b.geoms[0]["contype"], b.geoms[0]["conaffinity"] = 1, 2


def _limit_self_pairs(b: ModelBuilder):
    """Terrain vs everything; self pairs only shin-shin and hand-vs-leg/torso."""
    _only_terrain(b)
    for g in b.geoms[1:]:
        name = b.bodies[g["body"]].name
        if "knee" in name:
            g["contype"] |= 4
            g["conaffinity"] |= 4
        if g.get("name", "") and "hand" in g["name"]:
            g["contype"] |= 8
        if "hip_yaw" in name or name == "torso_link":
            g["conaffinity"] |= 8


def go1_like(rough: bool = False, seed: int = 0, actuator_kind: int = ACT_IMPLICIT, opt: Opt | None = None):
    b = ModelBuilder("go1_like", opt)
    _terrain(b, rough, seed)
    trunk = b.body("trunk", 0, pos=(0, 0, 0.33), mass=5.2, inertia=(0.016, 0.037, 0.046))
    b.free_joint(trunk)
    b.geom(trunk, GEOM_BOX, (0.19, 0.047, 0.05))
    arm = 0.01
    for leg, (sx, sy) in (("FR", (1, -1)), ("FL", (1, 1)), ("RR", (-1, -1)), ("RL", (-1, 1))):
        hip = b.body(f"{leg}_hip", trunk, pos=(0.1881 * sx, 0.04675 * sy, 0), mass=0.68, inertia=(5e-4, 8e-4, 6e-4))
        b.hinge(hip, (1, 0, 0), name=f"{leg}_hip_joint", range=(-0.86, 0.86), armature=arm)
        th = b.body(f"{leg}_thigh", hip, pos=(0, 0.08 * sy, 0), mass=1.0, inertia=(5e-3, 5e-3, 1e-3),
                    ipos=(0, 0, -0.03))
        b.hinge(th, (0, 1, 0), name=f"{leg}_thigh_joint", range=(-0.69, 4.5), armature=arm)
        b.geom(th, GEOM_CAPSULE, (0.02,), fromto=(0, 0, 0, 0, 0, -0.213))
        ca = b.body(f"{leg}_calf", th, pos=(0, 0, -0.213), mass=0.2, inertia=(2e-3, 2e-3, 1e-4), ipos=(0, 0, -0.1))
        b.hinge(ca, (0, 1, 0), name=f"{leg}_calf_joint", range=(-2.82, -0.89), armature=arm)
        b.geom(ca, GEOM_SPHERE, (0.02,), pos=(0, 0, -0.213), name=f"{leg}_foot")
    for j in list(b.joints):
        if j["type"] == 3:
            b.actuator(j["name"], kind=actuator_kind, kp=35.0, kv=0.5, effort=23.7 if "calf" not in j["name"] else 35.55)
    _only_terrain(b)
    return b.compile()


G1_DEFAULT_JOINTS = {
    "hip_pitch": -0.312, "knee": 0.669, "ankle_pitch": -0.363, "elbow": 0.6,
    "left_shoulder_roll": 0.2, "right_shoulder_roll": -0.2, "shoulder_pitch": 0.2,
}
GO1_DEFAULT_JOINTS = {"hip": 0.0, "thigh": 0.9, "calf": -1.8}


def default_qpos(model, table: dict) -> np.ndarray:
    """qpos0 with named joint defaults (substring match, longest key wins)."""
    q = model.qpos0.copy()
    for j, name in enumerate(model.jnt_names):
        if model.jnt_type[j] != 3:
            continue
        best = None
        for k in table:
            if k in name and (best is None or len(k) > len(best)):
                best = k
        if best is not None:
            q[model.jnt_qposadr[j]] = table[best]
    return q


ARM_DEFAULT_JOINTS = {"shoulder_yaw": 0.0, "shoulder_pitch": -0.5, "elbow": 1.1, "wrist_pitch": 0.971,
                      "wrist_roll": 0.0, "hand_yaw": 0.0, "finger_left": 0.3, "finger_right": -0.3}


def arm_cube_like(opt: Opt | None = None, cube_size: float = 0.025):
    """A fixed-base 6-dof arm with a two-finger claw (hinged fingers, sphere fingertips) on a table
    (the plane) and a free cube (BASELINE configs[3], cube lift). Two kinematic trees: the arm and the
    cube. Collision filter: arm links touch the table only; fingertip spheres and finger capsules touch
    the cube (sphere-box, capsule-box); the cube touches the table (box corners)."""
    b = ModelBuilder("arm_cube_like", opt)
    b.plane(friction=1.0)
    base = b.body("link0", 0, pos=(0, 0, 0), mass=2.0, inertia=(0.01, 0.01, 0.01))
    b.geom(base, GEOM_CAPSULE, (0.06,), fromto=(0, 0, 0.0, 0, 0, 0.1), name="base")
    l1 = b.body("link1", base, pos=(0, 0, 0.1), mass=2.0, inertia=(0.01, 0.01, 0.005), ipos=(0, 0, 0.12))
    b.hinge(l1, (0, 0, 1), name="shoulder_yaw", range=(-2.9, 2.9), armature=0.05, damping=1.0)
    b.geom(l1, GEOM_CAPSULE, (0.05,), fromto=(0, 0, 0.0, 0, 0, 0.25))
    l2 = b.body("link2", l1, pos=(0, 0, 0.25), mass=2.0, inertia=(0.005, 0.03, 0.03), ipos=(0.2, 0, 0))
    b.hinge(l2, (0, 1, 0), name="shoulder_pitch", range=(-1.8, 1.8), armature=0.05, damping=1.0)
    b.geom(l2, GEOM_CAPSULE, (0.045,), fromto=(0.0, 0, 0, 0.4, 0, 0))
    l3 = b.body("link3", l2, pos=(0.4, 0, 0), mass=1.5, inertia=(0.004, 0.02, 0.02), ipos=(0.17, 0, 0))
    b.hinge(l3, (0, 1, 0), name="elbow", range=(-0.2, 2.8), armature=0.05, damping=1.0)
    b.geom(l3, GEOM_CAPSULE, (0.04,), fromto=(0.0, 0, 0, 0.35, 0, 0))
    l4 = b.body("link4", l3, pos=(0.35, 0, 0), mass=0.6, inertia=(0.001, 0.001, 0.001), ipos=(0.03, 0, 0))
    b.hinge(l4, (0, 1, 0), name="wrist_pitch", range=(-2.0, 2.0), armature=0.02, damping=0.5)
    l5 = b.body("link5", l4, pos=(0.05, 0, 0), mass=0.4, inertia=(0.0008, 0.0008, 0.0008), ipos=(0.03, 0, 0))
    b.hinge(l5, (1, 0, 0), name="wrist_roll", range=(-2.9, 2.9), armature=0.02, damping=0.5)
    b.geom(l5, GEOM_CAPSULE, (0.035,), fromto=(0.0, 0, 0, 0.05, 0, 0))
    hand = b.body("hand", l5, pos=(0.05, 0, 0), mass=0.5, inertia=(0.001, 0.001, 0.001), ipos=(0.03, 0, 0))
    b.hinge(hand, (1, 0, 0), name="hand_yaw", range=(-2.9, 2.9), armature=0.02, damping=0.5)
    b.geom(hand, GEOM_CAPSULE, (0.03,), fromto=(0.0, -0.04, 0, 0.0, 0.04, 0), name="palm")
    for side, sy in (("left", 1.0), ("right", -1.0)):
        f = b.body(f"finger_{side}_link", hand, pos=(0.03, 0.03 * sy, 0), mass=0.05, inertia=(1e-5, 1e-5, 1e-5),
                   ipos=(0.04, 0, 0))
        b.hinge(f, (0, 0, 1), name=f"finger_{side}", range=(-0.6, 0.6), armature=0.005, damping=0.1)
        b.geom(f, GEOM_CAPSULE, (0.008,), fromto=(0.0, 0, 0, 0.07, 0, 0), name=f"{side}_finger")
        b.geom(f, GEOM_SPHERE, (0.012,), pos=(0.08, -0.005 * sy, 0), name=f"{side}_tip")
    cube = b.body("cube", 0, pos=(0.55, 0.0, cube_size), mass=0.1,
                  inertia=(0.1 * (2 * cube_size) ** 2 / 6,) * 3)
    b.free_joint(cube)
    b.geom(cube, GEOM_BOX, (cube_size, cube_size, cube_size), friction=1.0, name="cube")
    # collision filter: table (1), arm (2), fingertips (2|8), cube (4, affinity 1|8)
    for g in b.geoms:
        if g["type"] == 0:
            g["contype"], g["conaffinity"] = 1, 1
        elif g.get("name") == "base":
            g["contype"], g["conaffinity"] = 0, 0  # static: never collides
        elif g.get("name") == "cube":
            g["contype"], g["conaffinity"] = 4, 1 | 8
        elif g.get("name", "") and (g["name"].endswith("_tip") or g["name"].endswith("_finger")):
            g["contype"], g["conaffinity"] = 2 | 8, 1  # fingertip spheres and finger capsules touch the cube
        else:
            g["contype"], g["conaffinity"] = 2, 1
    gains = {"finger": dict(kp=40.0, kv=2.0, effort=20.0)}
    for j in b.joints:
        if j["type"] != 3:
            continue
        g = gains["finger"] if j["name"].startswith("finger") else dict(kp=300.0, kv=30.0, effort=150.0)
        b.actuator(j["name"], kind=ACT_IMPLICIT, **g)
    return b.compile()


def box_stack(opt: Opt | None = None, sizes=((0.25, 0.18, 0.08), (0.12, 0.09, 0.06), (0.07, 0.05, 0.04)),
              yaws=(0.1, 0.5, -0.3), condims=(3, 3, 3)):
    """Free boxes stacked on a plane (box-box and box-plane contacts; one kinematic tree per box), each
    resting 2 mm into the one below at a different yaw: the narrowphase scene for box-box contacts.
    ``condims``: each box's contact dimensionality (a pair of two condim-1 boxes is frictionless)."""
    b = ModelBuilder("box_stack", opt)
    b.plane(friction=1.0)
    z = 0.0
    for k, (h, yaw, cd) in enumerate(zip(sizes, yaws, condims)):
        z += h[2] - 0.002
        mass = 500.0 * 8 * h[0] * h[1] * h[2]
        inertia = tuple(mass / 3.0 * (h[(i + 1) % 3] ** 2 + h[(i + 2) % 3] ** 2) for i in range(3))
        body = b.body(f"box{k}", 0, pos=(0.02 * k, -0.01 * k, z), quat=(np.cos(0.5 * yaw), 0, 0, np.sin(0.5 * yaw)),
                      mass=mass, inertia=inertia)
        b.free_joint(body)
        b.geom(body, GEOM_BOX, h, friction=0.8, name=f"box{k}", condim=cd)
        z += h[2]
    return b.compile()
