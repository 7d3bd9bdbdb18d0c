"""3-D articulated model: builder + compiled MjModel-shaped arrays.

The reference (`stridesim`) is planar; its 3-D counterpart in mjlab is an
``MjModel`` compiled from MJCF. This module is the
host-side model compiler for the 3-D path: a small builder (bodies, hinge and
free joints, primitive geoms, actuators) that compiles to flat numpy arrays
named like MuJoCo's (``body_parentid``, ``jnt_qposadr``, ``dof_parentid``,
``geom_size`` ...), plus the derived tables the kernels need:

* per-dof ancestor chains (``dof_chain``: the tree-sparse pattern of M and
  of its L^T D L factor),
* per-body dof chains (``body_chain``: the nonzero columns of a point
  Jacobian on that body),
* candidate collision pairs (contype/conaffinity filter, parent/child and
  same-body exclusion) with their merged Jacobian column lists.

Quaternions are (w, x, y, z). There is no MJCF parser: robots are built in
code (``robots.py``). Setup only -- nothing here runs per step.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

# joint / geom / actuator type codes (MuJoCo's numbering where one exists)
JNT_FREE, JNT_HINGE = 0, 3
GEOM_PLANE, GEOM_HFIELD, GEOM_SPHERE, GEOM_CAPSULE, GEOM_BOX = 0, 1, 2, 3, 6
ACT_PD, ACT_DC, ACT_IMPLICIT = 0, 1, 2

# kernel capacity bounds (mirrored in include/sim3d_b200.h)
MAX_NV = 64
MAX_NBODY = 64
MAX_CHAIN = 32
MAX_CON = 16
MAX_LIM = 32
MAX_TREE = 4


class ModelError(ValueError):
    pass


def quat_mul(a, b):
    aw, ax, ay, az = a
    bw, bx, by, bz = b
    return np.array([aw * bw - ax * bx - ay * by - az * bz,
                     aw * bx + ax * bw + ay * bz - az * by,
                     aw * by - ax * bz + ay * bw + az * bx,
                     aw * bz + ax * by - ay * bx + az * bw])


def quat2mat(q):
    w, x, y, z = q
    return np.array([[1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y)],
                     [2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x)],
                     [2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)]])


def axis_angle(axis, angle):
    axis = np.asarray(axis, dtype=np.float64)
    axis = axis / np.linalg.norm(axis)
    s = np.sin(0.5 * angle)
    return np.array([np.cos(0.5 * angle), axis[0] * s, axis[1] * s, axis[2] * s])


@dataclass
class Opt:
    timestep: float = 0.005
    gravity: tuple = (0.0, 0.0, -9.81)
    iterations: int = 10          # Newton iterations per substep
    ls_iterations: int = 20       # exact line-search iterations
    tolerance: float = 1e-8
    ls_tolerance: float = 0.01
    solref: tuple = (0.02, 1.0)   # (timeconst, dampratio)
    solimp: tuple = (0.9, 0.95, 0.001, 0.5, 2.0)  # (dmin, dmax, width, mid, power)
    solver: str = "newton"        # "newton" or "cg" (MuJoCo's mjSOL_NEWTON / mjSOL_CG)


@dataclass
class _Body:
    name: str
    parent: int
    pos: np.ndarray
    quat: np.ndarray
    mass: float
    inertia: np.ndarray
    ipos: np.ndarray
    iquat: np.ndarray
    joints: list = field(default_factory=list)


class ModelBuilder:
    """Tree builder: bodies must be added parent-first (topological order)."""

    def __init__(self, name: str = "model", opt: Opt | None = None, ncon_max: int = MAX_CON):
        self.name = name
        self.opt = opt or Opt()
        if not 1 <= ncon_max <= MAX_CON:
            raise ModelError(f"ncon_max must be in [1, {MAX_CON}]")
        self.ncon_max = int(ncon_max)  # contact capacity per world (MJWarp's nconmax analog)
        self.bodies: list[_Body] = [_Body("world", -1, np.zeros(3), np.array([1.0, 0, 0, 0]), 0.0, np.zeros(3),
                                          np.zeros(3), np.array([1.0, 0, 0, 0]))]
        self.joints: list[dict] = []
        self.geoms: list[dict] = []
        self.actuators: list[dict] = []
        self.exclude: set[tuple[int, int]] = set()
        self.hfield = None

    # -- tree ---------------------------------------------------------------
    def body(self, name, parent, pos=(0, 0, 0), quat=(1, 0, 0, 0), mass=1.0, inertia=(0.01, 0.01, 0.01),
             ipos=(0, 0, 0), iquat=(1, 0, 0, 0)) -> int:
        pid = self.body_id(parent) if isinstance(parent, str) else int(parent)
        if pid < 0 or pid >= len(self.bodies):
            raise ModelError(f"unknown parent {parent!r}")
        q = np.asarray(quat, dtype=np.float64)
        self.bodies.append(_Body(name, pid, np.asarray(pos, dtype=np.float64), q / np.linalg.norm(q), float(mass),
                                 np.asarray(inertia, dtype=np.float64), np.asarray(ipos, dtype=np.float64),
                                 np.asarray(iquat, dtype=np.float64) / np.linalg.norm(iquat)))
        return len(self.bodies) - 1

    def body_id(self, name: str) -> int:
        for i, b in enumerate(self.bodies):
            if b.name == name:
                return i
        raise ModelError(f"unknown body {name!r}")

    def free_joint(self, body, name=None):
        b = self.body_id(body) if isinstance(body, str) else body
        if self.bodies[b].parent != 0:
            raise ModelError("free joints only on children of the world body")
        self.joints.append(dict(name=name or f"{self.bodies[b].name}_free", type=JNT_FREE, body=b, pos=np.zeros(3),
                                axis=np.array([0, 0, 1.0]), range=(0.0, 0.0), limited=False, damping=0.0,
                                armature=0.0, ref=0.0))
        self.bodies[b].joints.append(len(self.joints) - 1)

    def hinge(self, body, axis, name=None, pos=(0, 0, 0), range=None, damping=0.0, armature=0.0, ref=0.0):
        b = self.body_id(body) if isinstance(body, str) else body
        ax = np.asarray(axis, dtype=np.float64)
        self.joints.append(dict(name=name or f"{self.bodies[b].name}_joint", type=JNT_HINGE, body=b,
                                pos=np.asarray(pos, dtype=np.float64), axis=ax / np.linalg.norm(ax),
                                range=tuple(range) if range is not None else (0.0, 0.0), limited=range is not None,
                                damping=float(damping), armature=float(armature), ref=float(ref)))
        self.bodies[b].joints.append(len(self.joints) - 1)

    # -- geometry -------------------------------------------------------------
    def geom(self, body, type, size, pos=(0, 0, 0), quat=(1, 0, 0, 0), friction=1.0, contype=1, conaffinity=1,
             fromto=None, name=None, condim=3):
        """condim 3: pyramidal sliding friction; 1: frictionless (a pair takes the larger of its geoms')."""
        if condim not in (1, 3):
            raise ModelError(f"condim {condim} is not supported (1 or 3)")
        b = self.body_id(body) if isinstance(body, str) else body
        size = list(size) + [0.0] * (3 - len(size))
        pos = np.asarray(pos, dtype=np.float64)
        q = np.asarray(quat, dtype=np.float64)
        if fromto is not None:  # capsule between two points (MJCF fromto)
            a, c = np.asarray(fromto[:3], dtype=np.float64), np.asarray(fromto[3:], dtype=np.float64)
            pos = 0.5 * (a + c)
            d = c - a
            L = np.linalg.norm(d)
            size[1] = 0.5 * L
            z = np.array([0, 0, 1.0])
            v = np.cross(z, d / L)
            s = np.linalg.norm(v)
            if s < 1e-12:
                q = np.array([1.0, 0, 0, 0]) if d[2] > 0 else np.array([0.0, 1.0, 0, 0])
            else:
                q = axis_angle(v / s, np.arctan2(s, np.dot(z, d / L)))
        self.geoms.append(dict(name=name, type=int(type), body=b, size=np.asarray(size, dtype=np.float64), pos=pos,
                               quat=q / np.linalg.norm(q), friction=float(friction), contype=int(contype),
                               conaffinity=int(conaffinity), condim=int(condim)))
        return len(self.geoms) - 1

    def plane(self, friction=1.0, condim=3):
        return self.geom(0, GEOM_PLANE, (0, 0, 0), friction=friction, condim=condim)

    def heightfield(self, data, spacing, origin=(0.0, 0.0), friction=1.0):
        """Terrain as a (nrow, ncol) height grid (rows along y, cols along x), cell size ``spacing``,
        sample (0, 0) at world (origin[0], origin[1])."""
        data = np.ascontiguousarray(data, dtype=np.float64)
        self.hfield = dict(data=data, spacing=float(spacing), origin=np.asarray(origin, dtype=np.float64))
        return self.geom(0, GEOM_HFIELD, (0, 0, 0), friction=friction)

    def exclude_pair(self, body_a, body_b):
        a = self.body_id(body_a) if isinstance(body_a, str) else body_a
        b = self.body_id(body_b) if isinstance(body_b, str) else body_b
        self.exclude.add((min(a, b), max(a, b)))

    def actuator(self, joint, kind=ACT_IMPLICIT, kp=100.0, kv=2.0, effort=100.0, saturation=None, vmax=None):
        names = [j["name"] for j in self.joints]
        if joint not in names:
            raise ModelError(f"unknown joint {joint!r}")
        j = names.index(joint)
        if self.joints[j]["type"] != JNT_HINGE:
            raise ModelError("actuators drive hinge joints")
        self.actuators.append(dict(joint=j, kind=int(kind), kp=float(kp), kv=float(kv), effort=float(effort),
                                   saturation=float(saturation if saturation is not None else effort),
                                   vmax=float(vmax if vmax is not None else 1e9)))

    def compile(self) -> "Model":
        return Model(self)


def _rbound(g) -> float:
    t, s = g["type"], g["size"]
    if t == GEOM_SPHERE:
        return float(s[0])
    if t == GEOM_CAPSULE:
        return float(s[0] + s[1])
    if t == GEOM_BOX:
        return float(np.linalg.norm(s[:3]))
    return 0.0


class Model:
    """Compiled arrays (MjModel-shaped names); all float arrays are float64."""

    def __init__(self, b: ModelBuilder):
        self.name = b.name
        self.opt = b.opt
        self.ncon_max = b.ncon_max
        nb = len(b.bodies)
        self.nbody = nb
        self.body_names = [x.name for x in b.bodies]
        self.body_parentid = np.array([x.parent for x in b.bodies], dtype=np.int32)
        self.body_pos = np.array([x.pos for x in b.bodies])
        self.body_quat = np.array([x.quat for x in b.bodies])
        self.body_mass = np.array([x.mass for x in b.bodies])
        self.body_inertia = np.array([x.inertia for x in b.bodies])
        self.body_ipos = np.array([x.ipos for x in b.bodies])
        self.body_iquat = np.array([x.iquat for x in b.bodies])
        root = np.zeros(nb, dtype=np.int32)
        depth = np.zeros(nb, dtype=np.int32)
        for i in range(1, nb):
            p = self.body_parentid[i]
            if p >= i:
                raise ModelError("bodies must be added parent-first")
            root[i] = i if p == 0 else root[p]
            depth[i] = depth[p] + 1
        self.body_rootid = root
        self.body_depth = depth
        # kinematic trees (a robot, a free object, ...): each uses its own subtree com as c-frame origin
        roots = sorted(set(root[1:].tolist()))
        if len(roots) > MAX_TREE:
            raise ModelError(f"{len(roots)} kinematic trees exceed MAX_TREE={MAX_TREE}")
        self.ntree = len(roots)
        self.body_treeid = np.array([roots.index(root[i]) if i > 0 else 0 for i in range(nb)], dtype=np.int32)
        self.tree_mass = np.array([self.body_mass[1:][self.body_treeid[1:] == t].sum() for t in range(self.ntree)])

        # joints, qpos / dof addresses (body order)
        jorder = [j for bd in b.bodies for j in bd.joints]
        J = [b.joints[j] for j in jorder]
        self.njnt = len(J)
        self.jnt_names = [j["name"] for j in J]
        self.jnt_type = np.array([j["type"] for j in J], dtype=np.int32)
        self.jnt_bodyid = np.array([j["body"] for j in J], dtype=np.int32)
        self.jnt_pos = np.array([j["pos"] for j in J]).reshape(-1, 3)
        self.jnt_axis = np.array([j["axis"] for j in J]).reshape(-1, 3)
        self.jnt_range = np.array([j["range"] for j in J]).reshape(-1, 2)
        self.jnt_limited = np.array([j["limited"] for j in J], dtype=np.int32)
        qadr, dadr, nq, nv = [], [], 0, 0
        for j in J:
            qadr.append(nq)
            dadr.append(nv)
            nq += 7 if j["type"] == JNT_FREE else 1
            nv += 6 if j["type"] == JNT_FREE else 1
        self.nq, self.nv = nq, nv
        if nv > MAX_NV or nb > MAX_NBODY:
            raise ModelError(f"nv={nv} / nbody={nb} exceed the kernel bounds {MAX_NV}/{MAX_NBODY}")
        self.jnt_qposadr = np.array(qadr, dtype=np.int32)
        self.jnt_dofadr = np.array(dadr, dtype=np.int32)
        self.body_jntadr = np.full(nb, -1, dtype=np.int32)
        self.body_jntnum = np.zeros(nb, dtype=np.int32)
        self.body_dofadr = np.full(nb, -1, dtype=np.int32)
        self.body_dofnum = np.zeros(nb, dtype=np.int32)
        for k, j in enumerate(J):
            bd = j["body"]
            if self.body_jntadr[bd] < 0:
                self.body_jntadr[bd] = k
                self.body_dofadr[bd] = dadr[k]
            self.body_jntnum[bd] += 1
            self.body_dofnum[bd] += 6 if j["type"] == JNT_FREE else 1
        self.qpos0 = np.zeros(nq)
        for k, j in enumerate(J):
            if j["type"] == JNT_FREE:
                bd = j["body"]
                self.qpos0[qadr[k]:qadr[k] + 3] = self.body_pos[bd]
                self.qpos0[qadr[k] + 3:qadr[k] + 7] = self.body_quat[bd]
            else:
                self.qpos0[qadr[k]] = j["ref"]

        # dofs
        self.dof_bodyid = np.zeros(nv, dtype=np.int32)
        self.dof_jntid = np.zeros(nv, dtype=np.int32)
        self.dof_damping = np.zeros(nv)
        self.dof_armature = np.zeros(nv)
        for k, j in enumerate(J):
            n = 6 if j["type"] == JNT_FREE else 1
            for d in range(dadr[k], dadr[k] + n):
                self.dof_bodyid[d] = j["body"]
                self.dof_jntid[d] = k
                self.dof_damping[d] = j["damping"]
                self.dof_armature[d] = j["armature"]
        # dof_parentid: previous dof of the same body, else last dof of the nearest ancestor with dofs
        self.dof_parentid = np.full(nv, -1, dtype=np.int32)
        for d in range(nv):
            bd = self.dof_bodyid[d]
            if d > self.body_dofadr[bd]:
                self.dof_parentid[d] = d - 1
                continue
            p = self.body_parentid[bd]
            while p > 0 and self.body_dofnum[p] == 0:
                p = self.body_parentid[p]
            if p > 0:
                self.dof_parentid[d] = self.body_dofadr[p] + self.body_dofnum[p] - 1
        # ancestor chains (inclusive, ascending) per dof and per body
        self.dof_chain = []
        for d in range(nv):
            c, x = [], d
            while x >= 0:
                c.append(x)
                x = int(self.dof_parentid[x])
            self.dof_chain.append(c[::-1])
        self.body_chain = []
        for bd in range(nb):
            x = bd
            while x > 0 and self.body_dofnum[x] == 0:
                x = self.body_parentid[x]
            last = self.body_dofadr[x] + self.body_dofnum[x] - 1 if x > 0 else -1
            self.body_chain.append(self.dof_chain[last] if last >= 0 else [])
        if max(len(c) for c in self.body_chain) > MAX_CHAIN:
            raise ModelError("kinematic chain deeper than MAX_CHAIN dofs")

        # geoms
        G = b.geoms
        self.ngeom = len(G)
        self.geom_type = np.array([g["type"] for g in G], dtype=np.int32)
        self.geom_bodyid = np.array([g["body"] for g in G], dtype=np.int32)
        self.geom_size = np.array([g["size"] for g in G]).reshape(-1, 3)
        self.geom_pos = np.array([g["pos"] for g in G]).reshape(-1, 3)
        self.geom_quat = np.array([g["quat"] for g in G]).reshape(-1, 4)
        self.geom_friction = np.array([g["friction"] for g in G])
        self.geom_condim = np.array([g.get("condim", 3) for g in G], dtype=np.int32)
        self.geom_rbound = np.array([_rbound(g) for g in G])
        self.geom_contype = np.array([g["contype"] for g in G], dtype=np.int32)
        self.geom_conaffinity = np.array([g["conaffinity"] for g in G], dtype=np.int32)
        terrain = [i for i, g in enumerate(G) if g["type"] in (GEOM_PLANE, GEOM_HFIELD)]
        if len(terrain) != 1 or terrain[0] != 0:
            raise ModelError("exactly one terrain geom (plane or heightfield), added first")
        hf = b.hfield
        if hf is not None:
            self.hfield_data = hf["data"]
            self.hfield_spacing = hf["spacing"]
            self.hfield_origin = hf["origin"]
        else:
            self.hfield_data = np.zeros((2, 2))
            self.hfield_spacing = 1.0
            self.hfield_origin = np.zeros(2)
        self.terrain_is_hfield = int(self.geom_type[0] == GEOM_HFIELD)

        # collision pairs: terrain vs every collidable robot geom, then geom-geom self pairs
        pairs = []
        for g1 in range(self.ngeom):
            for g2 in range(g1 + 1, self.ngeom):
                b1, b2 = int(self.geom_bodyid[g1]), int(self.geom_bodyid[g2])
                if b1 == b2:
                    continue
                if not ((self.geom_contype[g1] & self.geom_conaffinity[g2]) or
                        (self.geom_contype[g2] & self.geom_conaffinity[g1])):
                    continue
                if b1 != 0 and (self.body_parentid[b2] == b1 or self.body_parentid[b1] == b2):
                    continue
                if (min(b1, b2), max(b1, b2)) in b.exclude:
                    continue
                t1, t2 = self.geom_type[g1], self.geom_type[g2]
                if t1 in (GEOM_PLANE, GEOM_HFIELD):
                    if t2 not in (GEOM_SPHERE, GEOM_CAPSULE, GEOM_BOX):
                        continue
                elif t1 == GEOM_BOX and t2 in (GEOM_SPHERE, GEOM_CAPSULE):
                    pairs.append((g2, g1))  # the narrowphase takes the box second
                    continue
                elif not ((t1 in (GEOM_SPHERE, GEOM_CAPSULE) and t2 in (GEOM_SPHERE, GEOM_CAPSULE, GEOM_BOX)) or
                          (t1 == GEOM_BOX and t2 == GEOM_BOX)):
                    continue  # supported pairs: sphere/capsule x sphere/capsule/box (box second), box x box
                pairs.append((g1, g2))
        self.npair = len(pairs)
        self.pair_geom = np.array(pairs, dtype=np.int32).reshape(-1, 2)
        # a pair's contact dimensionality is the larger of its geoms' (MuJoCo's rule at equal priority):
        # 1 = frictionless normal contact, 3 = pyramidal sliding friction
        self.pair_condim = np.array([max(self.geom_condim[g1], self.geom_condim[g2]) for g1, g2 in pairs],
                                    dtype=np.uint8)
        self.pair_chain = []
        for g1, g2 in pairs:
            c = sorted(set(self.body_chain[self.geom_bodyid[g1]]) | set(self.body_chain[self.geom_bodyid[g2]]))
            if len(c) > MAX_CHAIN:
                raise ModelError("pair Jacobian wider than MAX_CHAIN dofs")
            self.pair_chain.append(c)

        # actuators
        A = b.actuators
        self.nu = len(A)
        self.actuator_jntid = np.array([a["joint"] for a in A], dtype=np.int32)
        self.actuator_dofadr = np.array([self.jnt_dofadr[jorder.index(a["joint"])] for a in A], dtype=np.int32)
        self.actuator_qposadr = np.array([self.jnt_qposadr[jorder.index(a["joint"])] for a in A], dtype=np.int32)
        self.actuator_kind = np.array([a["kind"] for a in A], dtype=np.int32)
        self.actuator_kp = np.array([a["kp"] for a in A])
        self.actuator_kv = np.array([a["kv"] for a in A])
        self.actuator_effort = np.array([a["effort"] for a in A])
        self.actuator_saturation = np.array([a["saturation"] for a in A])
        self.actuator_vmax = np.array([a["vmax"] for a in A])
        if len(set(self.actuator_dofadr.tolist())) != self.nu:
            raise ModelError("one actuator per joint")

        self.nlim = int(self.jnt_limited.sum())
        if self.nlim > MAX_LIM:
            raise ModelError(f"{self.nlim} limited joints exceed MAX_LIM={MAX_LIM}")
        self.nefc_max = self.nlim + 4 * self.ncon_max  # a limited hinge violates at most one side
        # set by set_const (inverse weights at qpos0; computed from M(qpos0) by whoever owns a dynamics engine)
        self.dof_invweight0 = np.ones(nv)
        self.body_invweight0 = np.zeros(nb)
        self.meaninertia = 1.0

    # ------------------------------------------------------------------------
    def set_const(self, M0: np.ndarray, body_jacp0: list[np.ndarray]):
        """Inverse weights from the mass matrix at qpos0 (MuJoCo mj_setConst analog):
        dof_invweight0 = diag(M^-1); body_invweight0 = mean diagonal of J M^-1 J^T over the
        translational Jacobian of each body's com; meaninertia = trace(M)/nv."""
        Minv = np.linalg.inv(M0)
        self.dof_invweight0 = np.diag(Minv).copy()
        w = np.zeros(self.nbody)
        for bd in range(1, self.nbody):
            Jb = body_jacp0[bd]
            w[bd] = np.trace(Jb @ Minv @ Jb.T) / 3.0
        self.body_invweight0 = w
        self.meaninertia = float(np.trace(M0) / self.nv)

    def actuated_qposadr(self):
        return self.actuator_qposadr

    def summary(self) -> dict:
        return dict(name=self.name, nbody=self.nbody, nq=self.nq, nv=self.nv, nu=self.nu, ngeom=self.ngeom,
                    npair=self.npair, nlim=self.nlim, max_chain=max(len(c) for c in self.body_chain))
