"""Device-resident 3-D model + MjData-shaped batched state, stepped by the sm_100a kernel.

``DeviceModel`` packs a compiled ``Model`` (model.py) into one device buffer
in the kernel's element type, with the derived tables the warp-per-world
kernel indexes (tree levels, child lists, ancestor/descendant dof masks,
ancestor chains, per-pair Jacobian column lists). ``Data`` holds the batched
state as torch tensors with MuJoCo's field names, world index outermost:
``qpos (N, nq)``, ``qvel (N, nv)``, ``ctrl (N, nu)``, ``qacc_warmstart``,
``qfrc_applied``, ``time``; ``step(nsub)`` advances every world ``nsub``
physics substeps in ONE kernel launch. There is no CPU path: without the
built extension nothing runs.
"""

from __future__ import annotations

import ctypes
import os

import numpy as np
import torch

from . import native as N
from .model import MAX_CHAIN, MAX_CON, Model, quat2mat

_F = {"f64": (torch.float64, np.float64, 0), "f32": (torch.float32, np.float32, 1)}
MAX_ROWS = 96


class DeviceModel:
    """A compiled Model's tables on the GPU (+ the inverse weights set from the GPU mass matrix)."""

    def __init__(self, model: Model, dtype: str = "f64", device="cuda"):
        if dtype not in _F:
            raise ValueError("dtype must be 'f64' or 'f32'")
        self.model = model
        self.dtype = dtype
        self.tdtype, self.ndtype, code = _F[dtype]
        self.device = torch.device(device)
        if self.device.type == "cuda" and self.device.index is None:
            self.device = torch.device("cuda", torch.cuda.current_device())
        m = model
        self._arrays: dict[str, np.ndarray] = {}
        # tree levels (bodies sorted by depth), children in descending index
        depth = m.body_depth
        nlevel = int(depth.max()) + 1
        order = [b for L in range(nlevel) for b in range(m.nbody) if depth[b] == L]
        level_ptr = np.zeros(nlevel + 1, dtype=np.int32)
        for L in range(nlevel):
            level_ptr[L + 1] = level_ptr[L] + int((depth == L).sum())
        children = [[] for _ in range(m.nbody)]
        for b in range(1, m.nbody):
            children[m.body_parentid[b]].append(b)
        child_ptr = np.zeros(m.nbody + 1, dtype=np.int32)
        child_idx = []
        for b in range(m.nbody):
            ch = sorted(children[b], reverse=True) if b > 0 else []
            child_idx += ch
            child_ptr[b + 1] = len(child_idx)
        body_dofmask = np.zeros(m.nbody, dtype=np.uint64)
        for b in range(m.nbody):
            for d in m.body_chain[b]:
                body_dofmask[b] |= np.uint64(1) << np.uint64(d)
        desc = np.zeros(m.nv, dtype=np.uint64)
        dof_chain = np.zeros((m.nv, MAX_CHAIN), dtype=np.uint8)
        dof_chainlen = np.zeros(m.nv, dtype=np.int32)
        for d in range(m.nv):
            c = m.dof_chain[d]
            dof_chain[d, :len(c)] = c
            dof_chainlen[d] = len(c)
            for a in c[:-1]:
                desc[a] |= np.uint64(1) << np.uint64(d)
        pair_chain = np.zeros((max(m.npair, 1), MAX_CHAIN), dtype=np.uint8)
        pair_chainlen = np.zeros(max(m.npair, 1), dtype=np.int32)
        for p, c in enumerate(m.pair_chain):
            pair_chain[p, :len(c)] = c
            pair_chainlen[p] = len(c)
        self.chain_stride = int(max([len(c) for c in m.pair_chain] + [1]))
        # factorization update lists: for each k, pairs (i in anc(k), j in chain(i))
        ldl_ptr, ldl_pair = [0], []
        for k in range(m.nv):
            for i in m.dof_chain[k][:-1]:
                for j in m.dof_chain[i]:
                    ldl_pair.append((i << 8) | j)
            ldl_ptr.append(len(ldl_pair))
        ldl_norm = [(k << 8) | i for k in range(m.nv) for i in m.dof_chain[k][:-1]]
        tree_ent = [(i << 8) | j for i in range(m.nv) for j in m.dof_chain[i]]
        # level schedules of the tree factorization / solves: dofs of equal height (distance to the
        # deepest leaf below) eliminate together; equal depth for the root-to-leaf sweep
        kids = [[] for _ in range(m.nv)]
        for d in range(m.nv):
            if m.dof_parentid[d] >= 0:
                kids[m.dof_parentid[d]].append(d)
        height = [0] * m.nv
        for d in range(m.nv - 1, -1, -1):
            height[d] = 1 + max(height[c] for c in kids[d]) if kids[d] else 0
        nh = max(height) + 1 if m.nv else 0
        hlev = [[d for d in range(m.nv) if height[d] == L] for L in range(nh)]
        dlev = [[d for d in range(m.nv) if len(m.dof_chain[d]) - 1 == L]
                for L in range(max(len(c) for c in m.dof_chain))]
        fl_ptr, fl_ent, fl_kptr, fl_k = [0], [], [0], []
        bl_ptr, bl_ent, bl_iptr, bl_i = [0], [], [0], []
        for lev in hlev:
            ent, tgt = {}, {}
            for k in lev:
                for i in m.dof_chain[k][:-1]:
                    tgt.setdefault(i, []).append(k)
                    for j in m.dof_chain[i]:
                        ent.setdefault((i, j), []).append(k)
            for (i, j), ks in sorted(ent.items()):
                fl_ent.append((i << 8) | j)
                fl_k += ks
                fl_kptr.append(len(fl_k))
            fl_ptr.append(len(fl_ent))
            for j, srcs in sorted(tgt.items()):
                bl_ent.append(j)
                bl_i += srcs
                bl_iptr.append(len(bl_i))
            bl_ptr.append(len(bl_ent))
        fw_ptr, fw_dof = [0], []
        for lev in dlev:
            fw_dof += lev
            fw_ptr.append(len(fw_dof))
        hmask = np.array([sum(1 << d for d in lev) for lev in hlev] + [0], dtype=np.uint64)
        dmask_lv = np.array([sum(1 << d for d in lev) for lev in dlev] + [0], dtype=np.uint64)
        dof_chainmask = np.zeros(m.nv, dtype=np.uint64)
        for d in range(m.nv):
            for a in m.dof_chain[d]:
                dof_chainmask[d] |= np.uint64(1) << np.uint64(a)
        pair_dofmask = np.zeros(max(m.npair, 1), dtype=np.uint64)
        for p, c in enumerate(m.pair_chain):
            for a in c:
                pair_dofmask[p] |= np.uint64(1) << np.uint64(a)
        classes, pair_class, pair_tree = {}, [], []
        for p, (g1, g2) in enumerate(m.pair_geom):
            key = tuple(m.pair_chain[p])
            pair_class.append(classes.setdefault(key, len(classes)))
            b1, b2 = int(m.geom_bodyid[g1]), int(m.geom_bodyid[g2])
            c1, c2 = set(m.body_chain[b1]), set(m.body_chain[b2])
            pair_tree.append(int(c1 <= c2 or c2 <= c1))
        tri_tab = np.array([(a << 8) | b for a in range(MAX_CHAIN) for b in range(a + 1)], dtype=np.uint16)
        lim = np.nonzero(m.jnt_limited)[0]
        geom_lmat = np.array([quat2mat(q) for q in m.geom_quat]).reshape(-1, 9)
        body_ilmat = np.array([quat2mat(q) for q in m.body_iquat]).reshape(-1, 9)
        act_gain = np.stack([m.actuator_kp, m.actuator_kv, m.actuator_effort, m.actuator_saturation,
                             m.actuator_vmax], axis=1) if m.nu else np.zeros((1, 5))
        ints = dict(
            body_treeid=m.body_treeid,
            body_parentid=m.body_parentid, body_jntadr=np.maximum(m.body_jntadr, 0), body_jntnum=m.body_jntnum,
            body_dofadr=np.maximum(m.body_dofadr, 0), body_dofnum=m.body_dofnum, body_dofmask=body_dofmask,
            level_ptr=level_ptr, level_body=np.array(order, dtype=np.int32), child_ptr=child_ptr,
            child_idx=np.array(child_idx + [0], dtype=np.int32), jnt_type=m.jnt_type, jnt_qposadr=m.jnt_qposadr,
            jnt_dofadr=m.jnt_dofadr, dof_bodyid=m.dof_bodyid, dof_parentid=m.dof_parentid, dof_descmask=desc,
            dof_chain=dof_chain, dof_chainlen=dof_chainlen,
            lim_qposadr=np.append(m.jnt_qposadr[lim], 0).astype(np.int32),
            lim_dofadr=np.append(m.jnt_dofadr[lim], 0).astype(np.int32),
            geom_type=m.geom_type, geom_bodyid=m.geom_bodyid, pair_geom=np.append(m.pair_geom.reshape(-1), [0, 0]),
            pair_chain=pair_chain, pair_chainlen=pair_chainlen,
            pair_condim=np.append(m.pair_condim, 3).astype(np.uint8),
            act_dofadr=np.append(m.actuator_dofadr, 0).astype(np.int32),
            act_qposadr=np.append(m.actuator_qposadr, 0).astype(np.int32),
            act_kind=np.append(m.actuator_kind, 0).astype(np.int32),
            ldl_ptr=np.array(ldl_ptr, dtype=np.int32), ldl_pair=np.array(ldl_pair + [0], dtype=np.uint16),
            ldl_norm=np.array(ldl_norm + [0], dtype=np.uint16),
            tree_ent=np.array(tree_ent, dtype=np.uint16), dof_chainmask=dof_chainmask, pair_dofmask=pair_dofmask,
            fl_ptr=np.array(fl_ptr, dtype=np.int32), fl_ent=np.array(fl_ent + [0], dtype=np.uint16),
            fl_kptr=np.array(fl_kptr, dtype=np.int32), fl_k=np.array(fl_k + [0], dtype=np.uint8),
            bl_ptr=np.array(bl_ptr, dtype=np.int32), bl_ent=np.array(bl_ent + [0], dtype=np.uint8),
            bl_iptr=np.array(bl_iptr, dtype=np.int32), bl_i=np.array(bl_i + [0], dtype=np.uint8),
            fw_ptr=np.array(fw_ptr, dtype=np.int32), fw_dof=np.array(fw_dof + [0], dtype=np.uint8),
            hlev_mask=hmask, dlev_mask=dmask_lv,
            pair_class=np.array(pair_class + [0], dtype=np.int32), pair_tree=np.array(pair_tree + [1], dtype=np.int32),
            tri_tab=tri_tab)
        floats = dict(
            body_pos=m.body_pos, body_quat=m.body_quat, body_ipos=m.body_ipos, body_ilmat=body_ilmat,
            body_mass=m.body_mass, body_inertia=m.body_inertia, body_invweight0=m.body_invweight0,
            tree_mass=m.tree_mass,
            jnt_pos=m.jnt_pos, jnt_axis=m.jnt_axis, qpos0=m.qpos0, dof_damping=m.dof_damping,
            dof_armature=m.dof_armature, dof_invweight0=m.dof_invweight0,
            lim_range=np.append(m.jnt_range[lim].reshape(-1), [0.0, 0.0]), geom_pos=m.geom_pos, geom_lmat=geom_lmat,
            geom_size=m.geom_size, geom_friction=m.geom_friction, geom_rbound=m.geom_rbound, act_gain=act_gain,
            hfield=m.hfield_data)
        # one device buffer, 16-byte aligned slices
        chunks, offs, pos = [], {}, 0
        ints = {k: (v if np.asarray(v).dtype in (np.uint8, np.uint16, np.uint64) else np.asarray(v).astype(np.int32))
                for k, v in ints.items()}
        fields = {f for f, _ in N.ModelT._fields_}
        missing = {f for f, t in N.ModelT._fields_ if t is ctypes.c_void_p} - set(ints) - set(floats)
        if missing or (set(ints) | set(floats)) - fields:
            raise RuntimeError(f"model table mismatch with s3_model: {sorted(missing)}")
        for name, a in list(ints.items()) + [(k, np.asarray(v, dtype=self.ndtype)) for k, v in floats.items()]:
            b = np.ascontiguousarray(a).tobytes()
            offs[name] = pos
            chunks.append(b)
            pad = (-len(b)) % 16
            chunks.append(b"\0" * pad)
            pos += len(b) + pad
        self._float_names = list(floats)
        self._offs = offs
        host = np.frombuffer(b"".join(chunks), dtype=np.uint8).copy()
        self.buffer = torch.from_numpy(host).to(self.device)
        base = self.buffer.data_ptr()
        s = N.ModelT()
        s.dtype = code
        s.nbody, s.njnt, s.nq, s.nv = m.nbody, m.njnt, m.nq, m.nv
        s.ngeom, s.npair, s.nu, s.nlimjnt = m.ngeom, m.npair, m.nu, len(lim)
        s.nlevel, s.chain_stride, s.terrain_hfield = nlevel, self.chain_stride, m.terrain_is_hfield
        s.hf_nrow, s.hf_ncol = m.hfield_data.shape
        s.iterations, s.ls_iterations = m.opt.iterations, m.opt.ls_iterations
        s.nldl_norm = len(ldl_norm)
        s.ntree = len(tree_ent)
        s.nhlev, s.ndlev = len(hlev), len(dlev)
        # bit 0 off: partial Newton refactorization (only the subtrees a constraint touches); bits 3 + 5: block
        # phase sync at the start of each substep and after the Newton solve; bit 6 (latency-bound, large models):
        # balance warps per block over the waves of a launch -- measured defaults for both dtypes
        # (tools/ab_sim3d.sh); S3_FLAGS overrides
        s.flags = int(os.environ.get("S3_FLAGS", "40" if m.nv < 24 else "104"))  # bit 6: balanced waves
        if getattr(m.opt, "solver", "newton") == "cg":
            s.flags |= 128  # bit 7: conjugate-gradient solver (M^-1-preconditioned; its two vectors in the layout)
        elif getattr(m.opt, "solver", "newton") != "newton":
            raise ValueError(f"unknown solver {m.opt.solver!r} (newton or cg)")
        s.timestep = m.opt.timestep
        s.gravity[:] = m.opt.gravity
        s.tolerance, s.ls_tolerance = m.opt.tolerance, m.opt.ls_tolerance
        s.solref[:] = m.opt.solref
        s.solimp[:] = m.opt.solimp
        s.total_mass = float(m.body_mass[1:].sum())
        s.nkintree = m.ntree
        s.ncon_max = m.ncon_max
        s.nonroot_mask = sum(1 << d for d in range(m.nv) if m.dof_parentid[d] >= 0)
        s.nonleaf_mask = sum(1 << int(d) for d in set(m.dof_parentid.tolist()) if d >= 0)
        s.hf_spacing = m.hfield_spacing
        s.hf_origin[:] = m.hfield_origin
        s.hf_max = float(m.hfield_data.max())
        for name, off in offs.items():
            setattr(s, name, base + off)
        self.struct = s
        self.set_scale()
        self.layout = N.LayoutT()
        N.call("s3_plan", ctypes.byref(self.struct), int(os.environ.get("S3_WPB", "0")), ctypes.byref(self.layout))

    def set_scale(self):
        self.struct.scale = 1.0 / (self.model.meaninertia * max(1, self.model.nv))

    def upload_field(self, name: str, values: np.ndarray):
        """Overwrite one float table in place (inverse weights after set_const, randomized fields)."""
        a = np.ascontiguousarray(values, dtype=self.ndtype).reshape(-1)
        t = torch.from_numpy(a.view(np.uint8).copy()).to(self.device)
        off = self._offs[name]
        self.buffer[off:off + t.numel()].copy_(t)

    def set_const(self):
        """Inverse weights + mean inertia from the GPU mass matrix at qpos0 (model.set_const)."""
        m = self.model
        d = Data(self, 1)
        d.qpos[0] = torch.as_tensor(m.qpos0, dtype=self.tdtype)
        out = d.step(1, outputs=True)
        Mp = out["qM"][0].double().cpu().numpy()
        M = unpack_lower(Mp, m.nv)
        cdof = out["cdof"][0].double().cpu().numpy()
        xpos = out["xpos"][0].double().cpu().numpy()
        xquat = out["xquat"][0].double().cpu().numpy()
        coms = out["com"][0].double().cpu().numpy()
        jac = [np.zeros((3, m.nv))]
        for b in range(1, m.nbody):
            p = xpos[b] + quat2mat(xquat[b]) @ m.body_ipos[b]
            com = coms[m.body_treeid[b]]
            J = np.zeros((3, m.nv))
            for dd in m.body_chain[b]:
                J[:, dd] = cdof[dd, 3:] + np.cross(cdof[dd, :3], p - com)
            jac.append(J)
        m.set_const(M, jac)
        self.upload_field("dof_invweight0", m.dof_invweight0)
        self.upload_field("body_invweight0", m.body_invweight0)
        self.set_scale()
        return M


def unpack_lower(packed: np.ndarray, nv: int) -> np.ndarray:
    M = np.zeros((nv, nv))
    M[np.tril_indices(nv)] = packed
    return M + np.tril(M, -1).T


class Data:
    """Batched MjData-shaped state of N worlds (world index outermost)."""

    def __init__(self, dm: DeviceModel, nworld: int):
        m = dm.model
        self.dm = dm
        self.nworld = int(nworld)
        dev, dt = dm.device, dm.tdtype
        self.qpos = torch.tensor(np.tile(m.qpos0, (nworld, 1)), dtype=dt, device=dev)
        self.qvel = torch.zeros(nworld, m.nv, dtype=dt, device=dev)
        self.ctrl = torch.zeros(nworld, max(m.nu, 1), dtype=dt, device=dev)
        self.qacc_warmstart = torch.zeros(nworld, m.nv, dtype=dt, device=dev)
        self.qfrc_applied = None
        self.time = torch.zeros(nworld, dtype=dt, device=dev)
        self.friction_scale = None  # (N,) per-world friction multiplier (domain randomisation)
        self.mass_scale = None      # (N,) per-world scale of the base body's mass and inertia
        self.geom_xpos = None
        self.geom_xmat = None
        self._out = None

    def enable_geom_frames(self):
        m = self.dm.model
        self.geom_xpos = torch.zeros(self.nworld, m.ngeom, 3, dtype=self.dm.tdtype, device=self.dm.device)
        self.geom_xmat = torch.zeros(self.nworld, m.ngeom, 9, dtype=self.dm.tdtype, device=self.dm.device)

    def _outputs(self):
        if self._out is None:
            m, n, dt, dev = self.dm.model, self.nworld, self.dm.tdtype, self.dm.device
            np_ = m.nv * (m.nv + 1) // 2
            z = lambda *s: torch.zeros(*s, dtype=dt, device=dev)  # noqa: E731
            zi = lambda *s: torch.zeros(*s, dtype=torch.int32, device=dev)  # noqa: E731
            self._out = dict(xpos=z(n, m.nbody, 3), xquat=z(n, m.nbody, 4), com=z(n, N.S3_MAX_TREE, 3),
                             cdof=z(n, m.nv, 6),
                             qM=z(n, np_), qLD=z(n, np_), qfrc_bias=z(n, m.nv), qfrc_smooth=z(n, m.nv),
                             qacc_smooth=z(n, m.nv), qacc=z(n, m.nv), qfrc_constraint=z(n, m.nv),
                             ncon=zi(n), ndropped=zi(n), nefc=zi(n), con_pair=zi(n, MAX_CON),
                             con_dist=z(n, MAX_CON), con_pos=z(n, MAX_CON, 3), con_frame=z(n, MAX_CON, 9),
                             efc_force=z(n, MAX_ROWS), solver_niter=zi(n))
        return self._out

    def struct(self, outputs: bool):
        s = N.DataT()
        s.nworld = self.nworld
        for name in ("qpos", "qvel", "ctrl", "qacc_warmstart", "qfrc_applied", "time", "geom_xpos", "geom_xmat",
                     "friction_scale", "mass_scale"):
            t = getattr(self, name)
            setattr(s, name, None if t is None else t.data_ptr())
        if outputs:
            for k, t in self._outputs().items():
                setattr(s, k, t.data_ptr())
        return s

    def step(self, nsub: int = 1, outputs: bool = False, stream=None):
        """nsub physics substeps of every world in one launch (ctrl held). With outputs=True the last
        substep's intermediates (M, qLD, bias, contacts, forces, ...) are returned as tensors."""
        for name in ("qpos", "qvel", "ctrl", "qacc_warmstart"):
            t = getattr(self, name)
            if not t.is_contiguous() or t.dtype != self.dm.tdtype or t.device != self.dm.device:
                raise ValueError(f"{name} must be a contiguous {self.dm.tdtype} tensor on {self.dm.device}")
        s = self.struct(outputs)
        st = torch.cuda.current_stream(self.dm.device).cuda_stream if stream is None else stream
        N.call("s3_step", ctypes.byref(self.dm.struct), ctypes.byref(s), ctypes.byref(self.dm.layout), int(nsub), st,
               launch=True)
        return self._outputs() if outputs else None
