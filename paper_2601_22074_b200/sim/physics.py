"""Physics sub-boundary: StepPipeline.substep and kinematics on the GPU.

``StepPipeline(model, terrain).substep(state)`` advances every world by one
physics_dt exactly like the reference (sim/physics.py:133-254): contact at
the start-of-substep state, generalized forces, semi-implicit Euler, contact
cache, time += dt. It is one launch of the fused step kernel restricted to
the PHYS stage. The pipeline re-specializes (rebuilds its descriptor) when
the model layout changes, and ``generation`` tracks the model's.
"""

from __future__ import annotations

import numpy as np

from .. import native
from .model import Model
from .state import BatchState


def _flat_terrain_desc(t) -> None:
    t.samples = None
    t.n_samples = 0
    t.spacing = 1.0
    t.flat = 1
    t.rows = 1
    t.cols = 1
    t.patch_length = 0.0


class StepPipeline:
    """Specialized substep over the model's current field layout."""

    def __init__(self, model: Model, terrain=None, transient: bool = False):
        self.model = model
        self.terrain = terrain
        self._descs: dict[int, tuple] = {}
        self._built_generation = -1
        if not transient:
            model.on_layout_change(self._rebuild)
        self._rebuild()

    @property
    def generation(self) -> int:
        return self.model.generation

    def _rebuild(self) -> None:
        self._descs.clear()
        self._built_generation = self.model.generation

    def _desc(self, state: BatchState):
        key = id(state)
        entry = self._descs.get(key)
        if entry is None or entry[0] is not state or self._built_generation != self.model.generation:
            if self._built_generation != self.model.generation:
                self._rebuild()
            d = native.EnvDesc()
            d.abi_version = native.SS_ABI_VERSION
            d.n_worlds = self.model.n_worlds
            d.decimation = 1
            d.dt_control = self.model.physics_dt
            self.model.native_into(d)
            if self.terrain is None:
                _flat_terrain_desc(d.terrain)
            else:
                d.terrain = self.terrain.native(self.model.device)
            state.native_into(d.state)
            entry = (state, d)
            self._descs[key] = entry
        return entry[1]

    def substep(self, state: BatchState) -> None:
        """Advance every world by one physics_dt (in place, asynchronous)."""
        d = self._desc(state)
        u = native.Uniforms()
        u.stages = native.SS_ST_PHYS
        u.nsub = 1
        u.sim_step = state.sim_step
        native.call("ss_env_step", native.byref(d), native.byref(u), native.current_stream(self.model.device))
        state.sim_step += 1


def physics_step(model: Model, state: BatchState, terrain=None) -> None:
    """One-off substep without keeping a pipeline around (sim/physics.py:252-254)."""
    StepPipeline(model, terrain, transient=True).substep(state)


def _as_rows(model: Model, q):
    import torch

    t = torch.as_tensor(q, dtype=torch.float64, device=model.device)
    if t.dim() == 1:
        t = t.reshape(1, -1)
    return t.contiguous()


def fk_batch_trig(model: Model, q):
    """(thetas (N,k), attach (N,k,2), tips (N,k,2), sin, cos) (sim/physics.py:22-57)."""
    import torch

    qr = _as_rows(model, q)
    n, k = qr.shape[0], model.num_joints
    th = torch.empty((n, k), dtype=torch.float64, device=model.device)
    attach = torch.empty((n, k, 2), dtype=torch.float64, device=model.device)
    tips = torch.empty((n, k, 2), dtype=torch.float64, device=model.device)
    d = native.EnvDesc()
    model.native_into(d)
    native.call("ss_fk", native.byref(d), qr.data_ptr(), th.data_ptr(), attach.data_ptr(), tips.data_ptr(), n,
                native.current_stream(model.device))
    return th, attach, tips, torch.sin(th), torch.cos(th)


def fk_batch(model: Model, q):
    th, attach, tips, _, _ = fk_batch_trig(model, q)
    return th, attach, tips


def forward_kinematics(model: Model, q_row):
    """Base pose (3,) and link tips (k, 2) for one configuration row."""
    q_row = np.asarray(q_row.cpu() if hasattr(q_row, "cpu") else q_row, dtype=np.float64)
    if q_row.shape != (model.nq,):
        raise ValueError(f"expected q of shape ({model.nq},), got {q_row.shape}")
    _, _, tips = fk_batch(model, q_row[None, :])
    return q_row[:3].copy(), tips[0].cpu().numpy()
