"""Scene entities and their derived kinematics (entity.py of the reference).

``EntityData`` is the read-only window terms see. Inside the fused step the
kernel keeps the reference's refresh-point snapshot in registers; from
Python every field is derived on access from the current device state (the
copies the reference refreshes after each substep are views or one fused
torch expression here, so nothing extra is written to HBM per step).
"""

from __future__ import annotations

import re
from dataclasses import dataclass

import numpy as np


class EntityError(ValueError):
    pass


@dataclass
class DefaultState:
    base_pose: tuple[float, float, float] = (0.0, 0.5, 0.0)
    base_vel: tuple[float, float, float] = (0.0, 0.0, 0.0)
    joint_pos: tuple[float, ...] = ()
    joint_vel: tuple[float, ...] = ()


class Entity:
    """A named scene object with regex-resolvable joints (entity.py:41-105)."""

    def __init__(self, name: str, joint_names=None, default_state: DefaultState | None = None,
                 base_type: str = "floating", pos_limits=None):
        if base_type not in ("fixed", "floating"):
            raise EntityError(f"base_type must be 'fixed' or 'floating', got {base_type!r}")
        self.name = name
        self.joint_names = list(joint_names or [])
        self.body_names = [f"{name}_base"] + [f"{j}_link" for j in self.joint_names]
        self.base_type = base_type
        self.default_state = default_state or DefaultState()
        k = len(self.joint_names)
        if len(self.default_state.joint_pos) not in (0, k):
            raise EntityError(f"default joint_pos has {len(self.default_state.joint_pos)} entries for {k} joints")
        if pos_limits is not None and k:
            pos = np.asarray(self.default_state.joint_pos or np.zeros(k))
            if np.any(pos < pos_limits[:, 0]) or np.any(pos > pos_limits[:, 1]):
                raise EntityError("default joint positions violate position limits")

    @property
    def is_fixed_base(self) -> bool:
        return self.base_type == "fixed"

    @property
    def is_articulated(self) -> bool:
        return len(self.joint_names) > 0

    def find_joints(self, patterns) -> list[int]:
        hits: list[int] = []
        for pat in patterns:
            rx = re.compile(pat)
            hits.extend(i for i, nm in enumerate(self.joint_names) if rx.fullmatch(nm) and i not in hits)
        if not hits:
            raise EntityError(
                f"patterns {patterns!r} match no joints of {self.name!r}; "
                f"available: {', '.join(self.joint_names) or 'none'}"
            )
        return sorted(hits)

    def write_default_state(self, state, world_ids) -> None:
        """Reset q/qd/time of the listed worlds only (entity.py:91-105)."""
        import torch

        ids = torch.as_tensor(np.asarray(world_ids) if not torch.is_tensor(world_ids) else world_ids,
                              dtype=torch.int64).reshape(-1)
        if ids.numel() and (int(ids.min()) < 0 or int(ids.max()) >= state.n_worlds):
            raise EntityError(f"world ids {ids.tolist()} outside [0, {state.n_worlds})")
        ids = ids.to(state.device)
        ds = self.default_state
        dev = state.device
        state.q[ids, 0:3] = torch.as_tensor(ds.base_pose, dtype=torch.float64, device=dev)
        state.qd[ids, 0:3] = torch.as_tensor(ds.base_vel, dtype=torch.float64, device=dev)
        k = state.nq - 3
        if k:
            state.q[ids, 3:] = torch.as_tensor(ds.joint_pos or (0.0,) * k, dtype=torch.float64, device=dev)
            state.qd[ids, 3:] = torch.as_tensor(ds.joint_vel or (0.0,) * k, dtype=torch.float64, device=dev)
        state.time[ids] = 0.0


class EntityData:
    """Derived kinematics of the robot entity, one row per world."""

    def __init__(self, model, state=None):
        self._model = model
        self._state = state

    def refresh(self, model, state) -> None:
        self._model = model
        self._state = state

    def _qs(self):
        return self._state.q, self._state.qd

    root_pos = property(lambda self: self._state.q[:, 0:2])
    root_pitch = property(lambda self: self._state.q[:, 2])
    root_lin_vel_w = property(lambda self: self._state.qd[:, 0:2])
    root_ang_vel = property(lambda self: self._state.qd[:, 2])
    joint_pos = property(lambda self: self._state.q[:, 3:])
    joint_vel = property(lambda self: self._state.qd[:, 3:])
    foot_in_contact = property(lambda self: self._state.contact.in_contact)
    foot_vel = property(lambda self: self._state.contact.foot_vel)

    @property
    def root_lin_vel_b(self):
        """R(pitch)^T v_world (entity.py:153-155)."""
        import torch

        q, qd = self._qs()
        c, s = torch.cos(q[:, 2]), torch.sin(q[:, 2])
        return torch.stack([c * qd[:, 0] + s * qd[:, 1], -s * qd[:, 0] + c * qd[:, 1]], dim=1)

    @property
    def projected_gravity(self):
        import torch

        p = self._state.q[:, 2]
        return torch.stack([-torch.sin(p), -torch.cos(p)], dim=1)

    @property
    def foot_forces(self):
        """(N, F, 2): (tangent, normal) per foot."""
        import torch

        c = self._state.contact
        return torch.stack([c.tangent_force, c.normal_force], dim=-1)

    @property
    def body_pos(self):
        """(N, 1 + k, 2): base + each link tip, via the FK kernel."""
        import torch

        from .sim.physics import fk_batch

        _, _, tips = fk_batch(self._model, self._state.q)
        return torch.cat([self._state.q[:, None, 0:2], tips], dim=1)
