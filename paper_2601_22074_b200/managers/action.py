"""Action manager (managers/action.py of the reference) over device buffers.

``process`` (history update, clip, per-term targets) and ``apply`` (actuator
stacks -> ctrl, once per substep) are stages of the fused step kernel; the
standalone methods launch just that stage.
"""

from __future__ import annotations

import numpy as np

from .. import native
from ..actuators import Actuator
from .base import ActionTermCfg, ManagerError


class _ActionTerm:
    def __init__(self, name: str, cfg: ActionTermCfg, env, start: int):
        self.name = name
        self.cfg = cfg
        self.joint_ids = np.array(env.robot.find_joints(cfg.joint_patterns), dtype=np.int64)
        self.dim = len(self.joint_ids)
        self.slice = slice(start, start + self.dim)
        if cfg.offset_mode == "default":
            self.offset = np.asarray(env.default_joint_pos, dtype=np.float64)[self.joint_ids]
        elif cfg.offset_mode == "zero":
            self.offset = np.zeros(self.dim)
        else:
            raise ManagerError(f"action term {name!r}: unknown offset_mode {cfg.offset_mode!r}")
        self.actuators: list[Actuator] = []
        for act_name, act_cfg in cfg.actuators.items():
            patterns = act_cfg.joint_patterns
            if act_cfg.kind == "delayed" and not patterns:
                patterns = act_cfg.inner.joint_patterns
            ids = np.array(env.robot.find_joints(patterns), dtype=np.int64)
            outside = set(ids.tolist()) - set(self.joint_ids.tolist())
            if outside:
                raise ManagerError(f"actuator {act_name!r} drives joints {sorted(outside)} outside action term {name!r}")
            self.actuators.append(Actuator(f"{name}.{act_name}", act_cfg, env.model, ids, env.streams))


class ActionManager:
    def __init__(self, cfg: dict[str, ActionTermCfg], env):
        import torch

        self.env = env
        self.terms: dict[str, _ActionTerm] = {}
        start = 0
        for name, tcfg in cfg.items():
            t = _ActionTerm(name, tcfg, env, start)
            self.terms[name] = t
            start += t.dim
        self.total_dim = start
        if start > native.SS_MAX_ACTION or len(self.terms) > native.SS_MAX_ACTION_TERMS:
            raise ManagerError("action space exceeds the sm_100a build limits")
        driven: set[int] = set()
        for t in self.terms.values():
            for a in t.actuators:
                overlap = driven & set(a.joint_ids.tolist())
                if overlap:
                    raise ManagerError(f"joints {sorted(overlap)} driven by two actuators")
                driven |= set(a.joint_ids.tolist())
        if sum(len(t.actuators) for t in self.terms.values()) > native.SS_MAX_ACTUATORS:
            raise ManagerError(f"more than {native.SS_MAX_ACTUATORS} actuators")
        n, dev = env.num_envs, env.device
        self._action = torch.zeros((start, n), dtype=torch.float64, device=dev)
        self._prev = torch.zeros((start, n), dtype=torch.float64, device=dev)
        self._targets = torch.zeros((env.model.num_joints, n), dtype=torch.float64, device=dev)
        for t in self.terms.values():
            self.targets[:, t.joint_ids] = torch.as_tensor(t.offset, device=dev)

    action = property(lambda self: self._action.t())
    prev_action = property(lambda self: self._prev.t())
    targets = property(lambda self: self._targets.t())

    @property
    def actuators(self) -> list[Actuator]:
        return [a for t in self.terms.values() for a in t.actuators]

    def check_actions(self, actions):
        """Validate and stage a (N, total_dim) float64 CUDA tensor."""
        import torch

        from ..policies import RandomActions

        if actions.__class__ is torch.Tensor:
            # fast path: the common well-formed inputs (a few C-level checks)
            a = actions
            if a.dtype is torch.float64 and a.shape == self._shape and a.is_contiguous():
                dev = a.get_device()
                if dev == self._dev_index or (dev < 0 and self._pinned(a)):
                    return a
        if isinstance(actions, RandomActions):
            return actions
        if torch.is_tensor(actions):
            a = actions
        else:
            a = torch.as_tensor(np.asarray(actions, dtype=np.float64))
        if tuple(a.shape) != (self.env.num_envs, self.total_dim):
            raise ManagerError(
                f"action shape {tuple(a.shape)} does not match expected "
                f"{(self.env.num_envs, self.total_dim)} (sum of term dims)"
            )
        if a.device.type == "cpu" and a.dtype == torch.float64 and a.is_contiguous() and self._pinned(a):
            # pinned host rows are read by the step kernel in place over PCIe
            # (mapped memory): no separate host->device copy. Keep the buffer
            # unchanged until the step has completed on the stream.
            return a
        if a.dtype != torch.float64 or a.device != self.env.device or not a.is_contiguous():
            a = a.to(device=self.env.device, dtype=torch.float64).contiguous()
        return a

    @property
    def _shape(self):
        return (self.env.num_envs, self.total_dim)

    @property
    def _dev_index(self) -> int:
        return self.env._dev_index

    def _pinned(self, a) -> bool:
        """is_pinned() with a small cache of known pinned storages (the query
        is a driver call); cached entries hold a reference, so a cached range
        cannot be freed and reused by pageable memory."""
        p = a.data_ptr()
        cache = self.__dict__.setdefault("_pinned_cache", [])
        for lo, hi, _ref in cache:
            if lo <= p and p + a.numel() * 8 <= hi:
                return True
        if not a.is_pinned():
            return False
        st = a.untyped_storage()
        cache.insert(0, (st.data_ptr(), st.data_ptr() + st.nbytes(), a))
        del cache[4:]
        return True

    def process(self, actions) -> None:
        """Stage 1: history update, optional clip, per-term targets (managers/action.py:68-82)."""
        a = self.check_actions(actions)
        self.env._launch(native.SS_ST_ACTION, actions=a)

    def apply(self) -> None:
        """One substep of targets -> actuators -> ctrl (managers/action.py:84-90)."""
        self.env._launch(native.SS_ST_APPLY, nsub=1)

    def reset(self, ids) -> None:
        import torch

        ids_t = torch.as_tensor(np.asarray(ids), device=self.env.device, dtype=torch.int64)
        self.action[ids_t] = 0.0
        self.prev_action[ids_t] = 0.0
        for t in self.terms.values():
            jt = torch.as_tensor(t.joint_ids, device=self.env.device)
            self.targets[ids_t[:, None], jt[None, :]] = torch.as_tensor(t.offset, device=self.env.device)
            for a in t.actuators:
                a.reset(ids_t, self.targets)

    # -- host-side ring bookkeeping for the fused kernel ------------------------

    def bind(self, rt) -> None:
        """Hand the delay-ring heads to the native runtime (ss_rt_launch advances them)."""
        acts = self.actuators
        rt.n_act = len(acts)
        for i, a in enumerate(acts):
            if a.delay is not None:
                a.delay.bind(rt, i)
            else:
                rt.act_head[i] = 0
                rt.act_cap[i] = 0

    def native_into(self, d) -> None:
        d.n_action_terms = len(self.terms)
        d.action_dim = self.total_dim
        for i, t in enumerate(self.terms.values()):
            at = d.action_term[i]
            at.dim = t.dim
            at.start = t.slice.start
            for k, j in enumerate(t.joint_ids):
                at.joint[k] = int(j)
                at.offset[k] = float(t.offset[k])
            at.scale = float(t.cfg.scale)
            if t.cfg.clip is not None:
                at.has_clip = 1
                at.clip_lo, at.clip_hi = float(t.cfg.clip[0]), float(t.cfg.clip[1])
        d.action = self._action.data_ptr()
        d.prev_action = self._prev.data_ptr()
        d.targets = self._targets.data_ptr()
        acts = self.actuators
        d.n_actuators = len(acts)
        for i, a in enumerate(acts):
            a.native_into(d.actuator[i])
