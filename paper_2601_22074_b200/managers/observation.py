"""Observation manager (managers/observation.py): groups of processed,
delayed, history-stacked terms.

Per-term pipeline (raw -> clip -> scale -> noise -> delay -> history) runs
per world in the fused step and writes each group's row-major (N, D) output
directly. Delay and history rings are device arrays indexed by host-tracked
heads (the reference shifts the history physically; a ring with a head
gives the same oldest-first output without moving data). Reset worlds flood
both rings with the reset-time value.
"""

from __future__ import annotations

import numpy as np

from .. import native
from .base import (
    MAX_DELAY_STEPS,
    MAX_HISTORY,
    OBSERVATION_TERMS,
    ManagerError,
    ObsGroupCfg,
    ObsTermCfg,
    builtin_id,
    resolve,
)

_NOISE = {"none": native.SS_NOISE_NONE, "uniform": native.SS_NOISE_UNIFORM, "gaussian": native.SS_NOISE_GAUSSIAN}


def builtin_obs_dim(sid: int, env) -> int:
    k = env.model.num_joints
    return {
        native.SS_OBS_BASE_LIN_VEL: 2,
        native.SS_OBS_BASE_ANG_VEL: 1,
        native.SS_OBS_BASE_LIN_ACC: 2,
        native.SS_OBS_PROJECTED_GRAVITY: 2,
        native.SS_OBS_JOINT_POS_REL: k,
        native.SS_OBS_JOINT_VEL: k,
        native.SS_OBS_LAST_ACTION: env.action_manager.total_dim,
        native.SS_OBS_COMMAND: len(env.command_manager.channels),
        native.SS_OBS_BASE_HEIGHT: 1,
        native.SS_OBS_SIM_TIME: 1,
        native.SS_OBS_HEIGHT_SCAN: len(env.cfg.scene.ray_scan.offsets),
        native.SS_OBS_FOOT_CONTACT_FORCES: 2 * len(env.model.feet),
    }[sid]


def _as_rows(v, n, device):
    import torch

    t = torch.as_tensor(np.asarray(v) if not torch.is_tensor(v) else v, dtype=torch.float64).to(device)
    if t.dim() == 1:
        t = t.reshape(-1, 1) if t.shape[0] == n else t.reshape(1, -1)
    if t.shape[0] != n:
        t = t.T
    return t


class _ObsTerm:
    def __init__(self, group: str, name: str, cfg: ObsTermCfg, env):
        import torch

        self.name = name
        self.cfg = cfg
        self.func = resolve(OBSERVATION_TERMS, cfg.func, "observation")
        if cfg.clip is not None and not cfg.clip[0] < cfg.clip[1]:
            raise ManagerError(f"obs term {name!r}: clip range must be ordered")
        if not 0 <= cfg.delay_steps <= MAX_DELAY_STEPS:
            raise ManagerError(f"obs term {name!r}: delay_steps outside [0, {MAX_DELAY_STEPS}]")
        if not 1 <= cfg.history <= MAX_HISTORY:
            raise ManagerError(f"obs term {name!r}: history outside [1, {MAX_HISTORY}]")
        if cfg.noise.kind not in _NOISE:
            raise ManagerError(f"unknown noise kind {cfg.noise.kind!r}")
        self.sid = builtin_id(self.func)
        n = env.num_envs
        if self.sid is None:
            probe = _as_rows(self.func(env, **cfg.params), n, env.device)
            self.dim = int(probe.shape[1])
        else:
            self.dim = builtin_obs_dim(self.sid, env)
        max_dim = max(native.SS_MAX_JOINTS, 2 * native.SS_MAX_FEET)
        if self.dim > max_dim:
            raise ManagerError(f"obs term {name!r}: dim {self.dim} exceeds the sm_100a build ({max_dim})")
        self.noise_purpose = f"obs.{group}.{name}"
        self._heads = [0, cfg.history - 1]
        self._rt = None
        self._rt_idx = 0
        dev = env.device
        self._dring = (torch.zeros((cfg.delay_steps + 1, self.dim, n), dtype=torch.float64, device=dev)
                       if cfg.delay_steps > 0 else None)
        self._hring = (torch.zeros((cfg.history, self.dim, n), dtype=torch.float64, device=dev)
                       if cfg.history > 1 else None)
        self.ext = torch.zeros((n, self.dim), dtype=torch.float64, device=dev) if self.sid is None else None
        self.out_dim = self.dim * cfg.history

    def bind(self, rt, idx: int, group_idx: int) -> None:
        self._rt, self._rt_idx = rt, idx
        rt.obs_group[idx] = group_idx
        rt.obs_delay_len[idx] = self.cfg.delay_steps + 1
        rt.obs_hist_len[idx] = self.cfg.history
        rt.obs_delay_head[idx] = self._heads[0]
        rt.obs_hist_head[idx] = self._heads[1]

    @property
    def delay_head(self) -> int:
        return self._rt.obs_delay_head[self._rt_idx] if self._rt is not None else self._heads[0]

    @property
    def hist_head(self) -> int:
        return self._rt.obs_hist_head[self._rt_idx] if self._rt is not None else self._heads[1]


class ObservationManager:
    """Computes observation groups once per control step (cached by global_step)."""

    def __init__(self, groups: dict[str, ObsGroupCfg], env):
        import torch

        self.env = env
        self.group_cfgs = groups
        self.groups: dict[str, list[_ObsTerm]] = {}
        if len(groups) > native.SS_MAX_GROUPS:
            raise ManagerError(f"more than {native.SS_MAX_GROUPS} observation groups")
        n, dev = env.num_envs, env.device
        self._out: dict[str, object] = {}
        self._pending: dict[str, object] = {}
        for g, gc in groups.items():
            self.groups[g] = [_ObsTerm(g, name, tc, env) for name, tc in gc.terms.items()]
            self._out[g] = torch.zeros((n, self.group_dim(g)), dtype=torch.float64, device=dev)
            self._pending[g] = torch.zeros(n, dtype=torch.uint8, device=dev)
        if sum(len(t) for t in self.groups.values()) > native.SS_MAX_OBS_TERMS:
            raise ManagerError(f"more than {native.SS_MAX_OBS_TERMS} observation terms")
        self._any_pending = False
        self._rt = None
        self._bad = torch.zeros(n, dtype=torch.int32, device=dev)
        self._cache: dict[str, int] = {}
        self._report_terms: list[str] = []

    def bind(self, rt) -> None:
        """Hand the ring heads and the pending flag to the native runtime."""
        self._rt = rt
        names = list(self.groups)
        rt.n_groups = len(names)
        i = 0
        for g, terms in self.groups.items():
            for t in terms:
                t.bind(rt, i, names.index(g))
                i += 1
        rt.n_obs = i
        rt.any_pending = int(self._any_pending)

    @property
    def any_pending(self) -> bool:
        return bool(self._rt.any_pending) if self._rt is not None else self._any_pending

    @any_pending.setter
    def any_pending(self, v: bool) -> None:
        if self._rt is not None:
            self._rt.any_pending = int(v)
        else:
            self._any_pending = bool(v)

    def group_dim(self, group: str) -> int:
        return sum(t.out_dim for t in self.groups[group])

    def all_terms(self):
        return [t for g in self.groups.values() for t in g]

    @property
    def has_external(self) -> bool:
        return any(t.sid is None for t in self.all_terms())

    def mark_reset(self, ids) -> None:
        import torch

        ids_t = torch.as_tensor(np.asarray(ids) if not torch.is_tensor(ids) else ids, device=self.env.device)
        for p in self._pending.values():
            p[ids_t] = 1
        self.any_pending = True
        self._cache.clear()

    def eval_external(self, groups) -> None:
        for g in groups:
            for t in self.groups[g]:
                if t.sid is None:
                    t.ext.copy_(_as_rows(t.func(self.env, **t.cfg.params), self.env.num_envs, self.env.device))

    def begin(self, groups) -> int:
        """Host bookkeeping before an OBS launch (the runtime advances the ring
        heads of the masked groups); returns the group mask."""
        mask = 0
        names = list(self.groups)
        step = self.env.global_step
        for g in groups:
            mask |= 1 << names.index(g)
            self._cache[g] = step
        return mask

    def begin_all(self) -> int:
        """begin() for every group (the fused step)."""
        step = self.env.global_step
        for g in self.groups:
            self._cache[g] = step
        return (1 << len(self.groups)) - 1

    def compute(self, group: str):
        """Group output (N, sum of term dims x history) (managers/observation.py:99-137)."""
        if group not in self.groups:
            raise ManagerError(f"unknown observation group {group!r}; have {list(self.groups)}")
        if self._cache.get(group) == self.env.global_step:
            return self._out[group]
        self.eval_external([group])
        mask = self.begin([group])
        self.env._launch(native.SS_ST_OBS, groups_mask=mask)
        self._report_terms = [t.name for t in self.groups[group]]
        return self._out[group]

    def compute_all(self) -> dict:
        self._cache.clear()
        self.eval_external(list(self.groups))
        mask = self.begin(list(self.groups))
        self.env._launch(native.SS_ST_OBS, groups_mask=mask)
        return self.outputs()

    def outputs(self) -> dict:
        return dict(self._out)

    @property
    def nonfinite_report(self) -> dict:
        """{term: (N,) bool} for terms whose raw value had NaN/Inf in the last compute."""
        out = {}
        bad = self._bad
        for i, t in enumerate(self.all_terms()):
            m = ((bad >> i) & 1).bool()
            if bool(m.any()):
                out[t.name] = m
        return out

    def native_into(self, d) -> None:
        d.n_groups = len(self.groups)
        ti = 0
        for gi, (g, terms) in enumerate(self.groups.items()):
            G = d.group[gi]
            G.out = self._out[g].data_ptr()
            G.pending = self._pending[g].data_ptr()
            G.dim = self.group_dim(g)
            G.first_term = ti
            G.n_terms = len(terms)
            G.enable_noise = int(bool(self.group_cfgs[g].enable_noise))
            col = 0
            for t in terms:
                T = d.obs[ti]
                T.func = native.SS_OBS_EXTERNAL if t.sid is None else t.sid
                T.dim = t.dim
                T.group = gi
                T.col = col
                tc = t.cfg
                if tc.clip is not None:
                    T.has_clip = 1
                    T.clip_lo, T.clip_hi = float(tc.clip[0]), float(tc.clip[1])
                if tc.scale is not None:
                    T.has_scale = 1
                    T.scale = float(tc.scale)
                if self.group_cfgs[g].enable_noise and tc.noise.kind != "none" and tc.noise.scale:
                    T.noise = _NOISE[tc.noise.kind]
                    T.noise_scale = float(tc.noise.scale)
                    T.noise_slot = self.env.streams.slot(t.noise_purpose)
                T.delay = tc.delay_steps
                T.history = tc.history
                T.delay_ring = None if t._dring is None else t._dring.data_ptr()
                T.hist_ring = None if t._hring is None else t._hring.data_ptr()
                T.ext = None if t.ext is None else t.ext.data_ptr()
                col += t.out_dim
                ti += 1
        d.n_obs_terms = ti
        d.obs_bad = self._bad.data_ptr()
