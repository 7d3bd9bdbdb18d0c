"""Reward manager (managers/reward.py): total = sum_i w_i * r_i * dt_control.

Term values, episodic sums and raw sums are (T, N) device arrays written by
the fused step; weights stay host floats (a curriculum schedule edits them
between steps, exactly like the reference's dict) and reach the kernel as
per-launch uniforms.
"""

from __future__ import annotations

import math

import numpy as np

from .. import native
from .base import REWARD_TERMS, ManagerError, RewardTermCfg, builtin_id, resolve


class _Rows(dict):
    """name -> (N,) row view of a (T, N) device array (dict API of the reference)."""


class _Weights(dict):
    """Host float weights (a dict, like the reference) mirrored into the
    native runtime's per-launch uniforms on every write."""

    def __init__(self, items, order):
        super().__init__(items)
        self._order = list(order)
        self._rt = None

    def bind(self, rt) -> None:
        self._rt = rt
        rt.n_rewards = len(self._order)
        for i, k in enumerate(self._order):
            rt.weight[i] = float(dict.__getitem__(self, k))

    def __setitem__(self, k, v) -> None:
        super().__setitem__(k, v)
        if self._rt is not None and k in self._order:
            self._rt.weight[self._order.index(k)] = float(v)


class RewardManager:
    def __init__(self, cfg: dict[str, RewardTermCfg], env):
        import torch

        self.env = env
        self.cfg = cfg
        self.terms = {}
        for name, tc in cfg.items():
            if not math.isfinite(tc.weight):
                raise ManagerError(f"reward term {name!r}: weight must be finite")
            self.terms[name] = resolve(REWARD_TERMS, tc.func, "reward")
        if len(self.terms) > native.SS_MAX_REWARDS:
            raise ManagerError(f"more than {native.SS_MAX_REWARDS} reward terms")
        self.weights = _Weights(((name, c.weight) for name, c in cfg.items()), cfg)
        n, t, dev = env.num_envs, max(1, len(cfg)), env.device
        z = lambda: torch.zeros((t, n), dtype=torch.float64, device=dev)  # noqa: E731
        self._sums, self._raw, self._last, self._final = z(), z(), z(), z()
        self.reward = torch.zeros(n, dtype=torch.float64, device=dev)
        names = list(cfg)
        self.episodic_sums = _Rows((k, self._sums[i]) for i, k in enumerate(names))
        self.episodic_raw = _Rows((k, self._raw[i]) for i, k in enumerate(names))
        self.last_values = _Rows((k, self._last[i]) for i, k in enumerate(names))
        self.finalized = _Rows((k, self._final[i]) for i, k in enumerate(names))
        self.external = {name: fn for name, fn in self.terms.items() if builtin_id(fn) is None}
        self._ext_buf = {name: torch.zeros(n, dtype=torch.float64, device=dev) for name in self.external}

    @property
    def nonfinite_report(self) -> dict:
        """{term: (N,) bool} for terms that produced NaN/Inf in the last compute."""
        import torch

        out = {}
        for name, v in self.last_values.items():
            bad = ~torch.isfinite(v)
            if bool(bad.any()):
                out[name] = bad
        return out

    def eval_external(self) -> None:
        """Evaluate user-registered (plugin) terms into their kernel inputs."""
        import torch

        for name, fn in self.external.items():
            v = fn(self.env, **self.cfg[name].params)
            self._ext_buf[name].copy_(torch.as_tensor(np.asarray(v) if not torch.is_tensor(v) else v,
                                                      dtype=torch.float64).reshape(-1).to(self.env.device))

    def compute(self, dt: float | None = None):
        """Weighted, dt-scaled sum of terms at the current state (managers/reward.py:36-49)."""
        if dt is not None and dt != self.env.dt_control:
            raise ManagerError("the device reward path scales by the env's dt_control")
        self.eval_external()
        self.env._launch(native.SS_ST_REWARD)
        return self.reward

    def mean_raw(self, name: str, ids, steps):
        import torch

        steps = torch.as_tensor(steps, dtype=torch.float64, device=self.env.device)
        return self.episodic_raw[name][ids] / torch.clamp(steps, min=1.0)

    def reset(self, ids) -> dict:
        """Finalize and clear episodic sums for the given worlds (managers/reward.py:55-62)."""
        import torch

        ids_t = torch.as_tensor(np.asarray(ids) if not torch.is_tensor(ids) else ids, device=self.env.device)
        out = {}
        for name in self.terms:
            out[name] = self.episodic_sums[name][ids_t].clone()
            self.episodic_sums[name][ids_t] = 0.0
            self.episodic_raw[name][ids_t] = 0.0
        return out

    def native_into(self, d) -> None:
        d.n_rewards = len(self.terms)
        ids = {"constant": 1, "std": 3, "feet": 9}
        for i, (name, fn) in enumerate(self.terms.items()):
            r = d.reward[i]
            sid = builtin_id(fn)
            p = self.cfg[name].params
            if sid is None:
                r.func = native.SS_REW_EXTERNAL
                r.ext = self._ext_buf[name].data_ptr()
            else:
                r.func = sid
                if sid == native.SS_REW_CONSTANT:
                    r.p0 = float(p.get("value", 1.0))
                elif sid == native.SS_REW_TRACK_VX_EXP:
                    r.p0 = float(p.get("std", 0.25))
                elif sid == native.SS_REW_FEET_AIR_TIME:
                    r.p0 = float(p.get("target_air_time", 0.3))
        del ids
        d.reward_out = self.reward.data_ptr()
        d.ep_sums = self._sums.data_ptr()
        d.ep_raw = self._raw.data_ptr()
        d.last_values = self._last.data_ptr()
        d.finalized = self._final.data_ptr()

