"""Termination manager (managers/termination.py): failure terms, the timeout
term and the NaN/Inf guard, evaluated per world inside the fused step.
Trigger counts are device int64 counters fed by warp-aggregated atomics and
read lazily (no per-step host sync)."""

from __future__ import annotations

from collections.abc import Mapping

import numpy as np

from .. import native
from .base import TERMINATION_TERMS, ManagerError, TerminationTermCfg, builtin_id, resolve


class _Counts(Mapping):
    """Read-through view of the device counters (dict of ints in the reference)."""

    def __init__(self, names, counts):
        self._names = list(names) + ["nonfinite"]
        self._counts = counts

    def _host(self):
        return self._counts.cpu().numpy()

    def __getitem__(self, key):
        return int(self._host()[self._names.index(key)])

    def __iter__(self):
        return iter(self._names)

    def __len__(self):
        return len(self._names)

    def items(self):
        h = self._host()
        return [(k, int(h[i])) for i, k in enumerate(self._names)]

    def values(self):
        h = self._host()
        return [int(h[i]) for i in range(len(self._names))]


class TerminationManager:
    def __init__(self, cfg: dict[str, TerminationTermCfg], env):
        import torch

        self.env = env
        self.cfg = cfg
        self.terms = {name: resolve(TERMINATION_TERMS, c.func, "termination") for name, c in cfg.items()}
        timeouts = [name for name, c in cfg.items() if c.time_out]
        if len(timeouts) > 1:
            raise ManagerError(f"at most one timeout term allowed, got {timeouts}")
        if len(self.terms) > native.SS_MAX_TERMINATIONS:
            raise ManagerError(f"more than {native.SS_MAX_TERMINATIONS} termination terms")
        self.timeout_term = timeouts[0] if timeouts else None
        n, dev = env.num_envs, env.device
        self._counts = torch.zeros(len(self.terms) + 1, dtype=torch.int64, device=dev)
        self.trigger_counts = _Counts(self.terms, self._counts)
        self.terminated = torch.zeros(n, dtype=torch.bool, device=dev)
        self.truncated = torch.zeros(n, dtype=torch.bool, device=dev)
        self.last_nonfinite = torch.zeros(n, dtype=torch.bool, device=dev)
        self.external = {name: fn for name, fn in self.terms.items() if builtin_id(fn) is None}
        self._ext_buf = {name: torch.zeros(n, dtype=torch.uint8, device=dev) for name in self.external}

    def eval_external(self) -> None:
        import torch

        for name, fn in self.external.items():
            m = fn(self.env, **self.cfg[name].params)
            m = torch.as_tensor(np.asarray(m) if not torch.is_tensor(m) else m).reshape(-1)
            self._ext_buf[name].copy_(m.to(device=self.env.device, dtype=torch.bool).to(torch.uint8))

    def compute(self):
        """(terminated, truncated) at the current state (managers/termination.py:24-41)."""
        self.eval_external()
        self.env._launch(native.SS_ST_TERM, flags=native.SS_FLAG_NO_EPISODE)
        return self.terminated, self.truncated

    def native_into(self, d) -> None:
        d.n_terms = len(self.terms)
        for i, (name, fn) in enumerate(self.terms.items()):
            t = d.term[i]
            sid = builtin_id(fn)
            t.time_out = int(bool(self.cfg[name].time_out))
            p = self.cfg[name].params
            if sid is None:
                t.func = native.SS_TERM_EXTERNAL
                t.ext = self._ext_buf[name].data_ptr()
            else:
                t.func = sid
                if sid == native.SS_TERM_BASE_HEIGHT_BELOW:
                    t.p0 = float(p.get("min_height", 0.15))
                elif sid == native.SS_TERM_PITCH_BEYOND:
                    t.p0 = float(p.get("max_pitch", 1.0))
        d.terminated = self.terminated.data_ptr()
        d.truncated = self.truncated.data_ptr()
        d.trigger_counts = self._counts.data_ptr()
