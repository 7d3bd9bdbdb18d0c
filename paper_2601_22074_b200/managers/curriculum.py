"""Curriculum manager (managers/curriculum.py): difficulty adjustments.

World-scoped built-ins (terrain_levels, command_widen) run inside the fused
step on the worlds being reset, before their reset; schedule terms depend
only on ``global_step`` and run on the host (they edit host reward weights).
User-registered terms are called from Python with the reset ids.
"""

from __future__ import annotations

import numpy as np

from .. import native
from .base import CURRICULUM_TERMS, CurriculumTermCfg, ManagerError, builtin_id, resolve

HOST_TERMS = ("reward_weight_schedule",)


class CurriculumManager:
    def __init__(self, cfg: dict[str, CurriculumTermCfg], env):
        self.env = env
        self.cfg = cfg
        self.terms = {name: resolve(CURRICULUM_TERMS, c.func, "curriculum") for name, c in cfg.items()}
        n_dev = sum(1 for fn in self.terms.values() if builtin_id(fn) not in (None, 0))
        if n_dev > native.SS_MAX_CURRICULUM:
            raise ManagerError(f"more than {native.SS_MAX_CURRICULUM} device curriculum terms")

    def kind(self, name: str) -> str:
        sid = builtin_id(self.terms[name])
        if sid is None:
            return "external"
        return "host" if sid == 0 else "device"

    @property
    def has_external(self) -> bool:
        return any(self.kind(n) == "external" for n in self.terms)

    def update(self, reset_ids) -> None:
        """All terms on the given worlds, in registration order (curriculum.py:21-23)."""
        import torch

        ids = torch.as_tensor(np.asarray(reset_ids) if not torch.is_tensor(reset_ids) else reset_ids,
                              device=self.env.device).to(torch.int64).reshape(-1)
        if any(self.kind(n) == "device" for n in self.terms):
            mask = torch.zeros(self.env.num_envs, dtype=torch.uint8, device=self.env.device)
            mask[ids] = 1
            self.env._launch(native.SS_ST_CURRICULUM | native.SS_ST_RESET_EXT, reset_mask=mask)
        for name, fn in self.terms.items():
            if self.kind(name) != "device":
                fn(self.env, ids, **self.cfg[name].params)

    def run_host(self, reset_ids=None) -> None:
        """Host-side terms after a fused step (their result feeds the next step)."""
        host = self.__dict__.get("_host_terms")
        if host is None:  # the term set is fixed at construction
            host = self._host_terms = [(fn, self.cfg[name].params) for name, fn in self.terms.items()
                                       if self.kind(name) == "host"]
        for fn, params in host:
            fn(self.env, reset_ids, **params)

    def run_external(self, reset_ids) -> None:
        for name, fn in self.terms.items():
            if self.kind(name) == "external":
                fn(self.env, reset_ids, **self.cfg[name].params)

    def native_into(self, d) -> None:
        i = 0
        for name, fn in self.terms.items():
            if self.kind(name) != "device":
                continue
            c = d.curriculum[i]
            sid = builtin_id(fn)
            p = self.cfg[name].params
            c.func = sid
            if sid == native.SS_CUR_TERRAIN_LEVELS:
                c.p0 = float(p.get("promote_ratio", 0.8))
                c.p1 = float(p.get("demote_ratio", 0.4))
            elif sid == native.SS_CUR_COMMAND_WIDEN:
                term = p.get("term", "track_vx_exp")
                names = list(self.env.reward_manager.terms)
                if term not in names:
                    raise ManagerError(f"command_widen: unknown reward term {term!r}")
                c.term = names.index(term)
                c.p0 = float(p.get("threshold", 0.8))
                c.p1 = float(p.get("factor", 1.2))
            i += 1
        d.n_curriculum = i
