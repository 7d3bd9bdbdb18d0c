"""Event manager (managers/event.py): startup / reset / interval hooks.

Built-in reset and interval events (push, joint jitter, field randomization)
run per world inside the fused step; the per-world stopwatch and quantized
targets live on the device. Startup events and direct calls go through the
same device streams (``randomize_field`` is one ``ss_randomize`` launch).
User-registered event terms are called from Python with the world ids.
"""

from __future__ import annotations

import numpy as np

from .. import native
from .base import EVENT_TERMS, EventTermCfg, ManagerError, builtin_id, resolve

_DIST = {"uniform": native.SS_DIST_UNIFORM, "gaussian": native.SS_DIST_GAUSSIAN}
_OPS = {"set": native.SS_OP_SET, "scale": native.SS_OP_SCALE, "add": native.SS_OP_ADD}


def randomize_field(model, streams, field: str, distribution: str, rng_range, operation: str, world_ids,
                    purpose: str) -> None:
    """Expand (if needed) and redraw a model field for the listed worlds
    (managers/event.py:19-52). Draws apply against the compile-time base."""
    import torch

    if distribution not in _DIST:
        raise ManagerError(f"unknown distribution {distribution!r}")
    if operation not in _OPS:
        raise ManagerError(f"unknown field operation {operation!r}")
    model.expand_field(field)
    idx = model.field_index(field)
    ids = torch.as_tensor(np.asarray(world_ids) if not torch.is_tensor(world_ids) else world_ids,
                          device=model.device).to(torch.int64).reshape(-1).contiguous()
    if ids.numel() == 0:
        return
    slot = streams.slot(purpose)
    d = native.EnvDesc()
    d.abi_version = native.SS_ABI_VERSION
    d.n_worlds = model.n_worlds
    model.native_into(d)
    d.rng.world_id_offset = streams.world_id_offset
    d.rng.base[slot] = streams.bases[slot]
    d.rng.counter[slot] = streams.counters[slot].data_ptr()
    native.call("ss_randomize", native.byref(d), idx, _DIST[distribution], float(rng_range[0]),
                float(rng_range[1]), _OPS[operation], slot, ids.data_ptr(), int(ids.numel()),
                native.current_stream(model.device))


class EventManager:
    def __init__(self, cfg: dict[str, EventTermCfg], env):
        import torch

        self.env = env
        self.cfg = cfg
        self.terms = {}
        self._elapsed: dict[str, object] = {}
        self._target: dict[str, object] = {}
        self._fired: dict[str, object] = {}
        if len(cfg) > native.SS_MAX_EVENTS:
            raise ManagerError(f"more than {native.SS_MAX_EVENTS} event terms")
        for name, tc in cfg.items():
            if tc.mode not in ("startup", "reset", "interval"):
                raise ManagerError(f"event {name!r}: unknown mode {tc.mode!r}")
            self.terms[name] = resolve(EVENT_TERMS, tc.func, "event")
            if tc.mode == "interval":
                r = tc.interval_range
                if r is None or not 0 < r[0] <= r[1]:
                    raise ManagerError(f"event {name!r}: interval mode needs a positive ordered range")
                n = env.num_envs
                self._elapsed[name] = torch.zeros(n, dtype=torch.float64, device=env.device)
                self._target[name] = torch.zeros(n, dtype=torch.float64, device=env.device)
                self._fired[name] = torch.zeros(n, dtype=torch.bool, device=env.device)
                self._draw_targets(name, torch.arange(n, device=env.device))

    def is_external(self, name: str) -> bool:
        return builtin_id(self.terms[name]) is None

    def _quant(self, name):
        lo, hi = self.cfg[name].interval_range
        dt = self.env.dt_control
        return lo, hi, float(np.ceil(lo / dt) * dt), float(np.floor(hi / dt) * dt)

    def _draw_targets(self, name: str, ids) -> None:  # managers/event.py:75-84
        import torch

        lo, hi, lo_q, hi_q = self._quant(name)
        dt = self.env.dt_control
        draw = self.env.streams.uniform(f"event.{name}.interval", lo, hi, ids, 1)[:, 0]
        self._target[name][ids] = torch.clamp(torch.round(draw / dt) * dt, lo_q, hi_q)

    def apply_startup(self) -> None:
        import torch

        all_ids = torch.arange(self.env.num_envs, device=self.env.device)
        for name, tc in self.cfg.items():
            if tc.mode == "startup":
                self.terms[name](self.env, all_ids, **tc.params)

    def apply_reset(self, ids) -> None:
        import torch

        ids = torch.as_tensor(np.asarray(ids) if not torch.is_tensor(ids) else ids, device=self.env.device)
        if not ids.numel():
            return
        for name, tc in self.cfg.items():
            if tc.mode == "reset":
                self.terms[name](self.env, ids, **tc.params)
            elif tc.mode == "interval":
                self._elapsed[name][ids] = 0.0
                self._draw_targets(name, ids)

    def apply_interval(self, dt: float | None = None) -> None:
        """Stopwatch tick + fire (managers/event.py:103-114), as the fused stage."""
        self.env._launch(native.SS_ST_EVENTS)
        self.run_external_interval()

    def run_external_interval(self) -> None:
        """User-registered interval terms fire for the ids the kernel flagged."""
        import torch

        for name, tc in self.cfg.items():
            if tc.mode == "interval" and self.is_external(name):
                ids = torch.nonzero(self._fired[name]).reshape(-1)
                if ids.numel():
                    self.terms[name](self.env, ids, **tc.params)

    def run_external_reset(self, ids) -> None:
        for name, tc in self.cfg.items():
            if tc.mode == "reset" and self.is_external(name):
                self.terms[name](self.env, ids, **tc.params)

    def prepare_fields(self) -> None:
        """Expand every field a reset/interval randomization will write, so the
        fused step never changes layout mid-launch."""
        for name, tc in self.cfg.items():
            if tc.mode in ("reset", "interval") and builtin_id(self.terms[name]) == native.SS_EVT_RANDOMIZE_FIELD:
                self.env.model.expand_field(tc.params.get("field", "friction"))

    def native_into(self, d) -> None:
        env = self.env
        d.n_events = len(self.cfg)
        for i, (name, tc) in enumerate(self.cfg.items()):
            e = d.event[i]
            e.mode = {"startup": native.SS_MODE_STARTUP, "reset": native.SS_MODE_RESET,
                      "interval": native.SS_MODE_INTERVAL}[tc.mode]
            sid = builtin_id(self.terms[name])
            e.func = native.SS_EVT_EXTERNAL if sid is None else sid
            p = tc.params
            if tc.mode == "interval":
                lo, hi, lo_q, hi_q = self._quant(name)
                e.iv_lo, e.iv_hi, e.iv_lo_q, e.iv_hi_q = float(lo), float(hi), lo_q, hi_q
                e.iv_slot = env.streams.slot(f"event.{name}.interval")
                e.elapsed = self._elapsed[name].data_ptr()
                e.target = self._target[name].data_ptr()
                e.fired = self._fired[name].data_ptr()
            if sid == native.SS_EVT_RANDOMIZE_FIELD:
                fld = p.get("field", "friction")
                dist = p.get("distribution", "uniform")
                op = p.get("operation", "scale")
                if dist not in _DIST or op not in _OPS:
                    raise ManagerError(f"event {name!r}: bad distribution/operation")
                rr = tuple(p.get("rng_range", (0.8, 1.2)))
                e.field = env.model.field_index(fld)
                e.distribution = _DIST[dist]
                e.operation = _OPS[op]
                e.r0, e.r1 = float(rr[0]), float(rr[1])
                e.slot_a = env.streams.slot(f"event.randomize.{fld}")
            elif sid == native.SS_EVT_PUSH_BASE:
                fx = p.get("fx_range", (-50.0, 50.0))
                fz = p.get("fz_range", (0.0, 0.0))
                e.r0, e.r1, e.r2, e.r3 = float(fx[0]), float(fx[1]), float(fz[0]), float(fz[1])
                e.slot_a = env.streams.slot("event.push.fx")
                e.slot_b = env.streams.slot("event.push.fz")
            elif sid == native.SS_EVT_JOINT_JITTER:
                pr = p.get("pos_range", (-0.1, 0.1))
                e.r0, e.r1 = float(pr[0]), float(pr[1])
                e.slot_a = env.streams.slot("event.joint_jitter")
