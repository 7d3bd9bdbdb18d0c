"""Sensors (sensors.py of the reference): ray height scan and foot contacts.

The contact sensor's per-substep update runs inside the fused step
(``ContactSensor.update`` in csrc/ss_step.cu); its bookkeeping arrays are
device SoA tensors exposed with the reference's (N, F) shapes. The ray
scanner is evaluated per world by the observation stage; ``read`` is the
standalone form (one ``ss_heights`` launch), cached per sim_step.
"""

from __future__ import annotations

import numpy as np

from . import native
from .config import ContactSensorCfg, RayScanCfg

NEVER_TOUCHED = -(1 << 40)

__all__ = ["ContactSensor", "ContactSensorCfg", "NEVER_TOUCHED", "RayScanCfg", "RayScanner"]


class RayScanner:
    """Vertical probes: terrain height minus base height per offset (sensors.py:26-46)."""

    def __init__(self, cfg: RayScanCfg, n_worlds: int, device=None):
        self.cfg = cfg
        self.offsets = np.asarray(cfg.offsets, dtype=np.float64)
        if len(self.offsets) > native.SS_MAX_RAYS:
            raise ValueError(f"more than {native.SS_MAX_RAYS} rays")
        self._cache = None
        self._cached_step = -1
        self.compute_count = 0
        self.device = device

    def read(self, terrain, data, state):
        import torch

        if state.sim_step != self._cached_step or self._cache is None:
            off = torch.as_tensor(self.offsets, device=state.device)
            xs = (data.root_pos[:, 0:1] + off[None, :]).contiguous()
            h = torch.zeros_like(xs) if terrain is None else terrain.heights(xs)
            self._cache = h - data.root_pos[:, 1:2]
            self._cached_step = state.sim_step
            self.compute_count += 1
        return self._cache

    def native_into(self, d) -> None:
        d.n_rays = len(self.offsets)
        for i, o in enumerate(self.offsets):
            d.ray_offset[i] = float(o)


class ContactSensor:
    """Per-foot contact bookkeeping (sensors.py:59-118) on the device."""

    def __init__(self, cfg: ContactSensorCfg, n_worlds: int, n_feet: int, device=None):
        import torch

        if device is None:
            device = torch.device("cuda", torch.cuda.current_device())
        if cfg.history_length > native.SS_MAX_HIST:
            raise ValueError(f"contact history longer than {native.SS_MAX_HIST}")
        self.cfg = cfg
        self.n_worlds = n_worlds
        self.n_feet = n_feet
        self.device = device
        z = lambda *s, dt=torch.float64: torch.zeros(s, dtype=dt, device=device)  # noqa: E731
        self._in = z(n_feet, n_worlds, dt=torch.bool)
        self._normal = z(n_feet, n_worlds)
        self._tangent = z(n_feet, n_worlds)
        self._hist = z(cfg.history_length, n_feet, n_worlds)
        self._air = z(n_feet, n_worlds)
        self._last_air = z(n_feet, n_worlds)
        self._contact = z(n_feet, n_worlds)
        self._td = torch.full((n_feet, n_worlds), NEVER_TOUCHED, dtype=torch.int64, device=device)
        self._last_local = -1
        self._rt = None

    def bind(self, rt) -> None:
        self._rt = rt
        rt.sensor_last_update = self._last_local

    @property
    def _last_update_step(self) -> int:
        return self._rt.sensor_last_update if self._rt is not None else self._last_local

    @_last_update_step.setter
    def _last_update_step(self, v: int) -> None:
        if self._rt is not None:
            self._rt.sensor_last_update = v
        else:
            self._last_local = v

    in_contact = property(lambda self: self._in.t())
    normal_force = property(lambda self: self._normal.t())
    tangent_force = property(lambda self: self._tangent.t())
    force_history = property(lambda self: self._hist.permute(0, 2, 1))  # (H, N, F), newest first
    current_air_time = property(lambda self: self._air.t())
    last_air_time = property(lambda self: self._last_air.t())
    current_contact_time = property(lambda self: self._contact.t())
    last_touchdown_step = property(lambda self: self._td.t())

    def reset(self, ids) -> None:
        import torch

        ids = torch.as_tensor(np.asarray(ids) if not torch.is_tensor(ids) else ids, device=self.device)
        self.in_contact[ids] = False
        self.normal_force[ids] = 0.0
        self.tangent_force[ids] = 0.0
        self.force_history[:, ids] = 0.0
        self.current_air_time[ids] = 0.0
        self.last_air_time[ids] = 0.0
        self.current_contact_time[ids] = 0.0
        self.last_touchdown_step[ids] = NEVER_TOUCHED

    def enabled_mask(self, sim_step0: int, nsub: int, phys: bool = True) -> int:
        """Host side of "at most one update per sim_step" for a launch."""
        mask = 0
        for s in range(nsub):
            step = sim_step0 + s + (1 if phys else 0)
            if step != self._last_update_step:
                mask |= 1 << s
                self._last_update_step = step
        return mask

    def update(self, state, dt: float) -> None:
        """One update from the state's contact cache (sensors.py:91-115)."""
        d = native.EnvDesc()
        d.abi_version = native.SS_ABI_VERSION
        d.n_worlds = self.n_worlds
        d.model.n_feet = self.n_feet
        d.model.dt = float(dt)
        state.native_into(d.state)
        self.native_into(d)
        u = native.Uniforms()
        u.stages = native.SS_ST_SENSOR
        u.nsub = 1
        u.sim_step = state.sim_step
        u.sensor_mask = self.enabled_mask(state.sim_step, 1, phys=False)
        if u.sensor_mask:
            native.call("ss_env_step", native.byref(d), native.byref(u), native.current_stream(self.device))

    def touched_down_within(self, sim_step: int, substeps: int):
        return self.last_touchdown_step > sim_step - substeps

    def native_into(self, d) -> None:
        d.hist_len = self.cfg.history_length
        d.s_in_contact = self._in.data_ptr()
        d.s_normal = self._normal.data_ptr()
        d.s_tangent = self._tangent.data_ptr()
        d.s_force_hist = self._hist.data_ptr()
        d.s_cur_air = self._air.data_ptr()
        d.s_last_air = self._last_air.data_ptr()
        d.s_cur_contact = self._contact.data_ptr()
        d.s_last_td = self._td.data_ptr()
