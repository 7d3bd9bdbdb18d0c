"""ManagerBasedRlEnv on one B200: the reset/step state machine over N worlds.

Drop-in for the reference env (env.py:95-305): same constructor, reset/step
signatures, stage order and public attributes; state lives in HBM and a
control step is ONE launch of the fused sm_100a kernel when every term is a
built-in (act, d substeps, terminate, reward, curriculum + masked reset,
command, events, observe -- env.py:219-259). With user-registered Python
terms the same kernel runs stage by stage and the plugins are evaluated in
between on the device tensors ("staged" mode), preserving the order.

No step ever waits on the device: reset ids, trigger counts and extras are
materialized lazily; nonfinite detection rides a zero-copy flag in pinned
host memory and is processed at most ``NF_LAG`` steps later (the capture
ring keeps that many spare steps of frames so the dump is exact).
"""

from __future__ import annotations

import ctypes
import os
import warnings
from collections.abc import Mapping

import numpy as np

from . import mdp  # noqa: F401  (registers the built-in terms)
from . import jit, native
from .capture import CaptureRing, dump_capture, load_capture, model_field_metadata
from .policies import RandomActions
from .config import ContactSensorCfg, EnvCfg, InitStateCfg, SceneCfg, config_hash, to_dict
from .entity import DefaultState, Entity, EntityData
from .managers import (
    ActionManager,
    CommandManager,
    CurriculumManager,
    EventManager,
    ObservationManager,
    RewardManager,
    TerminationManager,
)
from .rng import StreamPack
from .sensors import ContactSensor, RayScanner
from .sim import BatchState, StepPipeline, compile_model, restore, snapshot
from .terrain import generate_grid

__all__ = ["EnvCfg", "SceneCfg", "InitStateCfg", "ManagerBasedRlEnv", "load_capture"]

# steps that may be in flight between step_async and step_wait (ss_pipe, 2..8; SS_PIPE_SLOTS overrides for A/B):
# eight keep the paired D2H copies (ss_pipe_post) fed with slack for host jitter -- 31.5-31.9 us per step at
# 4096 worlds vs 32.0-33.0 with six, 33.9 with four unpaired slots, 41.8 with four paired (tools/e2e_ab.py)
PIPE_SLOTS = int(os.environ.get("SS_PIPE_SLOTS", "8"))
# steps whose results cross PCIe as one copy (ss_pipe_post; read by the native pipe from SS_PIPE_GROUP too)
PIPE_GROUP = int(os.environ.get("SS_PIPE_GROUP", "2"))
NF_LAG = 4  # control steps the host may run ahead before it must look at nonfinite flags

_SIM = native.SS_ST_APPLY | native.SS_ST_PUSH | native.SS_ST_PHYS | native.SS_ST_SENSOR


class _Extras(Mapping):
    """Per-step extras (env.py:261-272), materialized on first access.

    Values refer to this step's device buffers and are valid until the next
    step (like the observation buffers)."""

    def __init__(self, env, step: int):
        self._env = env
        self._step = step
        self._data = None

    def _build(self):
        import torch

        if self._data is None:
            env = self._env
            tm, rm = env.termination_manager, env.reward_manager
            ids = torch.nonzero(tm.terminated | tm.truncated).reshape(-1)
            d = {"reset_ids": ids}
            if ids.numel():
                for name in rm.terms:
                    d[f"episode_reward/{name}"] = rm.finalized[name][ids]
            for name in rm.terms:
                d[f"reward/{name}"] = rm.last_values[name]
            for name, c in tm.trigger_counts.items():
                d[f"termination_count/{name}"] = np.int64(c)
            d["curriculum/terrain_rows"] = env.terrain_rows
            d["nonfinite_worlds"] = tm.last_nonfinite
            self._data = d
        return self._data

    def __getitem__(self, k):
        return self._build()[k]

    def __iter__(self):
        return iter(self._build())

    def __len__(self):
        return len(self._build())


class ManagerBasedRlEnv:
    def __init__(self, cfg: EnvCfg, task_id: str = "", device=None, copy_outputs: bool = False):
        """``copy_outputs=True`` makes ``step``/``reset`` return FRESH tensors every call, like the
        reference's fresh numpy arrays (one device copy of the output arena per step); by default they
        are views of persistent device buffers that the next step overwrites (mjlab's convention)."""
        import torch

        self.cfg = cfg
        self.copy_outputs = bool(copy_outputs)
        self.task_id = task_id
        self.device = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
        spec = cfg.scene.model
        if cfg.physics_dt is not None:
            spec.physics_dt = cfg.physics_dt
        if cfg.decimation is not None:
            spec.decimation = cfg.decimation
        self.physics_dt = spec.physics_dt
        self.decimation = spec.decimation
        self.dt_control = self.physics_dt * self.decimation
        self.max_episode_steps = int(np.ceil(cfg.episode_length_s / self.dt_control - 1e-9))
        self.num_envs = n = cfg.scene.num_envs

        self.config_hash = config_hash(cfg)
        self.terrain = generate_grid(cfg.scene.terrain, cfg.seed)
        self._dev_index = self.device.index if self.device.index is not None else torch.cuda.current_device()
        self.model = compile_model(spec, n, self.device)
        self.state = BatchState(self.model)
        self.world_ids = cfg.scene.world_id_offset + np.arange(n)
        self.streams = StreamPack(cfg.seed, cfg.scene.world_id_offset, n, self.device, self._invalidate)

        init = cfg.scene.init_state
        k = self.model.num_joints
        self.default_joint_pos = np.asarray(init.joint_pos or (0.0,) * k, dtype=np.float64)
        self.robot = Entity(
            spec.name,
            joint_names=self.model.joint_names,
            default_state=DefaultState(base_pose=init.base_pose, base_vel=init.base_vel,
                                       joint_pos=tuple(self.default_joint_pos),
                                       joint_vel=tuple(init.joint_vel or (0.0,) * k)),
            pos_limits=self.model.pos_limits,
        )
        self.entities = {spec.name: self.robot, "terrain": Entity("terrain", base_type="fixed")}
        self.entity_data = EntityData(self.model, self.state)
        self.contact_sensor = ContactSensor(ContactSensorCfg(history_length=cfg.scene.contact_history), n,
                                            len(self.model.feet), self.device)
        self.ray_scanner = RayScanner(cfg.scene.ray_scan, n, self.device)
        self.pipeline = StepPipeline(self.model, self.terrain)
        self.capture = CaptureRing(cfg.capture_len, n, self.model.nq, k, self.device,
                                   spare=self.decimation * (NF_LAG + 1))

        dev = self.device
        self.terrain_rows = torch.zeros(n, dtype=torch.int64, device=dev)
        self.terrain_cols = torch.as_tensor((self.world_ids % self.terrain.cols).astype(np.int64), device=dev)
        self.episode_steps = torch.zeros(n, dtype=torch.int64, device=dev)
        self.episode_start_x = torch.zeros(n, dtype=torch.float64, device=dev)
        self.commanded_distance = torch.zeros(n, dtype=torch.float64, device=dev)
        self._prev_lin_vel_b = torch.zeros((2, n), dtype=torch.float64, device=dev)
        self._dump_paths: list[str] = []
        self._startup_done = False
        self._desc = None
        self._desc_ref = None
        self._jit_handle = None
        self._jit_split = None  # (physics kernel, terms + observations kernel) of a split env
        self.use_jit = jit.enabled()
        self._lib = native.lib()

        # native runtime state shared with ss_rt_launch (counters, heads, weights)
        self._rt = native.RtState()
        self._rt_ref = ctypes.byref(self._rt)
        self._la = native.Launch()
        self._la_ref = ctypes.byref(self._la)
        self._la_key = None  # (stages, nsub, flags, groups_mask) last written into _la
        self._stats_req = None  # pending fused-statistics request (metrics.StatsPacker.request)
        self._rt.global_step = 0
        self._rt.sensor_last_update = -1
        # nonfinite bookkeeping: zero-copy flags (mapped pinned memory) + a ring of
        # per-step world masks, NF_LAG + 2 slots
        slots = NF_LAG + 2
        self._nf_flags = torch.zeros(native.SS_RT_SLOTS, dtype=torch.int32).pin_memory()
        self._nf_masks = torch.zeros((slots, n), dtype=torch.bool, device=dev)
        self._rt.nf_flags = self._nf_flags.data_ptr()
        self._rt.nf_slots = slots
        self._nf_out = (ctypes.c_int32 * slots)()
        self._nf_views = [self._nf_masks[i] for i in range(slots)]

        all_ids = torch.arange(n, device=dev)
        self.robot.write_default_state(self.state, all_ids)
        self._place_on_terrain(all_ids)

        self.action_manager = ActionManager(cfg.actions, self)
        self.command_manager = CommandManager(cfg.commands, self)
        self.reward_manager = RewardManager(cfg.rewards, self)
        self.termination_manager = TerminationManager(cfg.terminations, self)
        self.termination_manager.last_nonfinite = self._nf_masks[0]
        self.event_manager = EventManager(cfg.events, self)
        self.curriculum_manager = CurriculumManager(cfg.curriculum, self)
        self.observation_manager = ObservationManager(cfg.observations, self)
        self.model.on_layout_change(self._invalidate)
        self.staged = self._needs_staging()
        self._build_output_arena()
        self.capture.bind(self._rt)
        self.contact_sensor.bind(self._rt)
        self.action_manager.bind(self._rt)
        self.observation_manager.bind(self._rt)
        self.reward_manager.weights.bind(self._rt)

    def _build_output_arena(self) -> None:
        """Place every per-step output -- the observation groups, reward,
        terminated, truncated -- in ONE contiguous device block, so a consumer
        on the host moves a step's results with a single copy (see
        ``step_outputs`` / ``unpack_outputs``)."""
        import torch

        n = self.num_envs
        om, rm, tm = self.observation_manager, self.reward_manager, self.termination_manager
        layout = []
        off = 0
        for g in om.groups:
            nbytes = n * om.group_dim(g) * 8
            layout.append((f"obs/{g}", off, nbytes, torch.float64, (n, om.group_dim(g))))
            off += nbytes
        layout.append(("reward", off, n * 8, torch.float64, (n,)))
        off += n * 8
        layout.append(("terminated", off, n, torch.bool, (n,)))
        off += n
        layout.append(("truncated", off, n, torch.bool, (n,)))
        off += n
        self.step_outputs = torch.zeros(off, dtype=torch.uint8, device=self.device)
        self.step_output_layout = layout
        views = self.unpack_outputs(self.step_outputs)
        for g in om.groups:
            om._out[g] = views[f"obs/{g}"]
        rm.reward = views["reward"]
        tm.terminated = views["terminated"]
        tm.truncated = views["truncated"]

    def enable_host_outputs(self) -> dict:
        """Mirror every step's outputs into pinned host memory from the kernel.

        After this call each launch repeats its output-arena stores (the obs
        groups, reward, terminated, truncated) into a mapped pinned host block
        of the same layout, so the results cross PCIe while the kernel runs
        instead of through a separate device->host copy. Returns the typed
        host views (also ``host_outputs``); they hold a step's results once
        the launching stream has been synchronized. Device outputs are
        unchanged."""
        import torch

        if getattr(self, "_host_mirror", None) is None:
            self._host_mirror = torch.zeros(self.step_outputs.numel(), dtype=torch.uint8).pin_memory()
            self.host_outputs = self.unpack_outputs(self._host_mirror)
            self._invalidate()
        return self.host_outputs

    def unpack_outputs(self, block) -> dict:
        """Typed views into a copy of ``step_outputs`` (device or host)."""
        out = {}
        for name, off, nbytes, dtype, shape in self.step_output_layout:
            out[name] = block[off : off + nbytes].view(dtype).view(shape)
        return out

    def __del__(self):
        try:
            self._lib.ss_rt_release(self._rt_ref)
            if getattr(self, "_pipe", None) is not None:
                self._lib.ss_pipe_destroy(self._pipe["h"])
        except Exception:
            pass

    @property
    def global_step(self) -> int:
        return self._rt.global_step

    @global_step.setter
    def global_step(self, v: int) -> None:
        self._rt.global_step = int(v)

    # -- descriptor ---------------------------------------------------------------

    prev_lin_vel_b = property(lambda self: self._prev_lin_vel_b.t())

    def _invalidate(self, *_):
        self._desc = None
        self._jit_handle = None

    def _needs_staging(self) -> bool:
        return bool(self.termination_manager.external or self.reward_manager.external
                    or self.curriculum_manager.has_external
                    or any(self.event_manager.is_external(nm) and self.cfg.events[nm].mode != "startup"
                           for nm in self.event_manager.terms)
                    or self.observation_manager.has_external)

    def _get_desc(self):
        if self._desc is None:
            d = native.EnvDesc()
            d.abi_version = native.SS_ABI_VERSION
            d.n_worlds = self.num_envs
            d.decimation = self.decimation
            d.max_episode_steps = self.max_episode_steps
            d.dt_control = self.dt_control
            self.model.native_into(d)
            d.terrain = self.terrain.native(self.device)
            self.state.native_into(d.state)
            r = self.streams
            d.rng.world_id_offset = r.world_id_offset
            for s, base in enumerate(r.bases):
                d.rng.base[s] = base
                d.rng.counter[s] = r.counters[s].data_ptr()
            ds = self.robot.default_state
            for i in range(3):
                d.base_pose[i] = float(ds.base_pose[i])
                d.base_vel[i] = float(ds.base_vel[i])
            for j in range(self.model.num_joints):
                d.joint_pos[j] = float(ds.joint_pos[j])
                d.joint_vel[j] = float(ds.joint_vel[j])
            d.spawn_offset = float(self.cfg.scene.spawn_offset)
            self.action_manager.native_into(d)
            self.capture.native_into(d)
            self.contact_sensor.native_into(d)
            self.ray_scanner.native_into(d)
            self.termination_manager.native_into(d)
            self.reward_manager.native_into(d)
            self.command_manager.native_into(d)
            self.event_manager.native_into(d)
            self.curriculum_manager.native_into(d)
            d.episode_steps = self.episode_steps.data_ptr()
            d.episode_start_x = self.episode_start_x.data_ptr()
            d.commanded_distance = self.commanded_distance.data_ptr()
            d.terrain_rows = self.terrain_rows.data_ptr()
            d.terrain_cols = self.terrain_cols.data_ptr()
            d.prev_lin_vel_b = self._prev_lin_vel_b.data_ptr()
            self.observation_manager.native_into(d)
            d.nf_flags = self._nf_flags.data_ptr()
            d.probe = getattr(self, "_probe_ptr", None)
            hm = getattr(self, "_host_mirror", None)
            if hm is not None:
                delta = hm.data_ptr() - self.step_outputs.data_ptr()
                d.out_mirror = ctypes.c_int64(delta).value  # two's complement wrap
            d.nonfinite = self._nf_masks.data_ptr()
            # the descriptor may have allocated new stream slots: refresh their pointers
            for s, base in enumerate(r.bases):
                d.rng.base[s] = base
                d.rng.counter[s] = r.counters[s].data_ptr()
            self._desc = d
            self._desc_ref = ctypes.byref(d)
        return self._desc

    def _prepare_launch(self) -> None:
        """(Re)build the descriptor and, for the specialized kernel, its module
        handle and packed parameter block."""
        d = self._desc if self._desc is not None else self._get_desc()
        if self._desc is None:  # a stream slot was allocated while building
            d = self._get_desc()
        la = self._la
        if self.use_jit and self._jit_handle is None:
            try:
                hs = jit.modules_for(d)
                self._jit_handle = hs["main"]
                self._jit_split = (hs["phys"], hs["post"]) if "phys" in hs else None
                # the specialized kernel's parameter block: the descriptor
                # packed to this env's counts (4 KB instead of 13 KB)
                self._jit_packed = native.pack_desc(d, jit.desc_caps(d))
            except jit.JitUnsupported as err:
                warnings.warn(f"per-env specialization unavailable ({err}); using the generic sm_100a kernel")
                self.use_jit = False
        if self.use_jit:
            la.jit_desc = ctypes.addressof(self._jit_packed)
            la.jit_desc_bytes = ctypes.sizeof(self._jit_packed)
        else:
            la.jit_desc = None
            la.jit_desc_bytes = 0

    def _launch(self, stages: int, nsub: int = 0, actions=None, reset_mask=None, groups_mask: int = 0,
                flags: int = 0, handle=None) -> None:
        """One launch through the native runtime (ss_rt_launch): it derives the
        per-step uniforms from the shared ss_rt_state, launches the
        specialized (or generic) kernel and advances the counters."""
        fused = actions.__class__ is RandomActions
        if fused:
            slot = self.streams.slot("policy.random")  # first use invalidates the descriptor
        if self._desc is None or (self.use_jit and self._jit_handle is None):
            self._prepare_launch()
        rt = self._rt
        term = stages & native.SS_ST_TERM
        if term:
            # the launch retires old nonfinite slots itself (poll_keep)
            self.termination_manager.last_nonfinite = self._nf_views[rt.nf_slot]
        la = self._la
        key = (stages, nsub, flags, groups_mask)
        if key != self._la_key:  # the fused step repeats one signature: skip the ctypes writes
            la.stages, la.nsub, la.flags, la.groups_mask = key
            la.poll_keep = NF_LAG if term else -1
            self._la_key = key
        if fused:
            la.actions = None
            la.policy_slot, la.policy_lo, la.policy_hi = slot, float(actions.low), float(actions.high)
        else:
            la.actions = None if actions is None else actions.data_ptr()
            la.policy_slot = -1
        la.reset_mask = None if reset_mask is None else reset_mask.data_ptr()
        req = self._stats_req
        if req is not None and stages in (native.SS_ST_STEP_ALL, jit.SPLIT_POST):
            # metrics.StatsPacker.request: this step also reduces the job statistics (fused tail)
            la.stats_out, la.stats_partials, la.stats_ticket, la.stats_rows = req
            self._stats_req = None
        elif la.stats_out:
            la.stats_out = None
        rt.sim_step = self.state.sim_step
        native.LAUNCHES["count"] += 1
        rc = self._lib.ss_rt_launch(self._desc_ref, self._rt_ref, self._la_ref,
                                    (handle or self._jit_handle) if self.use_jit else None,
                                    native.current_stream(self._dev_index))
        if rc != 0:
            raise native.NativeError(f"ss_rt_launch failed ({rc}): {self._lib.ss_last_error().decode()}")
        self.state.sim_step = rt.sim_step
        if term and rt.nf_ready_n:
            # retired slots are never the one this launch used (ring of
            # NF_LAG + 2), so their metadata and masks are still intact
            for i in range(rt.nf_ready_n):
                slot = rt.nf_ready[i]
                self._dump_on_nonfinite(slot, rt.nf_pushes[slot], rt.nf_count[slot], rt.nf_sim_step[slot])

    # -- nonfinite detection (deferred, no per-step sync) ----------------------------

    def _nf_drain(self, keep: int) -> None:
        n = self._lib.ss_rt_poll(self._rt_ref, keep, self._nf_out, len(self._nf_out))
        if n < 0:
            raise native.NativeError(f"ss_rt_poll failed: {self._lib.ss_last_error().decode()}")
        rt = self._rt
        for i in range(n):
            slot = self._nf_out[i]
            self._dump_on_nonfinite(slot, rt.nf_pushes[slot], rt.nf_count[slot], rt.nf_sim_step[slot])

    @property
    def dump_paths(self) -> list[str]:
        self._nf_drain(0)
        return self._dump_paths

    def _dump_on_nonfinite(self, slot: int, pushes: int, count: int, sim_step: int) -> None:
        os.makedirs(self.cfg.capture_dir, exist_ok=True)
        path = os.path.join(self.cfg.capture_dir, f"capture_step{sim_step}.bin")
        self._write_dump(path, pushes, count, self._nf_masks[slot])
        self._dump_paths.append(path)

    def _write_dump(self, path: str, pushes=None, count=None, nonfinite=None) -> None:
        import torch

        nf = self.termination_manager.last_nonfinite if nonfinite is None else nonfinite
        meta = {
            "offending_observation_terms": sorted(self.observation_manager.nonfinite_report),
            "offending_reward_terms": sorted(self.reward_manager.nonfinite_report),
            "nonfinite_worlds": torch.nonzero(nf).reshape(-1).cpu().tolist(),
            "fields": model_field_metadata(self.model),
        }
        dump_capture(path, self.capture, self.config_hash, task_id=self.task_id, config_json=to_dict(self.cfg),
                     metadata=meta, pushes=pushes, count=count)

    def dump_capture(self, path: str) -> None:
        self._nf_drain(0)
        self._write_dump(path)

    # -- reset --------------------------------------------------------------------------

    def _place_on_terrain(self, ids) -> None:
        """Spawn on the world's curriculum patch + terrain height (env.py:171-180)."""
        import torch

        rows, cols = self.terrain_rows[ids], self.terrain_cols[ids]
        origin = (rows * self.terrain.cols + cols).to(torch.float64) * self.terrain.patch_length
        spawn_x = origin + self.cfg.scene.spawn_offset
        self.state.q[ids, 0] += spawn_x
        self.state.q[ids, 1] += self.terrain.heights(spawn_x)

    def _reset_worlds(self, ids) -> None:
        """Standalone masked reset of the listed worlds (env.py:182-200)."""
        import torch

        ids_t = torch.as_tensor(np.asarray(ids) if not torch.is_tensor(ids) else ids, device=self.device)
        mask = torch.zeros(self.num_envs, dtype=torch.uint8, device=self.device)
        mask[ids_t] = 1
        self.event_manager.prepare_fields()
        self._launch(native.SS_ST_RESET | native.SS_ST_RESET_EXT, reset_mask=mask)
        self.event_manager.run_external_reset(ids_t)
        self.ray_scanner._cached_step = -1

    def reset(self, seed: int | None = None) -> dict:
        """Start fresh episodes in every world and return the first obs (env.py:202-215)."""
        import torch

        if seed is not None:
            self.streams = StreamPack(seed, self.cfg.scene.world_id_offset, self.num_envs, self.device,
                                      self._invalidate)
            self._invalidate()
            self._startup_done = False
        if not self._startup_done:
            self.event_manager.apply_startup()
            self._startup_done = True
        self.event_manager.prepare_fields()
        om = self.observation_manager
        ext_reset = any(self.event_manager.is_external(nm) and tc.mode == "reset"
                        for nm, tc in self.cfg.events.items())
        all_ids = torch.arange(self.num_envs, device=self.device)
        om._cache.clear()
        if ext_reset or om.has_external:
            self._launch(native.SS_ST_RESET_ALL)
            self.event_manager.run_external_reset(all_ids)
            self._launch(native.SS_ST_PREV_BEFORE)
            om.eval_external(list(om.groups))
            mask = om.begin(list(om.groups))
            self._launch(native.SS_ST_OBS, groups_mask=mask)
        else:
            mask = om.begin(list(om.groups))
            self._launch(native.SS_ST_RESET_ALL | native.SS_ST_PREV_BEFORE | native.SS_ST_OBS, groups_mask=mask)
        self.ray_scanner._cached_step = -1
        if self.copy_outputs:
            return {g: t.clone() for g, t in om.outputs().items()}
        return om.outputs()

    # -- step -------------------------------------------------------------------------------

    def step(self, actions):
        """One control step through the fixed eight-stage pipeline.

        Returns (obs groups, reward, terminated, truncated, extras); all device
        tensors, valid until the next step."""
        self._step_checked(self.action_manager.check_actions(actions))
        tm = self.termination_manager
        if self.copy_outputs:
            v = self.unpack_outputs(self.step_outputs.clone())  # one D2D copy of the whole arena
            obs = {g: v[f"obs/{g}"] for g in self.observation_manager.outputs()}
            # extras too are fresh values of this step (built now, not lazily from live buffers)
            x = _Extras(self, self.global_step)
            x._data = {k: (t.clone() if hasattr(t, "clone") else t) for k, t in x._build().items()}
            return obs, v["reward"], v["terminated"], v["truncated"], x
        return (self.observation_manager.outputs(), self.reward_manager.reward, tm.terminated, tm.truncated,
                _Extras(self, self.global_step))

    def _step_checked(self, a) -> None:
        """The control step on already-validated actions (step / step_async)."""
        if not self._startup_done:
            self.event_manager.prepare_fields()
        self.global_step += 1
        om = self.observation_manager
        om._cache.clear()
        if not self.staged:
            mask = om.begin_all()
            if a.__class__ is RandomActions:
                self.streams.slot("policy.random")  # allocate before the handles are chosen
            if self._desc is None or (self.use_jit and self._jit_handle is None):
                self._prepare_launch()
            if self.use_jit and self._jit_split is not None:
                # split env (jit.split_enabled): physics, then terms + observations, two kernels each
                # compiled for its stage set (fewer registers, more warps per SM at large N)
                phys, post = self._jit_split
                self._launch(jit.SPLIT_PHYS, nsub=self.decimation, actions=a, handle=phys)
                self._launch(jit.SPLIT_POST, groups_mask=mask, handle=post)
            else:
                self._launch(native.SS_ST_STEP_ALL, nsub=self.decimation, actions=a, groups_mask=mask)
            self.curriculum_manager.run_host(None)
        else:
            self._step_staged(a)
        self.ray_scanner._cached_step = -1

    # -- pipelined host I/O (gym VectorEnv step_async / step_wait) -------------------------------

    def step_async(self, actions) -> None:
        """Enqueue one control step fed from, and delivered to, pinned host memory.

        gym VectorEnv-style ``step_async`` / ``step_wait``. The native pipe
        (``ss_pipe_*``, csrc/ss_runtime.cu) copies the step's actions
        host->device on one copy-engine stream, runs the step exactly like
        ``step`` on the device copy, snapshots the output arena with an SM copy
        kernel into one of ``PIPE_SLOTS`` staging buffers, and copies it to one
        of ``PIPE_SLOTS + 2`` pinned host blocks on a second copy-engine stream
        -- so the PCIe traffic of step i overlaps the kernels of the steps after
        it; an even step whose successor is enqueued before it is waited for
        crosses PCIe in one copy with it (two arenas per copy sustain ~6 % more
        bandwidth). ``step_wait()`` blocks until the oldest pending step's
        results are in host memory and returns its host views (obs groups,
        reward, terminated, truncated); ``PIPE_SLOTS + 2`` pinned host blocks
        rotate, so the views stay valid through at least the next two
        ``step_async`` calls, even with the pipeline full (the third may
        reuse them). At most ``PIPE_SLOTS`` steps may be
        pending; with several in flight the host enqueues step i+1 while
        earlier steps run, hiding its own per-step cost. The action tensor is
        read asynchronously: do not overwrite it before that step's
        step_wait() returns."""
        import torch

        if getattr(self, "_host_mirror", None) is not None:
            raise RuntimeError("step_async uses device outputs + copy-engine transfers; do not enable_host_outputs")
        P = getattr(self, "_pipe", None)
        if P is None:
            A = self.action_manager.total_dim
            nb = self.step_outputs.numel()
            S = PIPE_SLOTS
            G = PIPE_GROUP if 1 < PIPE_GROUP <= S else 1
            H = S + G if S % G == 0 else S + 1  # a multiple of G: groups of steps never wrap (ss_pipe_post)
            dev_actions = [torch.empty((self.num_envs, A), dtype=torch.float64, device=self.device) for _ in range(S)]
            # staging buffers and host blocks each carved from one allocation (contiguous for the paired
            # D2H when the arena size keeps them 16-byte aligned)
            pitch = (nb + 15) // 16 * 16
            stage_all = torch.empty(S * pitch, dtype=torch.uint8, device=self.device)
            host_all = torch.empty(H * pitch, dtype=torch.uint8).pin_memory()
            stage = [stage_all[k * pitch:k * pitch + nb] for k in range(S)]
            host = [host_all[k * pitch:k * pitch + nb] for k in range(H)]
            arr = lambda ts: (ctypes.c_void_p * S)(*[t.data_ptr() for t in ts])  # noqa: E731
            h = ctypes.c_void_p()
            hosts = (ctypes.c_void_p * H)(*[t.data_ptr() for t in host])
            rc = self._lib.ss_pipe_create(S, H, arr(dev_actions), arr(stage), hosts, self.num_envs * A * 8, nb,
                                          ctypes.byref(h))
            if rc != 0:
                raise native.NativeError(f"ss_pipe_create failed: {self._lib.ss_last_error().decode()}")
            P = self._pipe = dict(h=h, dev_actions=dev_actions, stage=stage, host=host, pinned=set(),
                                  keep=(stage_all, host_all), views=[self.unpack_outputs(x) for x in host])
        if (actions.__class__ is not torch.Tensor or actions.dtype is not torch.float64 or actions.is_cuda
                or not actions.is_contiguous() or actions.shape != P["dev_actions"][0].shape):
            raise ValueError(f"step_async takes a contiguous pinned float64 host tensor of shape "
                             f"{tuple(P['dev_actions'][0].shape)}")
        sp = actions.untyped_storage().data_ptr()
        if sp not in P["pinned"]:  # pinnedness is a property of the storage: check each storage once
            if not actions.is_pinned():
                raise ValueError("step_async takes PINNED host actions (tensor.pin_memory())")
            P["pinned"].add(sp)
        stream = native.current_stream(self._dev_index)
        k = self._lib.ss_pipe_pre(P["h"], actions.data_ptr(), stream)
        if k < 0:
            raise RuntimeError(self._lib.ss_last_error().decode())
        self._step_checked(P["dev_actions"][k])
        if self._lib.ss_pipe_post(P["h"], self.step_outputs.data_ptr(), stream) < 0:
            raise native.NativeError(self._lib.ss_last_error().decode())

    def step_wait(self) -> dict:
        """Host views (obs groups, reward, terminated, truncated) of the oldest step_async step."""
        P = getattr(self, "_pipe", None)
        k = -1 if P is None else self._lib.ss_pipe_wait(P["h"])
        if k < 0:
            raise RuntimeError("no pending step_async step")
        return P["views"][k]

    def _step_staged(self, a) -> None:
        import torch

        om, em, cm = self.observation_manager, self.event_manager, self.curriculum_manager
        self._launch(native.SS_ST_ACTION | _SIM, nsub=self.decimation, actions=a)
        self.termination_manager.eval_external()
        self._launch(native.SS_ST_TERM)
        self.reward_manager.eval_external()
        self._launch(native.SS_ST_REWARD)
        ext_reset = any(em.is_external(nm) and tc.mode == "reset" for nm, tc in self.cfg.events.items())
        if cm.has_external or ext_reset:
            tm = self.termination_manager
            ids = torch.nonzero(tm.terminated | tm.truncated).reshape(-1)
            self._launch(native.SS_ST_CURRICULUM)
            cm.run_external(ids)
            cm.run_host(ids)
            self._launch(native.SS_ST_RESET)
            em.run_external_reset(ids)
        else:
            self._launch(native.SS_ST_CURRICULUM | native.SS_ST_RESET)
            cm.run_host(None)
        self._launch(native.SS_ST_COMMAND | native.SS_ST_EVENTS)
        em.run_external_interval()
        om.eval_external(list(om.groups))
        mask = om.begin(list(om.groups))
        self._launch(native.SS_ST_OBS | native.SS_ST_PREV_AFTER, groups_mask=mask)

    # -- convenience passthroughs (tests, replay) ---------------------------------------------

    def snapshot(self):
        return snapshot(self.state)

    def restore(self, frame) -> None:
        restore(self.state, frame)

    def synchronize(self) -> None:
        import torch

        torch.cuda.synchronize(self.device)
        self._nf_drain(0)
