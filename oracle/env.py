"""numpy restatement of ManagerBasedRlEnv.reset/step (env.py:95-259) and
everything it calls: ActionManager + actuators (managers/action.py,
actuators.py), CaptureRing.push (capture.py:53-59), EntityData.refresh
(entity.py:145-165), ContactSensor (sensors.py:59-118), RayScanner
(sensors.py:26-46), TerminationManager (managers/termination.py),
RewardManager (managers/reward.py), CurriculumManager + terms
(managers/curriculum.py, mdp.py:227-275), CommandManager
(managers/command.py), EventManager (managers/event.py, mdp.py:186-220) and
ObservationManager (managers/observation.py, mdp.py:26-89).

Consumes the same EnvCfg dataclasses as the product and the host-generated
heightfield samples (terrain generation is setup, pinned separately). State
is a flat dict of row-major (N, C) arrays, exactly the reference layout.
Custom (non built-in) terms are passed in as ``custom={"func_id": fn}``
with fn(env, **params) for obs/reward/termination and fn(env, ids, **params)
for events/curriculum, like the reference registries (managers/base.py:36-70).
"""

from __future__ import annotations

import math
import re

import numpy as np

from .physics import OracleModel, heights_fn, new_state, oracle_substep, raw_heights
from .rng import OracleStreams

NEVER = -(1 << 40)  # sensors.py:51


def _load_mlp(path):
    """SSMLP1 container reader restated (actuators.py:140-174)."""
    import struct

    raw = open(path, "rb").read()
    assert raw[:6] == b"SSMLP1"
    _, n_layers = struct.unpack_from("<II", raw, 6)
    off, layers = 14, []
    for _ in range(n_layers):
        (ln,) = struct.unpack_from("<B", raw, off)
        act = raw[off + 1 : off + 1 + ln].decode()
        off += 1 + ln
        n_in, n_out = struct.unpack_from("<II", raw, off)
        off += 8
        w = np.frombuffer(raw, "<f8", n_in * n_out, off).reshape(n_out, n_in).copy()
        off += 8 * n_in * n_out
        b = np.frombuffer(raw, "<f8", n_out, off).copy()
        off += 8 * n_out
        layers.append((w, b, act))
    return layers


class OracleEnv:
    def __init__(self, cfg, samples=None, custom=None, capture=True):
        self.cfg = cfg
        self.custom = dict(custom or {})
        spec = cfg.scene.model
        if cfg.physics_dt is not None:
            spec.physics_dt = cfg.physics_dt
        if cfg.decimation is not None:
            spec.decimation = cfg.decimation
        self.physics_dt = spec.physics_dt
        self.decimation = spec.decimation
        self.dt_control = self.physics_dt * self.decimation
        self.max_episode_steps = int(np.ceil(cfg.episode_length_s / self.dt_control - 1e-9))
        n = self.n = cfg.scene.num_envs
        tcfg = cfg.scene.terrain
        self.samples = None if samples is None else np.asarray(samples, dtype=np.float64)
        self.spacing = tcfg.spacing
        self.t_rows, self.t_cols, self.patch_length = tcfg.rows, tcfg.cols, tcfg.patch_length
        self.m = OracleModel(spec, n)
        self.heights = heights_fn(self.samples, self.spacing)
        self.S = new_state(self.m)
        self.world_ids = cfg.scene.world_id_offset + np.arange(n)
        self.rng = OracleStreams(cfg.seed, self.world_ids)
        k, nf = self.m.k, len(self.m.feet)
        init = cfg.scene.init_state
        self.default_joint_pos = np.asarray(init.joint_pos or (0.0,) * k, dtype=np.float64)
        self.default_joint_vel = np.asarray(init.joint_vel or (0.0,) * k, dtype=np.float64)
        self.base_pose = np.asarray(init.base_pose, dtype=np.float64)
        self.base_vel = np.asarray(init.base_vel, dtype=np.float64)
        self.joint_names = [j.name for j in spec.joints]
        # sensors
        H = cfg.scene.contact_history
        self.sens = {
            "in": np.zeros((n, nf), dtype=bool),
            "normal": np.zeros((n, nf)),
            "tangent": np.zeros((n, nf)),
            "hist": np.zeros((H, n, nf)),
            "air": np.zeros((n, nf)),
            "last_air": np.zeros((n, nf)),
            "contact": np.zeros((n, nf)),
            "td": np.full((n, nf), NEVER, dtype=np.int64),
        }
        self.sens_last_update = -1
        self.ray_offsets = np.asarray(cfg.scene.ray_scan.offsets, dtype=np.float64)
        self.ray_cache = None
        self.ray_step = -1
        # capture ring (capture.py:41-59)
        self.capture = capture
        K = cfg.capture_len
        self.cap_q = np.zeros((K, n, self.m.nq))
        self.cap_qd = np.zeros((K, n, self.m.nq))
        self.cap_ctrl = np.zeros((K, n, k))
        self.cap_steps = np.zeros(K, dtype=np.int64)
        self.cap_head, self.cap_count = -1, 0
        # episode bookkeeping (env.py:146-151)
        self.terrain_rows = np.zeros(n, dtype=np.int64)
        self.terrain_cols = (self.world_ids % self.t_cols).astype(np.int64)
        self.episode_steps = np.zeros(n, dtype=np.int64)
        self.episode_start_x = np.zeros(n)
        self.commanded_distance = np.zeros(n)
        self.prev_lin_vel_b = np.zeros((n, 2))
        self.global_step = 0
        self._startup_done = False
        self._write_default(np.arange(n))
        self._place(np.arange(n))
        self.refresh()
        self._build_actions()
        self._build_commands()
        self._build_rewards()
        self._build_terminations()
        self._build_events()
        self.curriculum = dict(cfg.curriculum)
        self._build_observations()

    # ------------------------------------------------------------------ helpers

    def find_joints(self, patterns):  # entity.py:76-89
        out = []
        for p in patterns:
            prog = re.compile(p)
            for i, nm in enumerate(self.joint_names):
                if prog.fullmatch(nm) and i not in out:
                    out.append(i)
        if not out:
            raise ValueError(f"patterns {patterns!r} match no joints")
        return sorted(out)

    def field(self, name):
        return self.m.value(name)

    # ------------------------------------------------------------------ entity

    def refresh(self):  # entity.py:145-165
        q, qd, S = self.S["q"], self.S["qd"], self.S
        c, s = np.cos(q[:, 2]), np.sin(q[:, 2])
        self.ed = {
            "root_pos": q[:, 0:2].copy(),
            "root_pitch": q[:, 2].copy(),
            "lin_vel_w": qd[:, 0:2].copy(),
            "ang_vel": qd[:, 2].copy(),
            "lin_vel_b": np.stack([c * qd[:, 0] + s * qd[:, 1], -s * qd[:, 0] + c * qd[:, 1]], axis=1),
            "proj_grav": np.stack([-s, -c], axis=1),
            "joint_pos": q[:, 3:].copy(),
            "joint_vel": qd[:, 3:].copy(),
            "foot_in_contact": S["fin"].copy(),
            "foot_forces": np.stack([S["ft"], S["fn"]], axis=-1),
            "foot_vel": S["fvel"].copy(),
        }

    def _write_default(self, ids):  # entity.py:91-105
        q, qd = self.S["q"], self.S["qd"]
        q[ids, 0:3] = self.base_pose
        qd[ids, 0:3] = self.base_vel
        q[ids, 3:] = self.default_joint_pos
        qd[ids, 3:] = self.default_joint_vel
        self.S["time"][ids] = 0.0

    def _place(self, ids):  # env.py:171-180
        rows, cols = self.terrain_rows[ids], self.terrain_cols[ids]
        origin = np.array([(int(r) * self.t_cols + int(c)) * self.patch_length for r, c in zip(rows, cols)])
        sx = origin + self.cfg.scene.spawn_offset
        self.S["q"][ids, 0] += sx
        h = np.zeros_like(sx) if self.samples is None else raw_heights(self.samples, self.spacing, sx)
        self.S["q"][ids, 1] += h

    # ------------------------------------------------------------------ actions

    def _build_actions(self):  # managers/action.py:11-66
        self.act_terms = []
        start = 0
        k = self.m.k
        for name, tc in self.cfg.actions.items():
            jids = np.array(self.find_joints(tc.joint_patterns), dtype=np.int64)
            off = self.default_joint_pos[jids] if tc.offset_mode == "default" else np.zeros(len(jids))
            acts = []
            for an, ac in tc.actuators.items():
                pats = ac.joint_patterns
                if ac.kind == "delayed" and not pats:
                    pats = ac.inner.joint_patterns
                aid = np.array(self.find_joints(pats), dtype=np.int64)
                acts.append(self._make_actuator(f"{name}.{an}", ac, aid))
            self.act_terms.append(
                {"name": name, "cfg": tc, "ids": jids, "slice": slice(start, start + len(jids)), "offset": off,
                 "acts": acts}
            )
            start += len(jids)
        self.action_dim = start
        self.action = np.zeros((self.n, start))
        self.prev_action = np.zeros((self.n, start))
        self.targets = np.zeros((self.n, k))
        for t in self.act_terms:
            self.targets[:, t["ids"]] = t["offset"]

    def _make_actuator(self, name, cfg, ids):  # actuators.py:216-258
        a = {"name": name, "cfg": cfg, "ids": ids, "delay": None, "mlp": None}
        inner = cfg
        if cfg.kind == "delayed":
            inner = cfg.inner
            cap = int(np.ceil(cfg.latency_range[1] / self.physics_dt)) + 1
            a["delay"] = {"cap": cap, "ring": np.zeros((cap, self.n, len(ids))), "head": 0,
                          "steps": np.zeros(self.n, dtype=np.int64)}
            a["delay"]["steps"][...] = np.clip(self._draw_delays(a, np.arange(self.n)), 0, cap - 1)
        a["inner"] = inner
        if inner.kind in ("ideal_pd", "dc_motor"):
            self.m.add_field(f"actuator.{name}.kp", np.full(len(ids), inner.kp))
            self.m.add_field(f"actuator.{name}.kd", np.full(len(ids), inner.kd))
        if inner.kind == "mlp":
            a["mlp"] = _load_mlp(inner.weights_path)
            a["err"] = np.zeros((inner.error_history, self.n, len(ids)))
            a["vel"] = np.zeros((inner.velocity_history, self.n, len(ids)))
        return a

    def _draw_delays(self, a, ids):  # actuators.py:260-267
        lo, hi = a["cfg"].latency_range
        if hi == lo:
            lat = np.full(len(ids), lo)
        else:
            lat = self.rng.uniform(f"actuator.{a['name']}.latency", lo, hi, ids, 1)[:, 0]
        return np.round(lat / self.physics_dt).astype(np.int64)

    def action_process(self, actions):  # managers/action.py:68-82
        actions = np.asarray(actions, dtype=np.float64)
        self.prev_action[...] = self.action
        self.action[...] = actions
        for t in self.act_terms:
            x = actions[:, t["slice"]]
            if t["cfg"].clip is not None:
                x = np.clip(x, t["cfg"].clip[0], t["cfg"].clip[1])
            self.targets[:, t["ids"]] = t["offset"] + t["cfg"].scale * x

    def action_apply(self):  # managers/action.py:84-90, actuators.py:279-316
        q, qd = self.S["q"][:, 3:], self.S["qd"][:, 3:]
        for t in self.act_terms:
            for a in t["acts"]:
                ids = a["ids"]
                qdes = self.targets[:, ids]
                D = a["delay"]
                if D is not None:
                    D["head"] = (D["head"] + 1) % D["cap"]
                    D["ring"][D["head"]] = qdes
                    qdes = D["ring"][(D["head"] - D["steps"]) % D["cap"], np.arange(self.n), :]
                qj, qdj = q[:, ids], qd[:, ids]
                inner = a["inner"]
                if inner.kind == "mlp":
                    a["err"] = np.roll(a["err"], 1, axis=0)
                    a["err"][0] = qdes - qj
                    a["vel"] = np.roll(a["vel"], 1, axis=0)
                    a["vel"][0] = qdj
                    n, dim = qj.shape
                    x = np.concatenate([a["err"].transpose(1, 2, 0).reshape(n * dim, -1),
                                        a["vel"].transpose(1, 2, 0).reshape(n * dim, -1)], axis=1)
                    for w, b, act in a["mlp"]:
                        x = x @ w.T + b
                        x = np.maximum(x, 0.0) if act == "relu" else (np.tanh(x) if act == "tanh" else x)
                    tau = np.clip(x[:, 0].reshape(n, dim), -inner.effort_limit, inner.effort_limit)
                else:
                    kp = self.field(f"actuator.{a['name']}.kp")
                    kd = self.field(f"actuator.{a['name']}.kd")
                    tau = kp * (qdes - qj) + kd * (0.0 - qdj)
                    if inner.kind == "ideal_pd":
                        tau = np.clip(tau, -inner.effort_limit, inner.effort_limit)
                    else:
                        hi = np.clip(inner.saturation_effort * (1.0 - qdj / inner.velocity_limit), 0.0,
                                     inner.effort_limit)
                        lo = np.clip(inner.saturation_effort * (-1.0 - qdj / inner.velocity_limit),
                                     -inner.effort_limit, 0.0)
                        tau = np.clip(tau, lo, hi)
                self.S["ctrl"][:, ids] = tau

    def action_reset(self, ids):  # managers/action.py:92-97, actuators.py:269-277
        self.action[ids] = 0.0
        self.prev_action[ids] = 0.0
        for t in self.act_terms:
            self.targets[np.ix_(ids, t["ids"])] = t["offset"]
            for a in t["acts"]:
                D = a["delay"]
                if D is not None:
                    D["ring"][:, ids, :] = self.targets[:, a["ids"]][ids]
                    if a["cfg"].resample_on_reset:
                        D["steps"][ids] = np.clip(self._draw_delays(a, ids), 0, D["cap"] - 1)
                if a["mlp"] is not None:
                    a["err"][:, ids, :] = 0.0
                    a["vel"][:, ids, :] = 0.0

    # ------------------------------------------------------------------ sensors

    def sensor_update(self):  # sensors.py:91-115
        if self.S["sim_step"] == self.sens_last_update:
            return
        self.sens_last_update = self.S["sim_step"]
        z, dt = self.sens, self.physics_dt
        now, prev = self.S["fin"], z["in"]
        td = now & ~prev
        lo = ~now & prev
        z["last_air"] = np.where(td, z["air"], z["last_air"])
        z["td"] = np.where(td, self.S["sim_step"], z["td"])
        z["contact"] = np.where(now, np.where(td, dt, z["contact"] + dt), 0.0)
        z["air"] = np.where(now, 0.0, np.where(lo, dt, z["air"] + dt))
        z["in"] = now.copy()
        z["normal"][...] = self.S["fn"]
        z["tangent"][...] = self.S["ft"]
        z["hist"] = np.roll(z["hist"], 1, axis=0)
        z["hist"][0] = self.S["fn"]

    def sensor_reset(self, ids):  # sensors.py:81-89
        z = self.sens
        z["in"][ids] = False
        z["normal"][ids] = 0.0
        z["tangent"][ids] = 0.0
        z["hist"][:, ids] = 0.0
        z["air"][ids] = 0.0
        z["last_air"][ids] = 0.0
        z["contact"][ids] = 0.0
        z["td"][ids] = NEVER

    def ray_read(self):  # sensors.py:36-46
        if self.S["sim_step"] != self.ray_step:
            xs = self.ed["root_pos"][:, 0:1] + self.ray_offsets[None, :]
            h = np.zeros_like(xs) if self.samples is None else raw_heights(self.samples, self.spacing, xs)
            self.ray_cache = h - self.ed["root_pos"][:, 1:2]
            self.ray_step = self.S["sim_step"]
        return self.ray_cache

    # ------------------------------------------------------------------ capture

    def capture_push(self):  # capture.py:53-59
        K = self.cap_q.shape[0]
        self.cap_head = (self.cap_head + 1) % K
        self.cap_q[self.cap_head] = self.S["q"]
        self.cap_qd[self.cap_head] = self.S["qd"]
        self.cap_ctrl[self.cap_head] = self.S["ctrl"]
        self.cap_steps[self.cap_head] = self.S["sim_step"]
        self.cap_count = min(self.cap_count + 1, K)

    def capture_frames(self):  # capture.py:61-78
        K = self.cap_q.shape[0]
        out = []
        for i in range(self.cap_count):
            s = (self.cap_head - self.cap_count + 1 + i) % K
            out.append((self.cap_q[s].copy(), self.cap_qd[s].copy(), self.cap_ctrl[s].copy(), int(self.cap_steps[s])))
        return out

    # ------------------------------------------------------------------ commands

    def _build_commands(self):  # managers/command.py:15-31
        cc = self.cfg.commands
        self.cmd_channels = list(cc.ranges)
        base = np.array([cc.ranges[ch] for ch in self.cmd_channels]).reshape(len(self.cmd_channels), 2)
        self.init_ranges = np.broadcast_to(base, (self.n, len(self.cmd_channels), 2)).copy()
        self.ranges = self.init_ranges.copy()
        self.command = np.zeros((self.n, len(self.cmd_channels)))
        self.period_steps = max(1, int(round(cc.resample_period / self.dt_control)))
        self.countdown = np.full(self.n, self.period_steps, dtype=np.int64)

    def cmd_resample(self, ids):  # managers/command.py:33-39
        if not len(ids):
            return
        self.command[ids] = self.rng.uniform("command", self.ranges[ids, :, 0], self.ranges[ids, :, 1], ids,
                                             len(self.cmd_channels))
        self.countdown[ids] = self.period_steps

    def cmd_update(self):  # managers/command.py:41-45
        self.countdown -= 1
        self.cmd_resample(np.flatnonzero(self.countdown <= 0))

    def cmd_widen(self, ids, factor):  # managers/command.py:47-50
        bound = np.abs(self.init_ranges[ids]) * self.cfg.commands.cap_scale
        self.ranges[ids] = np.clip(self.ranges[ids] * factor, -bound, bound)

    # ------------------------------------------------------------------ rewards

    def _build_rewards(self):  # managers/reward.py:20-33
        self.rw = dict(self.cfg.rewards)
        self.weights = {k: c.weight for k, c in self.rw.items()}
        self.ep_sums = {k: np.zeros(self.n) for k in self.rw}
        self.ep_raw = {k: np.zeros(self.n) for k in self.rw}
        self.last_values = {k: np.zeros(self.n) for k in self.rw}
        self.rew_report = {}

    def _reward_term(self, func, p):  # mdp.py:96-160
        ed = self.ed
        if func == "constant":
            return np.full(self.n, p.get("value", 1.0))
        if func == "base_height":
            return self.S["q"][:, 1].copy()
        if func == "track_vx_exp":
            std = p.get("std", 0.25)
            err = self.command[:, 0] - ed["lin_vel_b"][:, 0]
            return np.exp(-(err * err) / (std * std))
        if func == "pitch_rate_penalty":
            return ed["ang_vel"] * ed["ang_vel"]
        if func == "angular_momentum_penalty":
            mom = np.broadcast_to(self.field("base_inertia"), (self.n,)) * ed["ang_vel"]
            return mom * mom
        if func == "action_rate_penalty":
            d = self.action - self.prev_action
            return (d * d).sum(axis=1)
        if func == "joint_limit_penalty":
            lim = self.m.limits
            mid = 0.5 * (lim[:, 0] + lim[:, 1])
            half = 0.5 * (lim[:, 1] - lim[:, 0]) * self.m.soft
            return np.maximum(0.0, np.abs(ed["joint_pos"] - mid) - half).sum(axis=1)
        if func == "foot_slip_penalty":
            return (np.abs(ed["foot_vel"][:, :, 0]) * ed["foot_in_contact"]).sum(axis=1)
        if func == "feet_air_time":
            landed = self.sens["td"] > self.S["sim_step"] - self.decimation
            return ((self.sens["last_air"] - p.get("target_air_time", 0.3)) * landed).sum(axis=1)
        return self.custom[func](self, **p)

    def reward_compute(self):  # managers/reward.py:36-49
        self.rew_report = {}
        total = np.zeros(self.n)
        dt = self.dt_control
        for k, c in self.rw.items():
            v = np.asarray(self._reward_term(c.func, c.params), dtype=np.float64)
            bad = ~np.isfinite(v)
            if bad.any():
                self.rew_report[k] = bad
            contrib = self.weights[k] * v * dt
            total += contrib
            self.ep_sums[k] += contrib
            self.ep_raw[k] += v
            self.last_values[k] = v
        return total

    def reward_reset(self, ids):  # managers/reward.py:55-62
        fin = {}
        for k in self.rw:
            fin[k] = self.ep_sums[k][ids].copy()
            self.ep_sums[k][ids] = 0.0
            self.ep_raw[k][ids] = 0.0
        return fin

    # ------------------------------------------------------------------ terminations

    def _build_terminations(self):
        self.tm = dict(self.cfg.terminations)
        self.trigger_counts = {k: 0 for k in self.tm}
        self.trigger_counts["nonfinite"] = 0
        self.last_nonfinite = np.zeros(self.n, dtype=bool)

    def termination_compute(self):  # managers/termination.py:24-41, mdp.py:167-179
        term = np.zeros(self.n, dtype=bool)
        trunc = np.zeros(self.n, dtype=bool)
        q = self.S["q"]
        for k, c in self.tm.items():
            p = c.params
            if c.func == "base_height_below":
                m = q[:, 1] < p.get("min_height", 0.15)
            elif c.func == "pitch_beyond":
                m = np.abs(q[:, 2]) > p.get("max_pitch", 1.0)
            elif c.func == "time_out":
                m = self.episode_steps >= self.max_episode_steps
            else:
                m = self.custom[c.func](self, **p)
            m = np.asarray(m, dtype=bool)
            self.trigger_counts[k] += int(m.sum())
            if c.time_out:
                trunc |= m
            else:
                term |= m
        bad = ~np.isfinite(self.S["q"]).all(axis=1)  # sim/state.py:69-74
        bad |= ~np.isfinite(self.S["qd"]).all(axis=1)
        bad |= ~np.isfinite(self.S["ctrl"]).all(axis=1)
        self.last_nonfinite = bad
        if bad.any():
            self.trigger_counts["nonfinite"] += int(bad.sum())
            term |= bad
        return term, trunc

    # ------------------------------------------------------------------ events

    def _build_events(self):  # managers/event.py:55-73
        self.ev = dict(self.cfg.events)
        self.ev_elapsed, self.ev_target = {}, {}
        for k, c in self.ev.items():
            if c.mode == "interval":
                self.ev_elapsed[k] = np.zeros(self.n)
                self.ev_target[k] = np.zeros(self.n)
                self._draw_targets(k, np.arange(self.n))

    def _draw_targets(self, k, ids):  # managers/event.py:75-84
        lo, hi = self.ev[k].interval_range
        dt = self.dt_control
        draw = self.rng.uniform(f"event.{k}.interval", lo, hi, ids, 1)[:, 0]
        self.ev_target[k][ids] = np.clip(np.round(draw / dt) * dt, np.ceil(lo / dt) * dt, np.floor(hi / dt) * dt)

    def randomize_field(self, field, distribution, rng_range, operation, ids, purpose):  # managers/event.py:19-52
        self.m.expand(field)
        f = self.m.fields[field]
        size = int(np.prod(f[2].shape)) if f[2].shape else 1
        if distribution == "uniform":
            draw = self.rng.uniform(purpose, rng_range[0], rng_range[1], ids, size)
        else:
            draw = rng_range[0] + self.rng.normal(purpose, rng_range[1], ids, size)
        draw = draw.reshape((len(ids),) + f[2].shape)
        base = np.broadcast_to(f[2], (len(ids),) + f[2].shape)
        if operation == "set":
            f[0][ids] = draw
        elif operation == "scale":
            f[0][ids] = base * draw
        else:
            f[0][ids] = base + draw

    def _event(self, func, ids, p):  # mdp.py:186-220
        ids = np.asarray(ids)
        if func == "randomize_model_field":
            fld = p.get("field", "friction")
            self.randomize_field(fld, p.get("distribution", "uniform"), tuple(p.get("rng_range", (0.8, 1.2))),
                                 p.get("operation", "scale"), ids, f"event.randomize.{fld}")
        elif func == "push_base":
            fx = p.get("fx_range", (-50.0, 50.0))
            fz = p.get("fz_range", (0.0, 0.0))
            self.S["ext"][ids, 0] += self.rng.uniform("event.push.fx", *fx, ids, 1)[:, 0]
            self.S["ext"][ids, 1] += self.rng.uniform("event.push.fz", *fz, ids, 1)[:, 0]
        elif func == "reset_joints_jitter":
            pr = p.get("pos_range", (-0.1, 0.1))
            self.S["q"][ids, 3:] += self.rng.uniform("event.joint_jitter", *pr, ids, self.m.k)
        else:
            self.custom[func](self, ids, **p)

    def event_startup(self):
        for k, c in self.ev.items():
            if c.mode == "startup":
                self._event(c.func, np.arange(self.n), c.params)

    def event_reset(self, ids):  # managers/event.py:92-101
        if not len(ids):
            return
        for k, c in self.ev.items():
            if c.mode == "reset":
                self._event(c.func, ids, c.params)
            elif c.mode == "interval":
                self.ev_elapsed[k][ids] = 0.0
                self._draw_targets(k, ids)

    def event_interval(self, dt):  # managers/event.py:103-114
        for k, c in self.ev.items():
            if c.mode != "interval":
                continue
            el = self.ev_elapsed[k]
            el += dt
            fire = el >= self.ev_target[k] - 0.5 * dt
            if fire.any():
                ids = np.flatnonzero(fire)
                self._event(c.func, ids, c.params)
                el[ids] = 0.0
                self._draw_targets(k, ids)

    # ------------------------------------------------------------------ curriculum

    def curriculum_update(self, ids):  # managers/curriculum.py:21-23, mdp.py:227-275
        for k, c in self.curriculum.items():
            p = c.params
            if c.func == "terrain_levels":
                if not len(ids):
                    continue
                walked = np.abs(self.S["q"][ids, 0] - self.episode_start_x[ids])
                cmd = self.commanded_distance[ids]
                rows = self.terrain_rows[ids]
                rows = np.where(walked >= p.get("promote_ratio", 0.8) * cmd, rows + 1, rows)
                rows = np.where(walked <= p.get("demote_ratio", 0.4) * cmd, rows - 1, rows)
                self.terrain_rows[ids] = np.clip(rows, 0, self.t_rows - 1)
            elif c.func == "command_widen":
                if not len(ids):
                    continue
                steps = self.episode_steps[ids].astype(np.float64)
                mean = self.ep_raw[p.get("term", "track_vx_exp")][ids] / np.maximum(steps, 1)
                good = ids[mean > p.get("threshold", 0.8)]
                if good.size:
                    self.cmd_widen(good, p.get("factor", 1.2))
            elif c.func == "reward_weight_schedule":
                span = max(1, p.get("end_step", 1000) - p.get("start_step", 0))
                frac = np.clip((self.global_step - p.get("start_step", 0)) / span, 0.0, 1.0)
                sw, ew = p.get("start_weight", 1.0), p.get("end_weight", 0.0)
                self.weights[p.get("term", "")] = sw + frac * (ew - sw)
            else:
                self.custom[c.func](self, ids, **p)

    # ------------------------------------------------------------------ observations

    def _build_observations(self):  # managers/observation.py:24-67
        self.groups = {}
        self.obs_pending = {}
        for g, gc in self.cfg.observations.items():
            terms = []
            for name, tc in gc.terms.items():
                probe = self._obs_raw(tc.func, tc.params)
                dim = probe.shape[1]
                terms.append({"name": name, "cfg": tc, "dim": dim, "purpose": f"obs.{g}.{name}",
                              "dring": np.zeros((tc.delay_steps + 1, self.n, dim)), "dhead": 0,
                              "hring": np.zeros((tc.history, self.n, dim))})
            self.groups[g] = (gc, terms)
            self.obs_pending[g] = np.zeros(self.n, dtype=bool)
        self.obs_report = {}

    def _obs_raw(self, func, p):  # mdp.py:26-89
        ed = self.ed
        if func == "base_lin_vel":
            v = ed["lin_vel_b"]
        elif func == "base_ang_vel":
            v = ed["ang_vel"][:, None]
        elif func == "base_lin_acc":
            v = (ed["lin_vel_b"] - self.prev_lin_vel_b) / self.dt_control
        elif func == "projected_gravity":
            v = ed["proj_grav"]
        elif func == "joint_pos_rel":
            v = ed["joint_pos"] - self.default_joint_pos
        elif func == "joint_vel":
            v = ed["joint_vel"]
        elif func == "last_action":
            v = self.action
        elif func == "command":
            v = self.command
        elif func == "base_height":
            v = self.S["q"][:, 1:2]
        elif func == "sim_time":
            v = self.S["time"][:, None]
        elif func == "height_scan":
            v = self.ray_read()
        elif func == "foot_contact_forces":
            v = ed["foot_forces"].reshape(self.n, -1)
        else:
            v = self.custom[func](self, **p)
        v = np.atleast_2d(np.asarray(v, dtype=np.float64))
        if v.shape[0] != self.n:
            v = v.T
        return v

    def obs_compute(self, g):  # managers/observation.py:99-137
        gc, terms = self.groups[g]
        pend = self.obs_pending[g]
        rids = np.flatnonzero(pend)
        pieces = []
        for t in terms:
            tc = t["cfg"]
            raw = self._obs_raw(tc.func, tc.params)
            bad = ~np.isfinite(raw).all(axis=1)
            if bad.any():
                self.obs_report[t["name"]] = bad
            v = raw
            if tc.clip is not None:
                v = np.clip(v, tc.clip[0], tc.clip[1])
            if tc.scale is not None:
                v = v * tc.scale
            nz = tc.noise
            if gc.enable_noise and nz.kind != "none" and nz.scale:
                if nz.kind == "uniform":
                    v = v + self.rng.uniform(t["purpose"], -nz.scale, nz.scale, None, t["dim"])
                else:
                    v = v + self.rng.normal(t["purpose"], nz.scale, None, t["dim"])
            if tc.delay_steps == 0 and tc.history == 1:
                pieces.append(v)
                continue
            D1 = tc.delay_steps + 1
            t["dhead"] = (t["dhead"] + 1) % D1
            t["dring"][t["dhead"]] = v
            if rids.size:
                t["dring"][:, rids, :] = v[rids]
            delayed = t["dring"][(t["dhead"] - tc.delay_steps) % D1]
            t["hring"][:-1] = t["hring"][1:]
            t["hring"][-1] = delayed
            if rids.size:
                t["hring"][:, rids, :] = delayed[rids]
            pieces.append(t["hring"].transpose(1, 0, 2).reshape(self.n, -1))
        out = pieces[0].copy() if len(pieces) == 1 else np.concatenate(pieces, axis=1)
        pend[:] = False
        return out

    def obs_all(self):
        self.obs_report = {}
        return {g: self.obs_compute(g) for g in self.groups}

    # ------------------------------------------------------------------ reset / step

    def _reset_worlds(self, ids):  # env.py:182-200
        self._write_default(ids)
        self._place(ids)
        self.event_reset(ids)
        self.cmd_resample(ids)
        self.action_reset(ids)
        self.sensor_reset(ids)
        self.ray_step = -1
        S = self.S
        S["fn"][ids] = 0.0
        S["ft"][ids] = 0.0
        S["fvel"][ids] = 0.0
        S["fin"][ids] = False
        for p in self.obs_pending.values():
            p[ids] = True
        fin = self.reward_reset(ids)
        self.episode_steps[ids] = 0
        self.episode_start_x[ids] = S["q"][ids, 0]
        self.commanded_distance[ids] = 0.0
        self.finalized = (ids, fin)

    def reset(self, seed=None):  # env.py:202-215
        if seed is not None:
            self.rng = OracleStreams(seed, self.world_ids)
            self._startup_done = False
        if not self._startup_done:
            self.event_startup()
            self._startup_done = True
        self._reset_worlds(np.arange(self.n))
        self.refresh()
        self.prev_lin_vel_b[...] = self.ed["lin_vel_b"]
        return self.obs_all()

    def step(self, actions):  # env.py:219-259
        self.global_step += 1
        self.action_process(actions)
        for _ in range(self.decimation):
            self.action_apply()
            if self.capture:
                self.capture_push()
            oracle_substep(self.m, self.heights, self.S)
            self.refresh()
            self.sensor_update()
        self.episode_steps += 1
        if len(self.cmd_channels):
            self.commanded_distance += np.abs(self.command[:, 0]) * self.dt_control
        term, trunc = self.termination_compute()
        reward = self.reward_compute()
        reset_ids = np.flatnonzero(term | trunc)
        self.finalized = (reset_ids, {})
        self.curriculum_update(reset_ids)
        if reset_ids.size:
            self._reset_worlds(reset_ids)
            self.refresh()
        self.cmd_update()
        self.event_interval(self.dt_control)
        obs = self.obs_all()
        self.prev_lin_vel_b[...] = self.ed["lin_vel_b"]
        return obs, reward, term, trunc, {"reset_ids": reset_ids}

    def random_actions(self):  # policies.py:14-16
        return self.rng.uniform("policy.random", -1.0, 1.0, None, self.action_dim)
