"""Algorithmic HBM bytes of one fused control step, per world.

This enumerates what the fused kernel must move for a world that does not
reset in that step (the steady state; ~3 % of worlds reset per step under
random actions and their extra reset writes are excluded). It is the
roofline numerator quoted by bench.py and DESIGN.md: state is resident in
HBM between steps, every array is read once and written once, nothing is
re-read. Counted per world per control step (d substeps included).
"""

from __future__ import annotations

F64, I64, U8, U32, U64 = 8, 8, 1, 4, 8


def step_bytes_per_world(env, fused_policy: bool = False) -> dict:
    """``fused_policy``: the step draws its actions from stream policy.random
    (policies.RandomActions) instead of reading an (N, A) action row."""
    m = env.model
    k, nq, nf = m.num_joints, m.nq, len(m.feet)
    d = env.decimation
    am, om, rm = env.action_manager, env.observation_manager, env.reward_manager
    A = am.total_dim
    C = len(env.command_manager.channels)
    T = len(rm.terms)
    H = env.contact_sensor.cfg.history_length
    rd, wr = {}, {}
    # physics state (BatchState): q, qd read+write; ctrl written; ext read+write; time r/w
    rd["q,qd,ext,time"] = F64 * (2 * nq + 2 + 1)
    wr["q,qd,ctrl,ext,time"] = F64 * (2 * nq + k + 2 + 1)
    # contact cache of the last substep
    wr["contact cache"] = F64 * (6 * nf) + U8 * nf
    # per-world expanded model fields
    n_exp = sum(f.size for f in m._fields.values() if f.expanded)
    rd["expanded fields"] = F64 * n_exp
    # actions: input row, previous action -> prev, action; targets
    if fused_policy:
        rd["policy counter + action"] = U64 + F64 * A
        wr["policy counter"] = U64
    else:
        rd["actions in + action"] = F64 * (2 * A)
    wr["action, prev, targets"] = F64 * (2 * A + k)
    # delayed actuators: ring push + read per substep, delays
    for a in am.actuators:
        if a.delay is not None:
            rd[f"delay {a.name}"] = I64 + F64 * d * len(a.joint_ids)
            wr[f"delay {a.name}"] = F64 * d * len(a.joint_ids)
    # capture ring: one frame per substep
    wr["capture ring"] = F64 * d * (2 * nq + k)
    # contact sensor
    need_hist = d < H
    rd["contact sensor"] = U8 * nf + F64 * 3 * nf + I64 * nf + (F64 * H * nf if need_hist else 0)
    wr["contact sensor"] = U8 * nf + F64 * 5 * nf + I64 * nf + F64 * H * nf
    # command (read), countdown r/w, episode bookkeeping r/w
    rd["command, countdown, episode"] = F64 * C + I64 + I64 + F64
    wr["countdown, episode"] = I64 + I64 + F64
    # termination flags
    wr["terminated, truncated, nonfinite"] = 3 * U8
    # rewards: sums + raw r/w, last values + total written
    rd["reward sums"] = F64 * 2 * T
    wr["reward sums, values, total"] = F64 * (3 * T + 1)
    # interval events: elapsed r/w, target read (+ fired byte for plugins)
    n_iv = sum(1 for tc in env.cfg.events.values() if tc.mode == "interval")
    rd["event stopwatch"] = F64 * 2 * n_iv
    wr["event stopwatch"] = F64 * n_iv
    # observations: outputs, rings, noise counters
    n_obs = sum(om.group_dim(g) for g in om.groups)
    wr["observations"] = F64 * n_obs + U32
    uses_acc = any(t.cfg.func == "base_lin_acc" for t in om.all_terms())
    rd["prev_lin_vel_b"] = F64 * 2 if uses_acc else 0
    wr["prev_lin_vel_b"] = F64 * 2
    rings_r = rings_w = 0
    noise_slots = 0
    for t in om.all_terms():
        if t.cfg.delay_steps > 0:
            rings_w += F64 * t.dim
            rings_r += F64 * t.dim
        if t.cfg.history > 1:
            rings_w += F64 * t.dim
            rings_r += F64 * t.dim * (t.cfg.history - 1)
        g = next(g for g, ts in om.groups.items() if t in ts)
        if om.group_cfgs[g].enable_noise and t.cfg.noise.kind != "none" and t.cfg.noise.scale:
            noise_slots += 1
    rd["obs rings"] = rings_r
    wr["obs rings"] = rings_w
    rd["rng counters"] = U64 * noise_slots
    wr["rng counters"] = U64 * noise_slots
    reads, writes = sum(rd.values()), sum(wr.values())
    return {"read": reads, "write": writes, "total": reads + writes, "read_items": rd, "write_items": wr}


def policy_bytes_per_world(env) -> int:
    """random_policy: one counter r/w + the (N, A) action row written."""
    return U64 * 2 + F64 * env.action_manager.total_dim
