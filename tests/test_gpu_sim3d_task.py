"""Fused 3-D velocity task (one launch per control step) vs the oracle's TaskOracle.

Parity unpinned w.r.t. the reference (no 3-D engine there).
float64: observations, rewards within 1e-8 (free-running, few control steps,
before chaotic contact divergence); termination / truncation flags and reset
worlds bit-exact; teacher-forced single steps bit-exact on flags across
forced terminations, truncations and command resampling.
"""

import numpy as np
import pytest

from oracle import sim3d as O
from paper_2601_22074_b200.sim3d import robots
from paper_2601_22074_b200.sim3d.task import VelocityTaskCfg

CASES = {
    "g1_flat": (lambda: robots.g1_like(), robots.G1_DEFAULT_JOINTS, dict()),
    "g1_curriculum": (lambda: robots.g1_like(rough="curriculum", seed=2), robots.G1_DEFAULT_JOINTS,
                      dict(height_scan=True, curriculum=(5, 6, 8.0), curriculum_max_init_level=3)),
    "g1_rough_scan": (lambda: robots.g1_like(rough=True, seed=1), robots.G1_DEFAULT_JOINTS, dict(height_scan=True)),
    "go1_flat": (lambda: robots.go1_like(), robots.GO1_DEFAULT_JOINTS, dict(min_height=0.15)),
}


def _pair(name, n, dtype="f64", **over):
    from paper_2601_22074_b200.sim3d.task import VelocityEnv3D

    make, table, kw = CASES[name]
    kw = dict(kw, **over)
    mg, mo = make(), make()
    cfg = VelocityTaskCfg(default_qpos=robots.default_qpos(mg, table), **kw)
    env = VelocityEnv3D(mg, cfg, n, seed=7, dtype=dtype)
    O.set_const(mo)
    ref = O.TaskOracle(mo, cfg, n, seed=7)
    return env, ref


@pytest.mark.gpu
@pytest.mark.parametrize("name", list(CASES))
def test_reset_and_free_running_steps_f64(name):
    import torch

    n = 8
    env, ref = _pair(name, n)
    o = env.reset().cpu().numpy()
    o_ref = ref.reset()
    np.testing.assert_allclose(o, o_ref, rtol=0, atol=1e-12)
    rng = np.random.default_rng(0)
    for k in range(4):
        a = rng.uniform(-1, 1, size=(n, env.model.nu))
        o, r, te, tr = env.step(torch.as_tensor(a, device="cuda"))
        o_ref, r_ref, te_ref, tr_ref = ref.step(a)
        torch.cuda.synchronize()
        np.testing.assert_array_equal(te.cpu().numpy().astype(bool), te_ref)
        np.testing.assert_array_equal(tr.cpu().numpy().astype(bool), tr_ref)
        np.testing.assert_allclose(r.cpu().numpy(), r_ref, rtol=1e-8, atol=1e-10)
        np.testing.assert_allclose(o.cpu().numpy(), o_ref, rtol=1e-7, atol=1e-7)


def _load(env, ref):
    import torch

    t = lambda x: torch.as_tensor(x, device="cuda")  # noqa: E731
    env.data.qpos.copy_(t(ref.qpos))
    env.data.qvel.copy_(t(ref.qvel))
    env.data.qacc_warmstart.copy_(t(ref.warm))
    env.action.copy_(t(ref.action))
    env.prev_action.copy_(t(ref.prev_action))
    env.command.copy_(t(ref.cmd))
    env.cmd_timer.copy_(t(ref.cmd_timer.astype(np.int32)))
    env.episode_step.copy_(t(ref.episode_step.astype(np.int32)))
    if getattr(env, "event_timer", None) is not None:
        env.event_timer.copy_(t(ref.ev_timer))
        env.data.friction_scale.copy_(t(ref.fscale))
        env.data.mass_scale.copy_(t(ref.mscale))
    if getattr(env, "terrain_level", None) is not None:
        env.terrain_level.copy_(t(ref.level.astype(np.int32)))
        env.spawn_xy.copy_(t(ref.spawn))
        env.cmd_dist.copy_(t(ref.cmd_dist))
    env.global_step = ref.global_step


@pytest.mark.gpu
def test_teacher_forced_resets_truncations_and_commands():
    """Short episodes and command periods force truncation resets and resamples; a tight height
    threshold forces terminations: every step's flags, reset state and draws must match."""
    import torch

    n = 8
    env, ref = _pair("g1_rough_scan", n, episode_steps=3, command_resample_steps=2, min_height=0.78)
    env.reset()
    ref.reset()
    rng = np.random.default_rng(3)
    saw_term = saw_trunc = 0
    for k in range(7):
        _load(env, ref)
        a = rng.uniform(-1, 1, size=(n, env.model.nu))
        o, r, te, tr = env.step(torch.as_tensor(a, device="cuda"))
        o_ref, r_ref, te_ref, tr_ref = ref.step(a)
        torch.cuda.synchronize()
        np.testing.assert_array_equal(te.cpu().numpy().astype(bool), te_ref)
        np.testing.assert_array_equal(tr.cpu().numpy().astype(bool), tr_ref)
        np.testing.assert_allclose(r.cpu().numpy(), r_ref, rtol=1e-8, atol=1e-10)
        np.testing.assert_allclose(o.cpu().numpy(), o_ref, rtol=1e-7, atol=1e-7)
        np.testing.assert_allclose(env.command.cpu().numpy(), ref.cmd, atol=1e-15)
        np.testing.assert_array_equal(env.cmd_timer.cpu().numpy(), ref.cmd_timer)
        np.testing.assert_array_equal(env.episode_step.cpu().numpy(), ref.episode_step)
        saw_term += int(te_ref.sum())
        saw_trunc += int(tr_ref.sum())
    assert saw_term > 0 and saw_trunc > 0


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["g1_rough_scan", "go1_flat"])
def test_velocity_penalties_angular_momentum_limits_foot_slip(name):
    """PAPER.md §6.1's velocity penalties, each isolated by its weight: the robot's centroidal angular
    momentum, joint-limit violation (joints loaded past their ranges) and foot slip (feet in ground contact,
    read from the per-foot contact sensors, with random base velocities): kernel vs oracle, every step;
    the feet's sensors equal the oracle's."""
    import torch

    n = 8
    for term in (6, 7, 8):
        wts = [0.0] * 9
        wts[term] = 1.0
        env, ref = _pair(name, n, reward_weights=tuple(wts), min_height=0.0, max_tilt_cos=1.0, push_interval=None)
        env.reset()
        ref.reset()
        m = ref.m
        lim = np.nonzero(m.jnt_limited)[0]
        for w in range(n):
            j = lim[w % lim.size]
            ref.qpos[w, m.jnt_qposadr[j]] = m.jnt_range[j][w % 2] + (0.5 if w % 2 else -0.5)
            ref.qvel[w, m.jnt_dofadr[j]] = 5.0 if w % 2 else -5.0  # still moving outwards
            ref.qvel[w, 0:6] += np.random.default_rng(w).normal(size=6) * 0.5
        rng = np.random.default_rng(4)
        seen = 0.0
        for k in range(2):
            _load(env, ref)
            a = rng.uniform(-1, 1, size=(n, env.model.nu))
            o, r, te, tr = env.step(torch.as_tensor(a, device="cuda"))
            o_ref, r_ref, te_ref, tr_ref = ref.step(a)
            torch.cuda.synchronize()
            np.testing.assert_allclose(r.cpu().numpy(), r_ref, rtol=1e-8, atol=1e-12)
            np.testing.assert_array_equal(env.sensor.cpu().numpy(), ref.sensor)
            seen = max(seen, float(np.abs(r_ref).max()))
        assert seen > 0, term  # (the limit constraint pushes the joints back in range within a step or two)
        assert len(env.sensor_names) == len(ref.cfg.foot_bodies(m)) and ref.sensor.max() > 0


@pytest.mark.gpu
def test_f32_task_close_to_oracle():
    import torch

    n = 8
    env, ref = _pair("g1_flat", n, dtype="f32")
    o = env.reset().double().cpu().numpy()
    np.testing.assert_allclose(o, ref.reset(), atol=1e-5)
    a = np.random.default_rng(1).uniform(-1, 1, size=(n, env.model.nu)).astype(np.float32)
    o, r, te, tr = env.step(torch.as_tensor(a, device="cuda"))
    o_ref, r_ref, te_ref, _ = ref.step(a.astype(np.float64))
    torch.cuda.synchronize()
    np.testing.assert_array_equal(te.cpu().numpy().astype(bool), te_ref)
    np.testing.assert_allclose(r.double().cpu().numpy(), r_ref, atol=1e-4)
    np.testing.assert_allclose(o.double().cpu().numpy(), o_ref, atol=5e-3 * max(1.0, np.abs(o_ref).max()))


@pytest.mark.gpu
def test_world_offset_partition_independence():
    """Two shards with world_id offsets reproduce one big batch (worlds are independent)."""
    import torch

    from paper_2601_22074_b200.sim3d.task import VelocityEnv3D

    make, table, kw = CASES["go1_flat"]
    cfg = VelocityTaskCfg(default_qpos=robots.default_qpos(make(), table), **kw)
    full = VelocityEnv3D(make(), cfg, 8, seed=3)
    a0 = VelocityEnv3D(make(), cfg, 4, seed=3, world_offset=0)
    a1 = VelocityEnv3D(make(), cfg, 4, seed=3, world_offset=4)
    of = full.reset().clone()
    assert torch.equal(of, torch.cat([a0.reset(), a1.reset()]))
    act = torch.rand(8, full.model.nu, dtype=torch.float64, device="cuda") * 2 - 1
    for _ in range(3):
        of, rf, _, _ = full.step(act)
        o0, r0, _, _ = a0.step(act[:4].contiguous())
        o1, r1, _, _ = a1.step(act[4:].contiguous())
    assert torch.equal(of, torch.cat([o0, o1])) and torch.equal(rf, torch.cat([r0, r1]))


@pytest.mark.gpu
@pytest.mark.parametrize("dtype", ["f32", "f64"])
def test_block_phase_sync_is_bit_identical(dtype):
    """The block barriers (flags bits 3-5) only change when warps run: results are bit-identical with
    and without them, including the partial last block (5000 worlds)."""
    import torch

    from paper_2601_22074_b200.sim3d.task import VelocityEnv3D

    m = robots.g1_like(rough=True, seed=2)
    cfg = VelocityTaskCfg(default_qpos=robots.default_qpos(m, robots.G1_DEFAULT_JOINTS), height_scan=True)
    n = 5000
    a = VelocityEnv3D(m, cfg, n, seed=5, dtype=dtype)
    b = VelocityEnv3D(robots.g1_like(rough=True, seed=2), cfg, n, seed=5, dtype=dtype)
    assert a.dm.struct.flags & 40 == 40
    b.dm.struct.flags = a.dm.struct.flags & ~56
    assert torch.equal(a.reset(), b.reset())
    g = torch.Generator(device="cuda").manual_seed(0)
    for _ in range(3):
        act = (torch.rand(n, m.nu, device="cuda", generator=g) * 2 - 1).to(a.data.qpos.dtype)
        oa, ra, ta, _ = a.step(act)
        ob, rb, tb, _ = b.step(act)
        assert torch.equal(oa, ob) and torch.equal(ra, rb) and torch.equal(ta, tb)
    assert torch.equal(a.data.qpos, b.data.qpos) and torch.equal(a.data.qvel, b.data.qvel)


@pytest.mark.gpu
@pytest.mark.parametrize("n", [700, 5000])
def test_launch_shape_is_bit_identical(n):
    """Warps per block only decide where a world runs: the wave-balanced launch (flags bit 6, the G1
    default), the maximal block and a fixed small block give bit-identical steps, for one partial wave
    (700 worlds) and several waves (5000)."""
    import torch

    from paper_2601_22074_b200.sim3d.task import VelocityEnv3D

    m = robots.g1_like(rough=True, seed=2)
    cfg = VelocityTaskCfg(default_qpos=robots.default_qpos(m, robots.G1_DEFAULT_JOINTS), height_scan=True)
    envs = [VelocityEnv3D(robots.g1_like(rough=True, seed=2), cfg, n, seed=5, dtype="f32") for _ in range(3)]
    assert envs[0].dm.struct.flags & 64
    envs[1].dm.struct.flags &= ~64
    envs[2].dm.layout.warps_per_block = 3
    envs[2].dm.layout.bytes_per_block = 3 * envs[2].dm.layout.elems_per_world * 4
    outs = [e.reset() for e in envs]
    assert all(torch.equal(outs[0], o) for o in outs[1:])
    g = torch.Generator(device="cuda").manual_seed(0)
    for _ in range(3):
        act = torch.rand(n, m.nu, device="cuda", generator=g) * 2 - 1
        res = [e.step(act) for e in envs]
        for r in res[1:]:
            assert all(torch.equal(a, b) for a, b in zip(res[0], r))
    assert all(torch.equal(envs[0].data.qpos, e.data.qpos) for e in envs[1:])


@pytest.mark.gpu
@pytest.mark.parametrize("dtype", ["f32", "f64"])
def test_cost_ordered_schedule_is_bit_identical(dtype, monkeypatch):
    """Sorting the worlds by their last solver cost before each step (s3_task.cost / order) only changes
    which warp steps which world: results are bit-identical to the identity schedule, and the order is a
    permutation sorted by cost (heaviest first)."""
    import torch

    from paper_2601_22074_b200.sim3d.task import VelocityEnv3D

    m = robots.g1_like(rough=True, seed=2)
    cfg = VelocityTaskCfg(default_qpos=robots.default_qpos(m, robots.G1_DEFAULT_JOINTS), height_scan=True)
    n = 5000
    a = VelocityEnv3D(m, cfg, n, seed=5, dtype=dtype)
    monkeypatch.setenv("S3_ORDER", "0")
    b = VelocityEnv3D(robots.g1_like(rough=True, seed=2), cfg, n, seed=5, dtype=dtype)
    assert a.world_order is not None and b.world_order is None
    assert torch.equal(a.reset(), b.reset())
    g = torch.Generator(device="cuda").manual_seed(0)
    for _ in range(4):
        act = (torch.rand(n, m.nu, device="cuda", generator=g) * 2 - 1).to(a.data.qpos.dtype)
        oa, ra, ta, _ = a.step(act)
        ob, rb, tb, _ = b.step(act)
        assert torch.equal(oa, ob) and torch.equal(ra, rb) and torch.equal(ta, tb)
    assert torch.equal(a.data.qpos, b.data.qpos) and torch.equal(a.data.qvel, b.data.qvel)
    order = a.world_order.long()
    assert torch.equal(order.sort().values, torch.arange(n, device="cuda"))
    assert int(a.solver_cost.min()) >= 0 and int(a.solver_cost.max()) > 0
    # the order the last step used was sorted by the costs of the step before it: re-sorting the current
    # costs must give non-increasing costs along the order the NEXT step will use
    a.step(act)
    prev = a.solver_cost.long().clamp(max=63)  # the sort's buckets
    a._launch(0, act)  # one more step: its order kernel sorted by `prev`
    used = a.world_order.long()
    assert bool((prev[used][1:] <= prev[used][:-1]).all())


def _motion_pair(n, dtype="f64", **over):
    from paper_2601_22074_b200.sim3d.motion import synthetic_walk_clip
    from paper_2601_22074_b200.sim3d.task import MotionTrackingCfg, VelocityEnv3D

    mg, mo = robots.g1_like(rough=True, seed=4), robots.g1_like(rough=True, seed=4)
    dq = robots.default_qpos(mg, robots.G1_DEFAULT_JOINTS)
    Q, V, fdt = synthetic_walk_clip(mg, dq, seconds=4.0)
    cfg = MotionTrackingCfg(default_qpos=dq, motion_qpos=Q, motion_qvel=V, motion_dt=fdt, **over)
    env = VelocityEnv3D(mg, cfg, n, seed=11, dtype=dtype)
    O.set_const(mo)
    return env, O.MotionTaskOracle(mo, cfg, n, seed=11)


@pytest.mark.gpu
def test_motion_imitation_free_running_f64():
    """BeyondMimic-style task (BASELINE configs[2]): reference state initialisation, tracking rewards,
    reference-aware observations match the oracle."""
    import torch

    n = 8
    env, ref = _motion_pair(n)
    np.testing.assert_allclose(env.reset().cpu().numpy(), ref.reset(), atol=1e-12)
    np.testing.assert_allclose(env.command.cpu().numpy(), ref.cmd, atol=1e-12)
    # the clip's body-state table (s3_motion_bodies) against the oracle's FK of every frame
    np.testing.assert_allclose(env.motion_body.cpu().numpy(), ref.body_table, rtol=1e-12, atol=1e-12)
    rng = np.random.default_rng(5)
    for k in range(4):
        a = rng.uniform(-1, 1, size=(n, env.model.nu))
        o, r, te, tr = env.step(torch.as_tensor(a, device="cuda"))
        o_ref, r_ref, te_ref, tr_ref = ref.step(a)
        torch.cuda.synchronize()
        np.testing.assert_array_equal(te.cpu().numpy().astype(bool), te_ref)
        np.testing.assert_array_equal(tr.cpu().numpy().astype(bool), tr_ref)
        np.testing.assert_allclose(r.cpu().numpy(), r_ref, rtol=1e-8, atol=1e-10)
        np.testing.assert_allclose(o.cpu().numpy(), o_ref, rtol=1e-7, atol=1e-7)
        np.testing.assert_array_equal(env.sensor.cpu().numpy(), ref.sensor)


@pytest.mark.gpu
def test_motion_body_terms_and_self_collision_teacher_forced():
    """BeyondMimic's relative body terms and the self-collision cost: worlds loaded with crossed legs
    (self contacts), a yawed / shifted robot (relative frame), and off-clip joint states; each reward term
    is isolated by its weight and compared with the oracle; the self-collision sensor fires."""
    import torch

    n = 8
    for term in range(5, 10):
        w = [0.0] * 10
        w[term] = 1.0
        env, ref = _motion_pair(n, reward_weights=tuple(w), max_height_error=10.0, max_ori_error=10.0)
        env.reset()
        ref.reset()
        m = ref.m
        for i in range(0, n, 2):  # crossed legs in half of the worlds
            ref.qpos[i, m.jnt_qposadr[m.jnt_names.index("left_hip_roll_joint")]] = -0.45
            ref.qpos[i, m.jnt_qposadr[m.jnt_names.index("right_hip_roll_joint")]] = 0.45
        ref.qpos[1, 0:2] += (0.4, -0.3)
        ref.qvel[3] += np.random.default_rng(1).normal(size=m.nv) * 0.5
        rng = np.random.default_rng(7)
        for k in range(2):
            _load(env, ref)
            a = rng.uniform(-1, 1, size=(n, env.model.nu))
            o, r, te, tr = env.step(torch.as_tensor(a, device="cuda"))
            o_ref, r_ref, te_ref, tr_ref = ref.step(a)
            torch.cuda.synchronize()
            np.testing.assert_array_equal(te.cpu().numpy().astype(bool), te_ref)
            np.testing.assert_allclose(r.cpu().numpy(), r_ref, rtol=1e-8, atol=1e-12)
            np.testing.assert_array_equal(env.sensor.cpu().numpy(), ref.sensor)
            assert np.abs(r_ref).max() > 0
        if term == 9:
            assert ref.sensor[:, 0].max() > 0


@pytest.mark.gpu
def test_motion_imitation_teacher_forced_terminations_and_clip_end():
    import torch

    n = 8
    env, ref = _motion_pair(n, max_height_error=0.02, motion_start_frac=1.0, adaptive_alpha=0.3)
    env.reset()
    ref.reset()
    ref.cmd[:4, 0] = ref.clip_end() - 0.01  # four worlds run off the end of the clip in one step
    rng = np.random.default_rng(6)
    saw_term = saw_trunc = 0
    for k in range(5):
        _load(env, ref)
        a = rng.uniform(-1, 1, size=(n, env.model.nu))
        o, r, te, tr = env.step(torch.as_tensor(a, device="cuda"))
        o_ref, r_ref, te_ref, tr_ref = ref.step(a)
        torch.cuda.synchronize()
        np.testing.assert_array_equal(te.cpu().numpy().astype(bool), te_ref)
        np.testing.assert_array_equal(tr.cpu().numpy().astype(bool), tr_ref)
        np.testing.assert_allclose(r.cpu().numpy(), r_ref, rtol=1e-8, atol=1e-10)
        np.testing.assert_allclose(o.cpu().numpy(), o_ref, rtol=1e-7, atol=1e-7)
        np.testing.assert_allclose(env.command.cpu().numpy(), ref.cmd, atol=1e-12)
        # adaptive start-time sampling: the failure average and the cumulative weights of the fold
        np.testing.assert_allclose(env.bin_failed.cpu().numpy(), ref.bin_failed, rtol=1e-14, atol=0)
        np.testing.assert_allclose(env.bin_cum.cpu().numpy(), ref.bin_cum, rtol=1e-14, atol=0)
        saw_term += int(te_ref.sum())
        saw_trunc += int(tr_ref.sum())
    assert saw_term > 0 and saw_trunc > 0 and ref.bin_failed.max() > 0


def _lift_pair(n, dtype="f64", **over):
    from paper_2601_22074_b200.sim3d.task import LiftTaskCfg, VelocityEnv3D

    mg, mo = robots.arm_cube_like(), robots.arm_cube_like()
    cfg = LiftTaskCfg.for_model(mg, robots.default_qpos(mg, robots.ARM_DEFAULT_JOINTS), **over)
    env = VelocityEnv3D(mg, cfg, n, seed=13, dtype=dtype)
    O.set_const(mo)
    return env, O.LiftTaskOracle(mo, cfg, n, seed=13)


@pytest.mark.gpu
def test_cube_lift_free_running_f64():
    """Cube lift (BASELINE configs[3]): reset, claw/cube/goal observations, reach/lift/goal rewards."""
    import torch

    n = 8
    env, ref = _lift_pair(n)
    np.testing.assert_allclose(env.reset().cpu().numpy(), ref.reset(), atol=1e-12)
    assert env.sensor_names == ("ee_cube", "ee_ground", "cube_ground")
    rng = np.random.default_rng(8)
    for k in range(4):
        a = rng.uniform(-1, 1, size=(n, env.model.nu))
        o, r, te, tr = env.step(torch.as_tensor(a, device="cuda"))
        o_ref, r_ref, te_ref, tr_ref = ref.step(a)
        torch.cuda.synchronize()
        np.testing.assert_array_equal(te.cpu().numpy().astype(bool), te_ref)
        np.testing.assert_array_equal(tr.cpu().numpy().astype(bool), tr_ref)
        np.testing.assert_allclose(r.cpu().numpy(), r_ref, rtol=1e-8, atol=1e-10)
        np.testing.assert_allclose(o.cpu().numpy(), o_ref, rtol=1e-7, atol=1e-7)
        np.testing.assert_array_equal(env.sensor.cpu().numpy(), ref.sensor)
    assert ref.sensor[:, 2].min() > 0  # the cube rests on the table


@pytest.mark.gpu
def test_cube_lift_claw_contact_sensors_teacher_forced():
    """End-effector contact sensors: a claw pushed into the table (ee_ground, costed by reward term 5) and
    a claw closed on the cube (ee_cube), compared with the oracle."""
    import torch

    n = 4
    env, ref = _lift_pair(n)
    env.reset()
    ref.reset()
    m, ca = ref.m, ref.cfg.cube_qposadr
    K = O.kinematics(m, ref.qpos[1])
    t0, t1 = K["geom_xpos"][list(ref.cfg.tip_geoms)]
    ref.qpos[1, ca:ca + 3] = t0 + 0.03 * (t1 - t0) / np.linalg.norm(t1 - t0)  # cube against a fingertip
    ref.qpos[2, m.jnt_qposadr[m.jnt_names.index("shoulder_pitch")]] += 0.6  # claw down into the table
    ref.qpos[3, m.jnt_qposadr[m.jnt_names.index("shoulder_pitch")]] += 0.6
    ref.qpos[3, ca:ca + 3] = (0.3, 0.4, ref.cfg.cube_half)
    seen = np.zeros(3)
    rng = np.random.default_rng(10)
    for k in range(3):
        _load(env, ref)
        a = rng.uniform(-0.2, 0.2, size=(n, env.model.nu))
        o, r, te, tr = env.step(torch.as_tensor(a, device="cuda"))
        o_ref, r_ref, te_ref, tr_ref = ref.step(a)
        torch.cuda.synchronize()
        np.testing.assert_array_equal(env.sensor.cpu().numpy(), ref.sensor)
        np.testing.assert_allclose(r.cpu().numpy(), r_ref, rtol=1e-8, atol=1e-10)
        seen = np.maximum(seen, ref.sensor.max(0))
    assert seen[0] > 0 and seen[1] > 0


@pytest.mark.gpu
@pytest.mark.parametrize("task", ["motion", "lift"])
def test_f32_motion_and_lift_close_to_oracle(task):
    """float32 builds of BASELINE configs[2] / [3] (partial Newton refactorization, phase sync, cost order):
    one control step from the oracle's reset within float32 tolerances; flags exact."""
    import torch

    n = 8
    env, ref = (_motion_pair if task == "motion" else _lift_pair)(n, dtype="f32")
    o = env.reset().double().cpu().numpy()
    o_ref = ref.reset()
    np.testing.assert_allclose(o, o_ref, atol=1e-5 * max(1.0, np.abs(o_ref).max()))
    a = np.random.default_rng(3).uniform(-1, 1, size=(n, env.model.nu)).astype(np.float32)
    o, r, te, tr = env.step(torch.as_tensor(a, device="cuda"))
    o_ref, r_ref, te_ref, tr_ref = ref.step(a.astype(np.float64))
    torch.cuda.synchronize()
    np.testing.assert_array_equal(te.cpu().numpy().astype(bool), te_ref)
    np.testing.assert_array_equal(tr.cpu().numpy().astype(bool), tr_ref)
    np.testing.assert_allclose(r.double().cpu().numpy(), r_ref, atol=1e-4 * max(1.0, np.abs(r_ref).max()))
    np.testing.assert_allclose(o.double().cpu().numpy(), o_ref, atol=5e-3 * max(1.0, np.abs(o_ref).max()))


@pytest.mark.gpu
def test_cube_lift_teacher_forced_lift_termination_and_truncation():
    import torch

    n = 8
    env, ref = _lift_pair(n, episode_steps=3)
    env.reset()
    ref.reset()
    ca = ref.cfg.cube_qposadr
    ref.qpos[0, ca + 2] = 0.2     # lifted cube (pays the lift and goal terms while it falls)
    ref.qpos[1, ca + 2] = -0.2    # cube below the table: terminates
    rng = np.random.default_rng(9)
    saw_term = saw_trunc = 0
    for k in range(5):
        _load(env, ref)
        a = rng.uniform(-1, 1, size=(n, env.model.nu))
        o, r, te, tr = env.step(torch.as_tensor(a, device="cuda"))
        o_ref, r_ref, te_ref, tr_ref = ref.step(a)
        torch.cuda.synchronize()
        np.testing.assert_array_equal(te.cpu().numpy().astype(bool), te_ref)
        np.testing.assert_array_equal(tr.cpu().numpy().astype(bool), tr_ref)
        np.testing.assert_allclose(r.cpu().numpy(), r_ref, rtol=1e-8, atol=1e-10)
        np.testing.assert_allclose(o.cpu().numpy(), o_ref, rtol=1e-7, atol=1e-7)
        np.testing.assert_allclose(env.command.cpu().numpy(), ref.cmd, atol=1e-15)
        saw_term += int(te_ref.sum())
        saw_trunc += int(tr_ref.sum())
    assert saw_term > 0 and saw_trunc > 0


@pytest.mark.gpu
def test_ppo_trains_on_the_3d_env():
    """The on-device PPO learner (flat-bucket gradient all-reduce) runs on the fused 3-D G1 task."""
    import torch

    from paper_2601_22074_b200.ppo import PpoCfg, PpoTrainer
    from paper_2601_22074_b200.sim3d.rl import ManagerView
    from paper_2601_22074_b200.sim3d.task import VelocityEnv3D

    m = robots.g1_like()
    cfg = VelocityTaskCfg(default_qpos=robots.default_qpos(m, robots.G1_DEFAULT_JOINTS))
    env = ManagerView(VelocityEnv3D(m, cfg, 256, seed=1, dtype="f32"))
    tr = PpoTrainer(env, PpoCfg(hidden=(64, 64), steps_per_env=8, epochs=2, minibatches=2))
    for _ in range(2):
        tr.collect()
        stats = tr.update()
    torch.cuda.synchronize()
    assert all(torch.isfinite(torch.as_tensor(float(v))) for v in stats.values())
    assert all(torch.isfinite(p).all() for p in tr.model.parameters())


@pytest.mark.gpu
@pytest.mark.parametrize("task", ["motion", "lift"])
def test_ppo_trains_on_the_motion_and_lift_tasks(task):
    """The on-device PPO learner on BASELINE configs[2] / [3] (BeyondMimic motion tracking, cube lift):
    rollouts through the fused kernel, finite losses and parameters after two updates."""
    import torch

    from paper_2601_22074_b200.ppo import PpoCfg, PpoTrainer
    from paper_2601_22074_b200.sim3d.rl import ManagerView

    env3, _ = (_motion_pair if task == "motion" else _lift_pair)(256, dtype="f32")
    tr = PpoTrainer(ManagerView(env3), PpoCfg(hidden=(64, 64), steps_per_env=8, epochs=2, minibatches=2))
    for _ in range(2):
        tr.collect()
        stats = tr.update()
    torch.cuda.synchronize()
    assert all(np.isfinite(float(v)) for v in stats.values())
    assert all(torch.isfinite(p).all() for p in tr.model.parameters())


@pytest.mark.gpu
@pytest.mark.parametrize("task", ["velocity", "motion"])
def test_domain_randomisation_events_match_oracle(task):
    """Startup friction and base-mass randomisation (per world) and interval pushes, on the velocity and the
    motion-imitation tasks: pushes every 1-3 control steps here, so the kicked base velocities, timers and
    both scales are all compared."""
    import torch

    n = 8
    kw = dict(push_interval=(0.02, 0.06), push_velocity=0.8)
    env, ref = _pair("g1_flat", n, **kw) if task == "velocity" else _motion_pair(n, max_height_error=10.0,
                                                                                 max_ori_error=10.0, **kw)
    np.testing.assert_allclose(env.reset().cpu().numpy(), ref.reset(), atol=1e-12)
    np.testing.assert_allclose(env.data.friction_scale.cpu().numpy(), ref.fscale, atol=1e-15)
    np.testing.assert_allclose(env.data.mass_scale.cpu().numpy(), ref.mscale, atol=1e-15)
    assert ref.fscale.std() > 0.01 and ref.mscale.std() > 0.01
    rng = np.random.default_rng(12)
    pushes = 0
    for k in range(5):
        _load(env, ref)
        before = ref.ev_timer.copy()
        a = rng.uniform(-1, 1, size=(n, env.model.nu))
        o, r, te, tr = env.step(torch.as_tensor(a, device="cuda"))
        o_ref, r_ref, te_ref, tr_ref = ref.step(a)
        torch.cuda.synchronize()
        pushes += int((ref.ev_timer > before).sum())
        np.testing.assert_array_equal(te.cpu().numpy().astype(bool), te_ref)
        np.testing.assert_allclose(r.cpu().numpy(), r_ref, rtol=1e-8, atol=1e-10)
        np.testing.assert_allclose(o.cpu().numpy(), o_ref, rtol=1e-7, atol=1e-7)
        np.testing.assert_allclose(env.event_timer.cpu().numpy(), ref.ev_timer, atol=1e-12)
        np.testing.assert_allclose(env.data.qvel.cpu().numpy(), ref.qvel, rtol=1e-8, atol=1e-8)
    assert pushes > 0


@pytest.mark.gpu
def test_terrain_curriculum_levels_match_oracle():
    """Terrain curriculum: spawn on the world's (level, column) patch, commanded-distance bookkeeping,
    promotion/demotion on finished episodes (short episodes and commands force both directions)."""
    import torch

    n = 12
    env, ref = _pair("g1_curriculum", n, episode_steps=2, command_ranges=((-0.05, 0.05), (-0.05, 0.05), (0, 0)),
                     curriculum_promote=0.5, curriculum_demote=0.2)
    np.testing.assert_allclose(env.reset().cpu().numpy(), ref.reset(), atol=1e-12)
    np.testing.assert_array_equal(env.terrain_level.cpu().numpy(), ref.level)
    np.testing.assert_allclose(env.spawn_xy.cpu().numpy(), ref.spawn, atol=1e-12)
    rng = np.random.default_rng(21)
    moved = 0
    for k in range(6):
        _load(env, ref)
        lv0 = ref.level.copy()
        a = rng.uniform(-1, 1, size=(n, env.model.nu))
        o, r, te, tr = env.step(torch.as_tensor(a, device="cuda"))
        o_ref, r_ref, te_ref, tr_ref = ref.step(a)
        torch.cuda.synchronize()
        moved += int((ref.level != lv0).sum())
        np.testing.assert_array_equal(env.terrain_level.cpu().numpy(), ref.level)
        np.testing.assert_allclose(env.spawn_xy.cpu().numpy(), ref.spawn, atol=1e-12)
        np.testing.assert_allclose(env.cmd_dist.cpu().numpy(), ref.cmd_dist, atol=1e-12)
        np.testing.assert_array_equal(te.cpu().numpy().astype(bool), te_ref)
        np.testing.assert_allclose(r.cpu().numpy(), r_ref, rtol=1e-8, atol=1e-10)
        np.testing.assert_allclose(o.cpu().numpy(), o_ref, rtol=1e-7, atol=1e-7)
    assert moved > 0


@pytest.mark.gpu
def test_metrics_record_one_allreduce():
    """Episode statistics of the 3-D env through metrics.pack_stats / unpack_stats (one collective)."""
    import torch

    env, ref = _pair("g1_curriculum", 8, episode_steps=2)
    env.reset()
    for _ in range(3):
        env.step(torch.rand(8, env.model.nu, dtype=torch.float64, device="cuda") * 2 - 1)
    rec = env.metrics_record(step=3)
    assert abs(rec.reward_mean - float(env.reward.mean())) < 1e-9  # the record rounds to 10 decimals
    assert sum(rec.terrain_row_histogram) == 8
    assert rec.termination_counts["terminated"] + rec.termination_counts["truncated"] >= 0


@pytest.mark.gpu
def test_models_on_two_streams_match_sequential():
    """Two different models (G1 float64, Go1 float32) stepped from two CUDA streams, interleaved without
    any user synchronization, give bit-identical results to stepping each alone on the default stream:
    the library serializes its constant-memory model slot across streams (s3_kernel.cu ModelSlot)."""
    import torch

    from paper_2601_22074_b200.sim3d.task import VelocityEnv3D

    def make(name, dtype):
        mk, table, kw = CASES[name]
        m = mk()
        return VelocityEnv3D(m, VelocityTaskCfg(default_qpos=robots.default_qpos(m, table), **kw), 256, seed=3,
                             dtype=dtype)

    steps = 6
    rng = np.random.default_rng(1)
    acts = {k: [torch.as_tensor(rng.uniform(-1, 1, size=(256, nu)), device="cuda") for _ in range(steps)]
            for k, nu in (("g1", make("g1_flat", "f64").model.nu), ("go1", make("go1_flat", "f32").model.nu))}
    solo = {}
    for key, name, dtype in (("g1", "g1_flat", "f64"), ("go1", "go1_flat", "f32")):
        env = make(name, dtype)
        env.reset()
        for a in acts[key]:
            env.step(a.to(env.dm.tdtype))
        torch.cuda.synchronize()
        solo[key] = (env.data.qpos.clone(), env.data.qvel.clone())
    e1, e2 = make("g1_flat", "f64"), make("go1_flat", "f32")
    torch.cuda.synchronize()  # construction ran on the default stream
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    with torch.cuda.stream(s1):
        e1.reset()
    with torch.cuda.stream(s2):
        e2.reset()
    for i in range(steps):
        with torch.cuda.stream(s1):
            e1.step(acts["g1"][i].to(e1.dm.tdtype))
        with torch.cuda.stream(s2):
            e2.step(acts["go1"][i].to(e2.dm.tdtype))
    torch.cuda.synchronize()
    assert torch.equal(e1.data.qpos, solo["g1"][0]) and torch.equal(e1.data.qvel, solo["g1"][1])
    assert torch.equal(e2.data.qpos, solo["go1"][0]) and torch.equal(e2.data.qvel, solo["go1"][1])
