"""Drop-in API behaviour on the GPU, modelled on the reference's own tests
(tests/test_env.py, test_managers.py, test_physics.py, test_sensors.py,
test_actuators.py of stridesim), run through the CUDA path."""

import numpy as np
import pytest

from helpers import pendulum_spec, two_leg_spec

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def _np(t):
    return t.detach().cpu().numpy() if hasattr(t, "detach") else np.asarray(t)


def quiet_cfg(n=4, **kw):
    from paper_2601_22074_b200.config import NoiseCfg
    from paper_2601_22074_b200.tasks import make_env_cfg

    cfg = make_env_cfg("Velocity-Flat", num_envs=n, **kw)
    cfg.events = {}
    cfg.curriculum = {}
    for g in cfg.observations.values():
        for t in g.terms.values():
            t.noise = NoiseCfg()
    return cfg


def quiet_env(n=4, **kw):
    from paper_2601_22074_b200.env import ManagerBasedRlEnv

    env = ManagerBasedRlEnv(quiet_cfg(n, **kw))
    env.reset()
    return env


def zeros(env):
    return torch.zeros((env.num_envs, env.action_manager.total_dim), dtype=torch.float64, device="cuda")


# ---------------------------------------------------------------------------
# physics (tests/test_physics.py of the reference)


def test_fk_matches_rotation_matrix_oracle(rng):
    from paper_2601_22074_b200.sim import compile_model, forward_kinematics

    spec = two_leg_spec()
    model = compile_model(spec, 1)

    def rotm(a):
        return np.array([[np.cos(a), -np.sin(a)], [np.sin(a), np.cos(a)]])

    for _ in range(10):
        q = rng.uniform(-2.0, 2.0, size=model.nq)
        frames, tips = {}, []
        for j, js in enumerate(spec.joints):
            if js.parent == -1:
                origin, angle = q[:2] + rotm(q[2]) @ np.array(js.attach_offset), q[2] + q[3 + j]
            else:
                po, pa = frames[js.parent]
                origin, angle = po + rotm(pa) @ np.array(js.attach_offset), pa + q[3 + j]
            frames[j] = (origin, angle)
            tips.append(origin + js.link_length * (rotm(angle) @ np.array([0.0, -1.0])))
        _, got = forward_kinematics(model, q)
        assert np.allclose(got, np.array(tips), atol=1e-12)


def test_free_fall_matches_scalar_recurrence():
    from paper_2601_22074_b200.sim import BatchState, StepPipeline, compile_model

    spec = pendulum_spec()
    model = compile_model(spec, 3)
    st = BatchState(model)
    st.q[:, 1] = 10.0
    pipe = StepPipeline(model, None)
    dt = spec.physics_dt
    m_total = spec.base_mass + spec.joints[0].link_mass
    inv = 1.0 / m_total
    z, vz = 10.0, 0.0
    for n in range(1, 101):
        pipe.substep(st)
        a = (0.0 - m_total * spec.gravity) * inv
        vz = vz + a * dt
        z = z + vz * dt
        assert float(st.qd[0, 1]) == vz
        assert float(st.q[0, 1]) == z


def test_static_equilibrium_penetration():
    from paper_2601_22074_b200.sim import BatchState, StepPipeline, compile_model

    spec = pendulum_spec()
    model = compile_model(spec, 1)
    st = BatchState(model)
    st.q[0, 1] = 0.5
    pipe = StepPipeline(model, None)
    for _ in range(int(2.0 / spec.physics_dt)):
        pipe.substep(st)
    phi_expect = (spec.base_mass + 0.5) * spec.gravity / spec.contact_stiffness
    phi = 0.0 - (float(st.q[0, 1]) - 0.5)
    assert abs(phi - phi_expect) / phi_expect < 0.01
    assert abs(float(st.qd[0, 1])) < 1e-6


def test_batched_step_equals_solo_step_bitwise(rng):
    from paper_2601_22074_b200.sim import BatchState, compile_model, physics_step

    spec = two_leg_spec()
    bm = compile_model(spec, 4)
    b = BatchState(bm)
    b.q = rng.uniform(-0.5, 0.8, size=(4, bm.nq))
    b.qd = rng.uniform(-1.0, 1.0, size=(4, bm.nq))
    b.ctrl = rng.uniform(-2.0, 2.0, size=(4, bm.num_joints))
    solos = []
    for w in range(4):
        sm = compile_model(spec, 1)
        s = BatchState(sm)
        s.q = _np(b.q[w : w + 1])
        s.qd = _np(b.qd[w : w + 1])
        s.ctrl = _np(b.ctrl[w : w + 1])
        for _ in range(50):
            physics_step(sm, s)
        solos.append(s)
    for _ in range(50):
        physics_step(bm, b)
    for w in range(4):
        assert np.array_equal(_np(b.q[w]), _np(solos[w].q[0]))
        assert np.array_equal(_np(b.qd[w]), _np(solos[w].qd[0]))


def test_contact_complementarity_over_rollout(rng):
    from paper_2601_22074_b200.sim import BatchState, StepPipeline, compile_model

    spec = two_leg_spec()
    model = compile_model(spec, 64)
    st = BatchState(model)
    st.q[:, 1] = torch.as_tensor(rng.uniform(0.3, 0.8, size=64), device="cuda")
    st.q[:, 3:] = torch.as_tensor(rng.uniform(-0.4, 0.4, size=(64, 4)), device="cuda")
    pipe = StepPipeline(model, None)
    for _ in range(200):
        pipe.substep(st)
        fn, ft, inc = _np(st.contact.normal_force), _np(st.contact.tangent_force), _np(st.contact.in_contact)
        assert (fn >= 0.0).all()
        assert (fn[~inc] == 0.0).all()
        assert (np.abs(ft) <= spec.friction * fn + 1e-12).all()


def test_ext_force_consumed_by_one_substep():
    from paper_2601_22074_b200.sim import BatchState, compile_model, physics_step

    spec = pendulum_spec()
    model = compile_model(spec, 1)
    a, b = BatchState(model), BatchState(model)
    a.q[0, 1] = 5.0
    b.q[0, 1] = 5.0
    a.ext_force[0, 0] = 40.0
    physics_step(model, a)
    physics_step(model, b)
    assert abs(float(a.qd[0, 0] - b.qd[0, 0]) - 40.0 * spec.physics_dt / 8.5) < 1e-12
    assert float(a.ext_force.abs().max()) == 0.0


def test_field_expansion_preserves_trajectories_bitwise():
    from paper_2601_22074_b200.sim import BatchState, StepPipeline, compile_model

    init = np.random.default_rng(5).uniform(-0.5, 0.5, size=(3, 7))

    def rollout(expand_at):
        model = compile_model(two_leg_spec(), 3)
        st = BatchState(model)
        st.q[:, 1] = 0.48
        st.qd = init
        pipe = StepPipeline(model, None)
        for i in range(60):
            if i == expand_at:
                assert model.expand_field("friction") == 1
            pipe.substep(st)
        return _np(st.q), _np(st.qd)

    a, b = rollout(-1), rollout(30)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])


def test_nan_propagates_and_is_flagged():
    from paper_2601_22074_b200.sim import BatchState, compile_model, detect_nonfinite, physics_step

    model = compile_model(pendulum_spec(), 2)
    st = BatchState(model)
    st.q[:, 1] = 0.4
    st.q[1, 0] = float("nan")
    physics_step(model, st)
    assert _np(detect_nonfinite(st)).tolist() == [False, True]


# ---------------------------------------------------------------------------
# env (tests/test_env.py of the reference)


def test_reset_same_seed_identical_observations():
    from paper_2601_22074_b200.env import ManagerBasedRlEnv
    from paper_2601_22074_b200.tasks import make_env_cfg

    env = ManagerBasedRlEnv(make_env_cfg("Velocity-Flat", num_envs=4))
    a = {k: _np(v).copy() for k, v in env.reset(seed=11).items()}
    b = {k: _np(v).copy() for k, v in env.reset(seed=11).items()}
    for g in a:
        assert np.array_equal(a[g], b[g])
    c = {k: _np(v).copy() for k, v in env.reset(seed=12).items()}
    assert not np.array_equal(a["policy"], c["policy"])


def test_control_arithmetic():
    env = quiet_env(2)
    assert env.dt_control == 0.02 and env.decimation == 4
    before = env.state.sim_step
    env.step(zeros(env))
    assert env.state.sim_step == before + 4


def test_stage_order_reward_pre_reset_obs_post_reset():
    from paper_2601_22074_b200.config import ObsGroupCfg, ObsTermCfg, RewardTermCfg
    from paper_2601_22074_b200.env import ManagerBasedRlEnv

    cfg = quiet_cfg(3)
    cfg.rewards = {"sentinel": RewardTermCfg(func="base_height", weight=1.0)}
    cfg.observations = {"g": ObsGroupCfg(terms={"h": ObsTermCfg(func="base_height")})}
    env = ManagerBasedRlEnv(cfg)
    env.reset()
    env.state.q[1, 1] = 2.0
    env.state.q[1, 2] = 1.5
    env.state.qd[1, :] = 0.0
    obs, rew, term, trunc, _ = env.step(zeros(env))
    assert bool(term[1]) and not bool(term[0])
    assert float(rew[1]) > 1.5 * env.dt_control
    assert abs(float(obs["g"][1, 0]) - 0.48) < 1e-9


def test_world_reset_restores_default_state():
    env = quiet_env(3)
    env.state.q[2, 2] = 1.4
    env.step(zeros(env))
    assert abs(float(env.state.q[2, 2])) < 1e-12
    assert np.allclose(_np(env.state.q[2, 3:]), env.default_joint_pos)
    assert int(env.episode_steps[2]) == 0


def test_truncation_at_exact_step_count():
    cfg = quiet_cfg(2)
    cfg.episode_length_s = 0.2
    from paper_2601_22074_b200.env import ManagerBasedRlEnv

    env = ManagerBasedRlEnv(cfg)
    env.reset()
    for i in range(9):
        _, _, term, trunc, _ = env.step(zeros(env))
        assert not bool(trunc.any()), i
    _, _, term, trunc, _ = env.step(zeros(env))
    assert bool(trunc.all()) and not bool(term.any())


def test_zero_action_smoke_no_nonfinite():
    from paper_2601_22074_b200.env import ManagerBasedRlEnv
    from paper_2601_22074_b200.tasks import make_env_cfg

    env = ManagerBasedRlEnv(make_env_cfg("Velocity-Flat", num_envs=8, seed=0))
    env.reset()
    for _ in range(300):
        _, _, _, _, extras = env.step(zeros(env))
    assert not bool(extras["nonfinite_worlds"].any())
    assert not env.dump_paths


def test_extras_keys():
    env = quiet_env(2)
    _, _, _, _, x = env.step(zeros(env))
    keys = set(x)
    assert "reset_ids" in keys and "nonfinite_worlds" in keys and "curriculum/terrain_rows" in keys
    assert any(k.startswith("reward/") for k in keys) and any(k.startswith("termination_count/") for k in keys)


def test_capture_dump_load_round_trip_and_replay_bit_exact(tmp_path):
    from paper_2601_22074_b200.capture import load_capture

    env = quiet_env(2)
    for _ in range(6):
        env.step(zeros(env))
    path = str(tmp_path / "dump.bin")
    env.dump_capture(path)
    dump = load_capture(path)
    assert dump.n_worlds == 2 and dump.config_hash == env.config_hash
    assert len(dump.frames) == min(env.cfg.capture_len, env.state.sim_step)
    steps = [f.sim_step for f in dump.frames]
    assert steps == sorted(steps) and len(set(steps)) == len(steps)
    for mine, theirs in zip(env.capture.frames(), dump.frames):
        assert np.array_equal(mine.q, theirs.q) and mine.sim_step == theirs.sim_step
    k = 9
    env.restore(dump.frames[k])
    env.pipeline.substep(env.state)
    assert np.array_equal(_np(env.state.q), dump.frames[k + 1].q)
    assert np.array_equal(_np(env.state.qd), dump.frames[k + 1].qd)


def test_nan_terminates_and_dumps(tmp_path):
    from paper_2601_22074_b200.capture import load_capture
    from paper_2601_22074_b200.env import ManagerBasedRlEnv

    cfg = quiet_cfg(3)
    cfg.capture_len = 10
    cfg.capture_dir = str(tmp_path)
    env = ManagerBasedRlEnv(cfg)
    env.reset()
    for _ in range(3):
        env.step(zeros(env))
    env.state.q[2, 1] = float("nan")
    _, _, term, _, extras = env.step(zeros(env))
    assert _np(term).tolist() == [False, False, True]
    assert _np(extras["nonfinite_worlds"]).tolist() == [False, False, True]
    assert len(env.dump_paths) == 1
    dump = load_capture(env.dump_paths[0])
    assert len(dump.frames) == min(10, env.state.sim_step)
    assert dump.metadata["nonfinite_worlds"] == [2]
    assert any(h["array"] == "q" and h["world"] == 2 for h in dump.nonfinite_summary())
    # a few more steps: no further dumps (the world was reset)
    for _ in range(5):
        env.step(zeros(env))
    assert len(env.dump_paths) == 1


def test_world_runs_identically_alone():
    from paper_2601_22074_b200.env import ManagerBasedRlEnv
    from paper_2601_22074_b200.tasks import make_env_cfg

    batch = ManagerBasedRlEnv(make_env_cfg("Velocity-Rough", num_envs=4, seed=9))
    batch.reset()
    hist = []
    for _ in range(60):
        batch.step(zeros(batch))
        hist.append(_np(batch.state.q[2]).copy())
    cfg = make_env_cfg("Velocity-Rough", num_envs=1, seed=9)
    cfg.scene.world_id_offset = 2
    solo = ManagerBasedRlEnv(cfg)
    solo.reset()
    for i in range(60):
        solo.step(zeros(solo))
        assert np.array_equal(_np(solo.state.q[0]), hist[i]), f"diverged at step {i}"


def test_two_envs_same_config_step_identically():
    from paper_2601_22074_b200.env import ManagerBasedRlEnv
    from paper_2601_22074_b200.tasks import make_env_cfg

    a = ManagerBasedRlEnv(make_env_cfg("Velocity-Flat", num_envs=4, seed=7))
    b = ManagerBasedRlEnv(make_env_cfg("Velocity-Flat", num_envs=4, seed=7))
    a.reset()
    b.reset()
    for i in range(40):
        act = torch.full((4, 4), float(np.sin(i * 0.3)), dtype=torch.float64, device="cuda")
        oa, ra, ta, _, _ = a.step(act)
        ob, rb, tb, _, _ = b.step(act)
        assert torch.equal(oa["policy"], ob["policy"]) and torch.equal(ra, rb) and torch.equal(ta, tb)


# ---------------------------------------------------------------------------
# managers (tests/test_managers.py of the reference)


def test_action_dim_mismatch_reports_expected():
    from paper_2601_22074_b200.managers import ManagerError

    env = quiet_env()
    with pytest.raises(ManagerError, match="does not match expected"):
        env.step(torch.zeros((4, 5), dtype=torch.float64, device="cuda"))


def pd_torque(kp, kd, effort_limit, q_des, qd_des, q, qd):
    """numpy restatement of actuators.py:104-107 (the expected values)."""
    return np.clip(kp * (q_des - q) + kd * (qd_des - qd), -effort_limit, effort_limit)


def test_action_clip_history_and_pd_apply():
    env = quiet_env()
    am = env.action_manager
    am.process(np.full((4, 4), 0.1))
    am.process(np.full((4, 4), 10.0))
    assert np.allclose(_np(am.prev_action), 0.1) and np.allclose(_np(am.action), 10.0)
    term = am.terms["joint_targets"]
    assert np.allclose(_np(am.targets[:, term.joint_ids]), term.offset + 0.5 * 2.0)
    actions = np.linspace(-1, 1, 16).reshape(4, 4)
    am.process(actions)
    am.apply()
    q_des = term.offset + 0.5 * np.clip(actions, -2, 2)
    want = pd_torque(40.0, 2.0, 30.0, q_des, 0.0, _np(env.state.q[:, 3:]), _np(env.state.qd[:, 3:]))
    assert np.allclose(_np(env.state.ctrl), want, atol=1e-13)


def test_delayed_actuator_first_substep_uses_reset_fill():
    from paper_2601_22074_b200.config import DelayedCfg, IdealPdCfg
    from paper_2601_22074_b200.env import ManagerBasedRlEnv

    cfg = quiet_cfg(2)
    cfg.actions["joint_targets"].actuators = {
        "legs": DelayedCfg(inner=IdealPdCfg(kp=40.0, kd=2.0, effort_limit=30.0), latency_range=(0.005, 0.005),
                           resample_on_reset=False)}
    env = ManagerBasedRlEnv(cfg)
    env.reset()
    am = env.action_manager
    term = am.terms["joint_targets"]
    am.process(np.full((2, 4), 1.0))
    am.apply()
    want = pd_torque(40.0, 2.0, 30.0, term.offset, 0.0, _np(env.state.q[:, 3:]), _np(env.state.qd[:, 3:]))
    assert np.allclose(_np(env.state.ctrl), want, atol=1e-13)
    am.apply()
    want2 = pd_torque(40.0, 2.0, 30.0, term.offset + 0.5, 0.0, _np(env.state.q[:, 3:]), _np(env.state.qd[:, 3:]))
    assert np.allclose(_np(env.state.ctrl), want2, atol=1e-13)


def test_reward_formula_and_dt_scaling():
    from paper_2601_22074_b200.config import RewardTermCfg
    from paper_2601_22074_b200.env import ManagerBasedRlEnv

    def rew(decimation, weight):
        cfg = quiet_cfg(2)
        cfg.decimation = decimation
        cfg.rewards = {"flat": RewardTermCfg(func="constant", weight=weight, params={"value": 1.0})}
        env = ManagerBasedRlEnv(cfg)
        env.reset()
        _, r, _, _, _ = env.step(zeros(env))
        return _np(r).copy(), env

    r4, env = rew(4, 2.0)
    assert np.all(r4 == 2.0 * 1.0 * 0.02)
    assert rew(2, 1.0)[0][0] == rew(4, 1.0)[0][0] / 2.0
    for _ in range(4):
        env.step(zeros(env))
    assert np.allclose(_np(env.reward_manager.episodic_sums["flat"]), 5 * 2.0 * 0.02)
    env.reset()
    assert float(env.reward_manager.episodic_sums["flat"].abs().max()) == 0.0


def test_custom_python_terms_run_in_staged_mode():
    """User-registered terms (the plugin boundary, managers/base.py:36-70)."""
    from paper_2601_22074_b200.config import ObsTermCfg, RewardTermCfg, TerminationTermCfg
    from paper_2601_22074_b200.env import ManagerBasedRlEnv
    from paper_2601_22074_b200.managers import observation_term, reward_term, termination_term

    @reward_term("test_nan_reward_gpu")
    def _nan_reward(env):
        out = np.zeros(env.num_envs)
        out[1] = np.nan
        return out

    @observation_term("test_inf_obs_gpu")
    def _inf_obs(env):
        out = np.ones((env.num_envs, 2))
        out[0, 1] = np.inf
        return out

    @termination_term("test_kill_world0")
    def _kill(env):
        m = torch.zeros(env.num_envs, dtype=torch.bool, device=env.device)
        m[0] = env.global_step % 3 == 0
        return m

    cfg = quiet_cfg(3)
    cfg.rewards["bad"] = RewardTermCfg(func="test_nan_reward_gpu", weight=1.0)
    cfg.observations["policy"].terms["bad"] = ObsTermCfg(func="test_inf_obs_gpu")
    cfg.terminations["kill"] = TerminationTermCfg(func="test_kill_world0")
    env = ManagerBasedRlEnv(cfg)
    assert env.staged
    env.reset()
    for i in range(1, 7):
        obs, rew, term, trunc, x = env.step(zeros(env))
        assert bool(term[0]) == (i % 3 == 0)
    assert set(env.reward_manager.nonfinite_report) == {"bad"}
    assert _np(env.reward_manager.nonfinite_report["bad"]).tolist() == [False, True, False]
    rep = env.observation_manager.nonfinite_report
    assert set(rep) == {"bad"} and _np(rep["bad"]).tolist() == [True, False, False]
    assert env.termination_manager.trigger_counts["kill"] == 2


def test_interval_event_gaps_stay_in_range():
    from paper_2601_22074_b200.config import EventTermCfg
    from paper_2601_22074_b200.env import ManagerBasedRlEnv
    from paper_2601_22074_b200.managers.base import event_term

    fires = {0: [], 1: []}

    @event_term("test_fire_logger_gpu")
    def _log(env, ids):
        for w in _np(ids):
            fires[int(w)].append(env.global_step)

    cfg = quiet_cfg(2)
    cfg.episode_length_s = 1000.0
    cfg.terminations = {k: v for k, v in cfg.terminations.items() if k == "time_out"}
    cfg.events = {"tick": EventTermCfg(func="test_fire_logger_gpu", mode="interval", interval_range=(0.1, 0.2))}
    env = ManagerBasedRlEnv(cfg)
    env.reset()
    for _ in range(400):
        env.step(zeros(env))
    for w, steps in fires.items():
        assert len(steps) >= 30
        gaps = np.diff(steps) * env.dt_control
        assert gaps.min() >= 0.1 - 1e-9 and gaps.max() <= 0.2 + 1e-9


def test_startup_event_expands_field_and_draws_in_range():
    from paper_2601_22074_b200.env import ManagerBasedRlEnv
    from paper_2601_22074_b200.tasks import make_env_cfg

    env = ManagerBasedRlEnv(make_env_cfg("Velocity-Flat", num_envs=8))
    assert env.model.generation == 0
    env.reset()
    f = env.model.field("base_mass")
    assert f.expanded and env.model.generation == 1
    v = _np(f.value)
    assert np.all(v >= 0.8 * 8.0) and np.all(v <= 1.2 * 8.0) and len(np.unique(v)) > 1


def test_randomize_field_set_scale_add():
    from paper_2601_22074_b200.managers.event import randomize_field

    env = quiet_env(4)
    ids = np.array([0, 1])
    randomize_field(env.model, env.streams, "friction", "uniform", (2.0, 2.0), "set", ids, "t")
    v = _np(env.model.field("friction").value)
    assert v[:2].tolist() == [2.0, 2.0] and v[2] == 1.0
    randomize_field(env.model, env.streams, "friction", "uniform", (0.5, 0.5), "scale", ids, "t")
    assert float(env.model.field("friction").value[0]) == 0.5
    randomize_field(env.model, env.streams, "friction", "uniform", (0.25, 0.25), "add", ids, "t")
    assert float(env.model.field("friction").value[0]) == 1.25


def test_command_widen_caps_and_is_per_world():
    env = quiet_env(16)
    cm = env.command_manager
    cm.widen(np.array([1]), 2.0)
    assert float(cm.ranges[1, 0, 1]) == 2.0 and float(cm.ranges[0, 0, 1]) == 1.0
    ids = np.arange(16)
    for _ in range(10):
        cm.widen(ids, 1.5)
    assert np.all(_np(cm.ranges[:, 0, 1]) == 2.0)
    seen = False
    for _ in range(30):
        cm.resample(ids)
        seen |= bool((cm.command[:, 0].abs() > 1.0).any())
    assert seen


def test_terrain_levels_promote_and_demote():
    from paper_2601_22074_b200.config import CurriculumTermCfg
    from paper_2601_22074_b200.env import ManagerBasedRlEnv
    from paper_2601_22074_b200.tasks import make_env_cfg

    cfg = quiet_cfg(2, seed=3)
    cfg.scene.terrain = make_env_cfg("Velocity-Rough").scene.terrain
    cfg.curriculum = {"terrain_levels": CurriculumTermCfg(func="terrain_levels")}
    env = ManagerBasedRlEnv(cfg)
    env.reset()
    env.terrain_rows[:] = 2
    env.episode_start_x[:] = env.state.q[:, 0]
    env.commanded_distance[:] = 5.0
    env.state.q[0, 0] += 4.5
    env.state.q[1, 0] += 1.0
    env.curriculum_manager.update(np.array([0, 1]))
    assert _np(env.terrain_rows).tolist() == [3, 1]


def test_reward_weight_schedule_linear_midpoint():
    from paper_2601_22074_b200.config import CurriculumTermCfg
    from paper_2601_22074_b200.env import ManagerBasedRlEnv

    cfg = quiet_cfg(2)
    cfg.curriculum = {"fade": CurriculumTermCfg(func="reward_weight_schedule",
                                                params={"term": "track_vx_exp", "start_weight": 1.0,
                                                        "end_weight": 0.0, "start_step": 0, "end_step": 1000})}
    env = ManagerBasedRlEnv(cfg)
    env.reset()
    env.global_step = 500
    env.curriculum_manager.update(np.array([], dtype=np.int64))
    assert env.reward_manager.weights["track_vx_exp"] == 0.5


def test_obs_delay_exact_and_history_oldest_first():
    from paper_2601_22074_b200.config import ObsGroupCfg, ObsTermCfg
    from paper_2601_22074_b200.env import ManagerBasedRlEnv

    cfg = quiet_cfg(2)
    cfg.episode_length_s = 1000.0
    cfg.observations = {"d": ObsGroupCfg(terms={"t": ObsTermCfg(func="sim_time", delay_steps=3)}),
                        "h": ObsGroupCfg(terms={"t": ObsTermCfg(func="sim_time", history=4)})}
    env = ManagerBasedRlEnv(cfg)
    env.reset()
    raws, outs, hist = [0.0], [], None
    for _ in range(10):
        obs, *_ = env.step(zeros(env))
        raws.append(float(env.state.time[0]))
        outs.append(float(obs["d"][0, 0]))
        hist = _np(obs["h"][0]).tolist()
    for t, out in enumerate(outs, start=1):
        assert out == (raws[t - 3] if t >= 3 else raws[0])
    assert hist == raws[-4:]


def test_obs_group_dims_and_unknown_group():
    from paper_2601_22074_b200.managers import ManagerError

    env = quiet_env()
    om = env.observation_manager
    assert om.group_dim("policy") == 2 + 1 + 2 + 4 + 4 + 4 + 2
    with pytest.raises(ManagerError, match="unknown observation group"):
        om.compute("nope")


def test_obs_noise_respects_group_flag():
    from paper_2601_22074_b200.config import NoiseCfg, ObsGroupCfg, ObsTermCfg
    from paper_2601_22074_b200.env import ManagerBasedRlEnv

    cfg = quiet_cfg(4)
    cfg.observations = {
        "noisy": ObsGroupCfg(terms={"h": ObsTermCfg(func="base_height", noise=NoiseCfg("uniform", 0.1))}),
        "clean": ObsGroupCfg(terms={"h": ObsTermCfg(func="base_height", noise=NoiseCfg("uniform", 0.1))},
                             enable_noise=False),
    }
    env = ManagerBasedRlEnv(cfg)
    obs = env.reset()
    z = _np(env.state.q[:, 1])
    assert np.array_equal(_np(obs["clean"][:, 0]), z)
    assert not np.array_equal(_np(obs["noisy"][:, 0]), z)
    assert np.allclose(_np(obs["noisy"][:, 0]), z, atol=0.1 + 1e-12)


# ---------------------------------------------------------------------------
# sensors + actuators


def test_contact_sensor_update_once_per_sim_step_and_history_newest_first():
    from paper_2601_22074_b200.config import ContactSensorCfg
    from paper_2601_22074_b200.sensors import ContactSensor
    from paper_2601_22074_b200.sim import BatchState, compile_model

    model = compile_model(two_leg_spec(), 2)
    st = BatchState(model)
    sensor = ContactSensor(ContactSensorCfg(history_length=3), 2, 2)
    for k in range(1, 5):
        st.contact.normal_force[:] = float(k)
        st.contact.in_contact[:] = k % 2 == 0
        st.sim_step = k
        sensor.update(st, 0.005)
        sensor.update(st, 0.005)  # second call in the same sim_step is a no-op
    assert _np(sensor.force_history[:, 0, 0]).tolist() == [4.0, 3.0, 2.0]
    assert _np(sensor.last_touchdown_step[0]).tolist() == [4, 4]


def test_dc_motor_envelope_on_device(rng):
    from paper_2601_22074_b200.actuators import dc_motor_torque

    kp, kd, eff, sat, vl = 40.0, 1.0, 30.0, 45.0, 20.0
    q_des, q, qd = rng.uniform(-2, 2, 50), rng.uniform(-2, 2, 50), rng.uniform(-30, 30, 50)
    tau = kp * (q_des - q) + kd * (0.0 - qd)  # numpy restatement of actuators.py:110-117
    hi = np.clip(sat * (1.0 - qd / vl), 0.0, eff)
    lo = np.clip(sat * (-1.0 - qd / vl), -eff, 0.0)
    host = np.clip(tau, lo, hi)
    assert np.array_equal(host, _np(dc_motor_torque(kp, kd, eff, sat, vl, q_des, 0.0, q, qd)))  # host inputs
    dev = dc_motor_torque(torch.full((50,), kp, device="cuda", dtype=torch.float64), kd, eff, sat, vl,
                          torch.as_tensor(q_des, device="cuda"), 0.0, torch.as_tensor(q, device="cuda"),
                          torch.as_tensor(qd, device="cuda"))
    assert np.array_equal(host, _np(dev))


@pytest.mark.parametrize("task,n", [("Velocity-Rough", 300), ("Velocity-Flat", 300), ("Velocity-Rough", 2048),
                                    ("Velocity-Flat-Quad12", 300), ("Velocity-Rough-Humanoid10", 1100)])
def test_jit_specialization_bitwise_equals_generic_kernel(task, n):
    """The per-env NVRTC specialization and the generic AOT kernel run the same
    source; they must agree bit for bit (no reassociation, --fmad=false)."""
    from paper_2601_22074_b200 import jit
    from paper_2601_22074_b200.env import ManagerBasedRlEnv
    from paper_2601_22074_b200.policies import random_policy
    from paper_2601_22074_b200.tasks import make_env_cfg

    a = ManagerBasedRlEnv(make_env_cfg(task, num_envs=n, seed=4))
    b = ManagerBasedRlEnv(make_env_cfg(task, num_envs=n, seed=4))
    assert a.use_jit
    b.use_jit = False
    oa, ob = a.reset(), b.reset()
    for i in range(40):
        act = random_policy(a, i)
        random_policy(b, i)
        oa, ra, ta, _, _ = a.step(act)
        ob, rb, tb, _, _ = b.step(act)
        for k in oa:
            assert torch.equal(oa[k], ob[k]), (i, k)
        assert torch.equal(ra, rb) and torch.equal(ta, tb)
        assert torch.equal(a.state.q, b.state.q)
    assert jit.STATS["compiled"] + jit.STATS["disk_hits"] + jit.STATS["memory_hits"] > 0


def test_step_outputs_arena_holds_every_result():
    """One contiguous block (obs groups, reward, dones) for a single D2H copy."""
    from paper_2601_22074_b200.env import ManagerBasedRlEnv
    from paper_2601_22074_b200.policies import random_policy
    from paper_2601_22074_b200.tasks import make_env_cfg

    env = ManagerBasedRlEnv(make_env_cfg("Velocity-Rough", num_envs=64, seed=2))
    env.reset()
    obs, rew, term, trunc, _ = env.step(random_policy(env, 0))
    host = env.unpack_outputs(env.step_outputs.cpu())
    for g in obs:
        assert torch.equal(host[f"obs/{g}"], obs[g].cpu())
    assert torch.equal(host["reward"], rew.cpu())
    assert torch.equal(host["terminated"], term.cpu()) and torch.equal(host["truncated"], trunc.cpu())


def test_ppo_trainer_runs_on_device():
    from paper_2601_22074_b200.env import ManagerBasedRlEnv
    from paper_2601_22074_b200.ppo import PpoCfg, PpoTrainer
    from paper_2601_22074_b200.tasks import make_env_cfg

    env = ManagerBasedRlEnv(make_env_cfg("Velocity-Flat", num_envs=256, seed=1))
    tr = PpoTrainer(env, PpoCfg(hidden=(64, 64), steps_per_env=8, epochs=2, minibatches=2))
    for _ in range(3):
        tr.collect()
        st = tr.update()
    assert st["allreduces"] == 4 and np.isfinite(st["loss"])
    assert tr.buf["obs_p"].is_cuda and tr.reducer.numel > 0


@pytest.mark.parametrize("mode", ["jit", "generic", "staged"])
def test_fused_random_policy_equals_separate_draw(mode):
    """env.step(RandomActions()) draws policy.random inside the step kernel:
    actions, stream counters and every output equal the two-launch form
    env.step(random_policy(env)) bit for bit (policies.py:14-16)."""
    from paper_2601_22074_b200.config import RewardTermCfg
    from paper_2601_22074_b200.env import ManagerBasedRlEnv
    from paper_2601_22074_b200.managers import reward_term
    from paper_2601_22074_b200.policies import random_policy
    from paper_2601_22074_b200.tasks import make_env_cfg

    @reward_term("test_host_const_reward")
    def _const(env):
        return np.full(env.num_envs, 0.5)

    def make():
        cfg = make_env_cfg("Velocity-Rough", num_envs=257, seed=11)
        if mode == "staged":
            cfg.rewards["host"] = RewardTermCfg(func="test_host_const_reward", weight=1.0)
        e = ManagerBasedRlEnv(cfg)
        if mode == "generic":
            e.use_jit = False
        return e

    a, b = make(), make()
    assert a.staged == (mode == "staged")
    a.reset()
    b.reset()
    for i in range(30):
        oa, ra, ta, xa, _ = a.step(random_policy(a, i))
        ob, rb, tb, xb, _ = b.step(random_policy(b, i, fused=True))
        assert torch.equal(a.action_manager.action, b.action_manager.action), i
        for k in oa:
            assert torch.equal(oa[k], ob[k]), (i, k)
        assert torch.equal(ra, rb) and torch.equal(ta, tb) and torch.equal(xa, xb)
    assert torch.equal(a.streams.counter("policy.random"), b.streams.counter("policy.random"))
    assert torch.equal(a.state.q, b.state.q) and torch.equal(a.state.qd, b.state.qd)


@pytest.mark.parametrize("generic", [False, True])
def test_host_io_zero_copy_equals_device_path(generic):
    """Pinned host actions read in place by the kernel and outputs mirrored
    into pinned host memory by the kernel (enable_host_outputs) give the same
    bits as device actions + device outputs."""
    from paper_2601_22074_b200.env import ManagerBasedRlEnv
    from paper_2601_22074_b200.tasks import make_env_cfg

    a = ManagerBasedRlEnv(make_env_cfg("Velocity-Rough", num_envs=300, seed=5))
    b = ManagerBasedRlEnv(make_env_cfg("Velocity-Rough", num_envs=300, seed=5))
    if generic:
        a.use_jit = b.use_jit = False
    host = b.enable_host_outputs()
    a.reset()
    b.reset()
    rng = np.random.default_rng(3)
    pinned = torch.empty((300, a.action_manager.total_dim), dtype=torch.float64).pin_memory()
    for i in range(25):
        pinned.copy_(torch.from_numpy(rng.uniform(-1, 1, size=tuple(pinned.shape))))
        oa, ra, ta, xa, _ = a.step(pinned.cuda())
        b.step(pinned)
        torch.cuda.synchronize()
        for g in oa:
            assert torch.equal(oa[g].cpu(), host[f"obs/{g}"]), (i, g)
        assert torch.equal(ra.cpu(), host["reward"]) and torch.equal(ta.cpu(), host["terminated"])
        assert torch.equal(xa.cpu(), host["truncated"])
    assert torch.equal(a.state.q, b.state.q)
    assert torch.equal(a.step_outputs, b.step_outputs)


@pytest.mark.gpu
def test_step_async_delivers_each_steps_results_to_host():
    """Pipelined host I/O (step_async / step_wait: D2D snapshot + copy-engine D2H overlapping the
    next step) returns, for every step, the same bits as a synchronous step."""
    from paper_2601_22074_b200.env import ManagerBasedRlEnv
    from paper_2601_22074_b200.tasks import make_env_cfg

    a = ManagerBasedRlEnv(make_env_cfg("Velocity-Rough", num_envs=300, seed=6))
    b = ManagerBasedRlEnv(make_env_cfg("Velocity-Rough", num_envs=300, seed=6))
    a.reset()
    b.reset()
    rng = np.random.default_rng(4)
    acts = [torch.from_numpy(rng.uniform(-1, 1, size=(300, a.action_manager.total_dim))).pin_memory()
            for _ in range(12)]
    expected = []
    for i, x in enumerate(acts):
        oa, ra, ta, xa, _ = a.step(x.cuda())
        expected.append(({g: oa[g].cpu().clone() for g in oa}, ra.cpu().clone(), ta.cpu().clone(), xa.cpu().clone()))
        b.step_async(x)
        if i >= 2:  # up to three steps in flight
            got = b.step_wait()
            eo, er, et, ex = expected[i - 2]
            for g in eo:
                assert torch.equal(eo[g], got[f"obs/{g}"]), (i, g)
            assert torch.equal(er, got["reward"]) and torch.equal(et, got["terminated"])
            assert torch.equal(ex, got["truncated"])
    assert torch.equal(expected[-2][1], b.step_wait()["reward"])
    assert torch.equal(expected[-1][1], b.step_wait()["reward"])
    with pytest.raises(RuntimeError):
        b.step_wait()


@pytest.mark.gpu
@pytest.mark.parametrize("n,group,slots", [(256, 2, 6), (300, 2, 6), (256, 4, 6), (256, 1, 6), (256, 2, 2),
                                           (256, 2, 3)])
def test_step_async_paired_and_sequential_waits(monkeypatch, n, group, slots):
    """The grouped D2H (ss_pipe_post: the copies of `group` consecutive steps deferred and issued as one)
    under every wait pattern: strictly sequential (each deferred copy issued alone by step_wait), 2 to 6
    in flight (whole and partial groups); 300 worlds give an arena that is not a multiple of 16 bytes (no
    grouping). Every step's host results equal a synchronous step's."""
    from paper_2601_22074_b200 import env as envmod
    from paper_2601_22074_b200.env import ManagerBasedRlEnv
    from paper_2601_22074_b200.tasks import make_env_cfg

    monkeypatch.setenv("SS_PIPE_GROUP", str(group))
    monkeypatch.setattr(envmod, "PIPE_GROUP", group)
    monkeypatch.setattr(envmod, "PIPE_SLOTS", slots)
    a = ManagerBasedRlEnv(make_env_cfg("Velocity-Rough", num_envs=n, seed=3))
    b = ManagerBasedRlEnv(make_env_cfg("Velocity-Rough", num_envs=n, seed=3))
    a.reset()
    b.reset()
    rng = np.random.default_rng(11)
    pattern = [k for k in (1, 1, 1, 2, 2, 3, 1, 3, 2, 4, 5, 6, 4) if k <= slots]  # steps in flight per round
    acts = [torch.from_numpy(rng.uniform(-1, 1, size=(n, a.action_manager.total_dim))).pin_memory()
            for _ in range(sum(pattern))]
    want = []
    for x in acts:
        o, r, _, tr, _ = a.step(x.cuda())
        want.append((o["policy"].cpu().clone(), r.cpu().clone(), tr.cpu().clone()))
    i = 0
    for k in pattern:
        for j in range(k):
            b.step_async(acts[i + j])
        for j in range(k):
            got = b.step_wait()
            wo, wr, wt = want[i + j]
            assert torch.equal(got["obs/policy"], wo) and torch.equal(got["reward"], wr), (i + j, k)
            assert torch.equal(got["truncated"], wt)
        i += k


@pytest.mark.gpu
def test_step_wait_view_survives_the_next_step_async():
    """With the pipeline full (PIPE_SLOTS steps pending), the host view step_wait returned survives the
    next two step_async calls (PIPE_SLOTS + 2 host blocks, ss_pipe_*)."""
    from paper_2601_22074_b200.env import PIPE_SLOTS, ManagerBasedRlEnv
    from paper_2601_22074_b200.tasks import make_env_cfg

    a = ManagerBasedRlEnv(make_env_cfg("Velocity-Rough", num_envs=256, seed=2))
    b = ManagerBasedRlEnv(make_env_cfg("Velocity-Rough", num_envs=256, seed=2))
    a.reset()
    b.reset()
    rng = np.random.default_rng(8)
    acts = [torch.from_numpy(rng.uniform(-1, 1, size=(256, a.action_manager.total_dim))).pin_memory()
            for _ in range(PIPE_SLOTS + 7)]
    want = []
    for x in acts:
        _, r, _, _, _ = a.step(x.cuda())
        want.append(r.cpu().clone())
    for i in range(PIPE_SLOTS):
        b.step_async(acts[i])
    nxt, k = PIPE_SLOTS, 0  # next step to submit, next step to wait for
    while nxt + 1 < len(acts):
        view = b.step_wait()  # step k
        b.step_async(acts[nxt])  # the pipeline is full again
        view2 = b.step_wait()  # step k + 1
        b.step_async(acts[nxt + 1])  # a second enqueue
        torch.cuda.synchronize()  # every copy issued so far has landed
        assert torch.equal(view["reward"], want[k]) and torch.equal(view2["reward"], want[k + 1]), k
        nxt, k = nxt + 2, k + 2
    while k < nxt:  # drain the submitted steps
        assert torch.equal(b.step_wait()["reward"], want[k]), k
        k += 1


@pytest.mark.gpu
def test_copy_outputs_returns_fresh_tensors():
    """copy_outputs=True: every step returns new tensors (the reference returns fresh arrays), equal to
    the persistent buffers of that step; the default mode returns views the next step overwrites."""
    from paper_2601_22074_b200.env import ManagerBasedRlEnv
    from paper_2601_22074_b200.policies import random_policy
    from paper_2601_22074_b200.tasks import make_env_cfg

    fresh = ManagerBasedRlEnv(make_env_cfg("Velocity-Rough", num_envs=128, seed=4), copy_outputs=True)
    views = ManagerBasedRlEnv(make_env_cfg("Velocity-Rough", num_envs=128, seed=4))
    o0 = fresh.reset()
    views.reset()
    kept, first = [], None
    for i in range(5):
        o, r, te, tr, _ = fresh.step(random_policy(fresh, i))
        ov, rv, tev, trv, _ = views.step(random_policy(views, i))
        assert torch.equal(r, rv) and torch.equal(te, tev) and torch.equal(tr, trv)
        for g in o:
            assert torch.equal(o[g], ov[g])
        kept.append((o["policy"].clone(), r.clone(), o, r))
        if first is None:
            first = rv
    for snap_o, snap_r, o, r in kept:  # earlier steps' tensors were not overwritten
        assert torch.equal(o["policy"], snap_o) and torch.equal(r, snap_r)
    _, _, _, _, x1 = fresh.step(random_policy(fresh, 10))
    rows = x1["curriculum/terrain_rows"].clone()
    fresh.terrain_rows.add_(1)  # later changes to the env do not reach an earlier step's extras
    assert torch.equal(x1["curriculum/terrain_rows"], rows)
    fresh.terrain_rows.sub_(1)
    assert first.data_ptr() == views.reward_manager.reward.data_ptr()  # default: persistent buffer
    assert o0["policy"].data_ptr() != fresh.observation_manager.outputs()["policy"].data_ptr()


@pytest.mark.gpu
def test_split_launch_bitwise_equals_fused(monkeypatch):
    """Large envs step as two kernels compiled for fixed stage sets (physics | terms + observations,
    jit.split_enabled): bit-identical to the single fused launch, outputs and state."""
    from paper_2601_22074_b200.env import ManagerBasedRlEnv
    from paper_2601_22074_b200.policies import random_policy
    from paper_2601_22074_b200.tasks import make_env_cfg

    envs = []
    for mode in ("0", "1"):
        monkeypatch.setenv("SS_SPLIT", mode)
        e = ManagerBasedRlEnv(make_env_cfg("Velocity-Rough", num_envs=4096, seed=8), "Velocity-Rough")
        e.reset()
        e.step(random_policy(e, 0, fused=True))
        envs.append(e)
    a, b = envs
    assert a._jit_split is None and b._jit_split is not None
    for i in range(1, 40):
        for e in envs:
            e.step(random_policy(e, i, fused=True))
    torch.cuda.synchronize()
    assert torch.equal(a.step_outputs, b.step_outputs)
    for name in ("q", "qd", "ctrl", "ext_force", "time"):
        assert torch.equal(getattr(a.state, name), getattr(b.state, name)), name
    assert torch.equal(a.terrain_rows, b.terrain_rows)
    assert np.array_equal(np.array(list(a.termination_manager.trigger_counts.values())),
                          np.array(list(b.termination_manager.trigger_counts.values())))


@pytest.mark.gpu
def test_ppo_update_graph_equals_eager():
    """The CUDA-graph minibatch step trains exactly like the eager one (same parameters after the
    update, from the same rollout and the same random permutations)."""
    from paper_2601_22074_b200.env import ManagerBasedRlEnv
    from paper_2601_22074_b200.ppo import PpoCfg, PpoTrainer
    from paper_2601_22074_b200.tasks import make_env_cfg

    params = []
    for graph in (False, True):
        env = ManagerBasedRlEnv(make_env_cfg("Velocity-Flat", num_envs=256, seed=1))
        tr = PpoTrainer(env, PpoCfg(hidden=(64, 64), steps_per_env=8, epochs=2, minibatches=2, cuda_graph=graph),
                        seed=3)
        torch.manual_seed(5)
        tr.collect()
        torch.manual_seed(6)
        tr.update()
        torch.manual_seed(7)
        tr.collect()
        torch.manual_seed(8)
        st = tr.update()
        torch.cuda.synchronize()
        assert (tr._graph is not None) == graph and np.isfinite(st["loss"])
        params.append(tr.reducer.flat_param.clone())
    torch.testing.assert_close(params[0], params[1], rtol=1e-5, atol=1e-6)
