"""Pin the numpy oracle to the reference's own outputs (tests/golden, made by
tests/golden/make_golden.py from the unmodified reference). CPU only."""

import numpy as np
import pytest

from helpers import cfg_from_golden, golden, samples_for, spec_from_json
from oracle import OracleEnv, OracleModel, OracleStreams
from oracle.physics import heights_fn, new_state, oracle_substep
from paper_2601_22074_b200 import config as C

ROLLOUTS = ["rollout_flat.npz", "rollout_rough.npz", "rollout_soup.npz", "rollout_quad.npz", "rollout_mlp.npz"]


def test_terrain_generation_matches_reference():
    g = golden("terrain_rough_seed0.npz")
    from paper_2601_22074_b200.tasks import make_env_cfg
    from paper_2601_22074_b200.terrain import generate_grid

    t = generate_grid(make_env_cfg("Velocity-Rough").scene.terrain, 0)
    assert np.array_equal(t.samples, g["samples"])
    assert np.array_equal(t.difficulty, g["difficulty"])
    assert np.array_equal(t.type_index, g["type_index"])


def test_rng_matches_reference():
    g = golden("rng.npz")
    sp = OracleStreams(7, 100 + np.arange(6))
    assert np.array_equal(sp.uniform("a.b", -2.0, 3.0, None, 5), g["u_all"])
    assert np.array_equal(sp.uniform("a.b", 0.0, 1.0, np.array([1, 4]), 3), g["u_sel"])
    assert np.array_equal(sp.uniform("c", np.arange(6.0), np.arange(6.0) + 2.0, None, 2), g["u_rowlo"])
    assert np.array_equal(sp.normal("d", 0.5, None, 3), g["n_all"])
    assert np.array_equal(sp.normal("d", 2.0, np.array([0, 5]), 2), g["n_sel"])
    u = sp.uniform("e", 0.0, 1.0, None, 7)
    assert np.array_equal(-3 + np.floor(u * 8).astype(np.int64), g["i_all"])


@pytest.mark.parametrize("case", ["biped_flat", "biped_rough", "quad_flat", "quad_rough", "humanoid_flat",
                                  "humanoid_rough"])
def test_oracle_physics_matches_reference(case):
    g = golden("physics.npz")
    spec = spec_from_json(g[f"{case}/spec_json"])
    q0 = g[f"{case}/q0"]
    m = OracleModel(spec, q0.shape[0])
    samples = None
    if case.endswith("rough"):
        from paper_2601_22074_b200.tasks import make_env_cfg
        samples = golden("terrain_rough_seed0.npz")["samples"]
    S = new_state(m)
    S["q"][...] = q0
    S["qd"][...] = g[f"{case}/qd0"]
    S["ctrl"][...] = g[f"{case}/ctrl"]
    S["ext"][...] = g[f"{case}/ext0"]
    h = heights_fn(samples, 0.05)
    for i in range(g[f"{case}/q"].shape[0]):
        oracle_substep(m, h, S)
        assert np.array_equal(S["q"], g[f"{case}/q"][i]), i
        assert np.array_equal(S["qd"], g[f"{case}/qd"][i]), i
    for k in ("fn", "ft", "fin", "fpos", "fvel"):
        assert np.array_equal(S[k], g[f"{case}/{k}"]), k


@pytest.mark.parametrize("name", ROLLOUTS)
def test_oracle_rollout_matches_reference(name):
    g = golden(name)
    cfg = cfg_from_golden(g)
    assert C.config_hash(cfg) == str(g["config_hash"])
    env = OracleEnv(cfg, samples_for(cfg))
    obs0 = env.reset()
    for gname in obs0:
        assert np.array_equal(obs0[gname], g[f"obs0/{gname}"]), gname
    for i in range(g["actions"].shape[0]):
        obs, rew, term, trunc, _ = env.step(g["actions"][i])
        assert np.array_equal(env.S["q"], g["q"][i]), i
        assert np.array_equal(env.S["qd"], g["qd"][i]), i
        assert np.array_equal(env.S["ctrl"], g["ctrl"][i]), i
        assert np.array_equal(rew, g["reward"][i]), i
        assert np.array_equal(term, g["terminated"][i]), i
        assert np.array_equal(trunc, g["truncated"][i]), i
        for gname in obs:
            assert np.array_equal(obs[gname], g[f"obs/{gname}"][i]), (i, gname)
    counts = np.array(list(env.trigger_counts.values()), dtype=np.int64)
    assert np.array_equal(counts, g["trigger_counts"])
    assert np.array_equal(env.terrain_rows, g["terrain_rows"])
    assert np.array_equal(env.ranges, g["ranges"])
    assert np.array_equal(env.sens["last_air"], g["sensor_last_air"])
    assert env.S["sim_step"] == int(g["sim_step"])
    for k in g.files:
        if k.startswith("field/"):
            assert np.array_equal(np.asarray(env.field(k[6:])), g[k]), k


def test_oracle_random_policy_matches_recorded_actions():
    g = golden("rollout_rough.npz")
    cfg = cfg_from_golden(g)
    env = OracleEnv(cfg, samples_for(cfg))
    env.reset()
    for i in range(5):
        a = env.random_actions()
        assert np.array_equal(a, g["actions"][i])
        env.step(a)
