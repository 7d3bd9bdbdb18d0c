"""Parity at the exact configurations bench.py times.

The headline bench line runs Velocity-Rough at N=4096 worlds with the random
policy drawn inside the step kernel (``random_policy(env, i, fused=True)``,
the reference's benchmark loop, cli.py:155-172); its ``at_scale`` leg runs the
same step at N=262,144, where the per-env specialization folds N into every
immediate offset. These tests run exactly those launches against the pinned
numpy oracle (tests/test_oracle_golden.py pins it bit-for-bit to the
reference's golden vectors):

* N=4096, fused policy: 10 free-running control steps within the north
  star's fp32 tolerance (1e-6), then 30 teacher-forced steps (the GPU env is
  loaded with the oracle's state before each step) with contact sets,
  termination/truncation flags and reset ids exact and floats within 1e-9;
  the fused draw itself must equal the oracle's ``policy.random`` draw bit for
  bit every step.
* N=262,144, fused policy: the oracle runs contiguous world slices built with
  ``world_id_offset`` = slice start (partition independence, SPEC.md:113,
  reference tests/test_env.py:256-270) and teacher-forces only its slice of
  the GPU state; the same exactness rules hold on every slice.
"""

import numpy as np
import pytest

from helpers import sync_from_oracle

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

RTOL = ATOL = 1e-9
FP32 = 1e-6
TASK = "Velocity-Rough"


def _close(a, b, what, tol):
    a = a.detach().cpu().numpy() if hasattr(a, "detach") else np.asarray(a)
    np.testing.assert_allclose(a, b, rtol=tol, atol=tol, err_msg=what)


def _check(env, ref, out_gpu, out_ref, sl, i, tol):
    o1, r1, t1, tr1, x1 = out_gpu
    o2, r2, t2, tr2, x2 = out_ref
    t1 = t1.cpu().numpy()[sl]
    tr1 = tr1.cpu().numpy()[sl]
    assert np.array_equal(t1, t2), f"terminated step {i}"
    assert np.array_equal(tr1, tr2), f"truncated step {i}"
    assert np.array_equal(np.flatnonzero(t1 | tr1), x2["reset_ids"]), f"reset ids step {i}"
    assert np.array_equal(env.state.contact.in_contact.cpu().numpy()[sl], ref.S["fin"]), f"contact set step {i}"
    _close(env.state.q[sl], ref.S["q"], f"q step {i}", tol)
    _close(env.state.qd[sl], ref.S["qd"], f"qd step {i}", tol)
    _close(env.state.ctrl[sl], ref.S["ctrl"], f"ctrl step {i}", tol)
    _close(r1[sl], r2, f"reward step {i}", tol)
    for k in o2:
        _close(o1[k][sl], o2[k], f"obs {k} step {i}", tol)


def test_headline_config_fused_policy_lockstep():
    """bench.py's headline launch: Velocity-Rough, 4096 worlds, fused random policy."""
    from oracle import OracleEnv
    from paper_2601_22074_b200.env import ManagerBasedRlEnv
    from paper_2601_22074_b200.policies import random_policy
    from paper_2601_22074_b200.tasks import make_env_cfg

    n, seed = 4096, 0
    env = ManagerBasedRlEnv(make_env_cfg(TASK, num_envs=n, seed=seed), TASK)
    ref = OracleEnv(make_env_cfg(TASK, num_envs=n, seed=seed), env.terrain.samples)
    assert env.use_jit, "the bench runs the per-env specialized kernel"
    o1, o2 = env.reset(), ref.reset()
    for k in o2:
        _close(o1[k], o2[k], f"reset obs {k}", RTOL)
    sl = slice(None)
    resets = 0
    for i in range(40):
        forced = i >= 10
        if forced:
            sync_from_oracle(env, ref)
        a = ref.random_actions()
        out_gpu = env.step(random_policy(env, i, fused=True))
        out_ref = ref.step(a)
        # the fused draw equals the oracle's policy.random draw (worlds reset in this step hold zeros,
        # ActionManager.reset, managers/action.py:92-97)
        drawn = a.copy()
        drawn[out_ref[4]["reset_ids"]] = 0.0
        assert np.array_equal(env.action_manager.action.cpu().numpy(), drawn), f"fused policy draw step {i}"
        assert np.array_equal(drawn, ref.action), f"oracle action step {i}"
        _check(env, ref, out_gpu, out_ref, sl, i, RTOL if forced else FP32)
        resets += len(out_ref[4]["reset_ids"])
    assert resets > 0, "the window must exercise the masked reset path"


@pytest.mark.parametrize("n,m,starts", [(262144, 2048, (0, 131072 - 1024, 262144 - 2048)),
                                         (1048576, 1024, (0, 1048576 - 1024)),  # the at_scale leg's 4x point
                                         # block 128 with a partial last block (70001 = 546 x 128 + 113)
                                         (70001, 1500, (0, 70001 - 1500))])
def test_at_scale_config_world_slices(n, m, starts):
    """bench.py's at_scale launch: 262,144 worlds, fused random policy, world slices vs the oracle
    (and a large world count that is not a multiple of the block)."""
    from oracle import OracleEnv
    from paper_2601_22074_b200.env import ManagerBasedRlEnv
    from paper_2601_22074_b200.policies import random_policy
    from paper_2601_22074_b200.tasks import make_env_cfg

    seed = 0
    env = ManagerBasedRlEnv(make_env_cfg(TASK, num_envs=n, seed=seed), TASK)
    assert env.use_jit
    refs = []
    for a0 in starts:
        cfg = make_env_cfg(TASK, num_envs=m, seed=seed)
        cfg.scene.world_id_offset = a0
        refs.append((a0, OracleEnv(cfg, env.terrain.samples)))
    o1 = env.reset()
    for a0, ref in refs:
        o2 = ref.reset()
        for k in o2:
            _close(o1[k][a0 : a0 + m], o2[k], f"reset obs {k} slice {a0}", RTOL)
    resets = 0
    for i in range(36):
        forced = i >= 6
        if forced:
            for a0, ref in refs:
                sync_from_oracle(env, ref, world_start=a0)
        acts = [ref.random_actions() for _, ref in refs]
        out_gpu = env.step(random_policy(env, i, fused=True))
        drawn = env.action_manager.action.cpu().numpy()
        for (a0, ref), a in zip(refs, acts):
            sl = slice(a0, a0 + m)
            out_ref = ref.step(a)
            want = a.copy()
            want[out_ref[4]["reset_ids"]] = 0.0  # reset worlds hold zeros (managers/action.py:92-97)
            assert np.array_equal(drawn[sl], want), f"fused policy draw step {i} slice {a0}"
            _check(env, ref, out_gpu, out_ref, sl, i, RTOL if forced else FP32)
            resets += len(out_ref[4]["reset_ids"])
    assert resets > 0
