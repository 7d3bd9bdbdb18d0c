"""The multi-GPU contract on one device.

Rank r of an R-GPU job steps worlds [r*N, (r+1)*N) through
``SceneCfg.world_id_offset`` (reference env.py:67-69, :114; RNG keyed by the
global world id, terrain regenerated from the seed). On one B200 the ranks'
CUDA envs can be built side by side: two half-size envs with offsets 0 and
N/2, stepped with the fused policy draw, must reproduce one N-world env bit
for bit -- every state array, output and counter. The per-log-interval
statistics kernel (``ss_stats_pack``) must equal the torch restatement of
``metrics.build_record``'s packing, and the two shards' vectors must sum to
the single env's (the all-reduce the job performs).
"""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

TASK = "Velocity-Rough"


def _env(n, offset, seed=3):
    from paper_2601_22074_b200.env import ManagerBasedRlEnv
    from paper_2601_22074_b200.tasks import make_env_cfg

    cfg = make_env_cfg(TASK, num_envs=n, seed=seed)
    cfg.scene.world_id_offset = offset
    env = ManagerBasedRlEnv(cfg, TASK)
    env.reset()
    return env


@pytest.mark.parametrize("n", [2048, 4096])
def test_two_shards_equal_one_env_bitwise(n):
    from paper_2601_22074_b200.metrics import pack_stats
    from paper_2601_22074_b200.policies import random_policy

    whole, lo, hi = _env(n, 0), _env(n // 2, 0), _env(n // 2, n // 2)
    h = n // 2
    resets = 0
    for i in range(60):
        out = [e.step(random_policy(e, i, fused=True)) for e in (whole, lo, hi)]
        torch.cuda.synchronize()
        ow, rw, tw, trw, xw = out[0]
        for k in ow:
            assert torch.equal(ow[k], torch.cat([out[1][0][k], out[2][0][k]])), f"obs {k} step {i}"
        assert torch.equal(rw, torch.cat([out[1][1], out[2][1]])), f"reward step {i}"
        assert torch.equal(tw, torch.cat([out[1][2], out[2][2]])), f"terminated step {i}"
        assert torch.equal(trw, torch.cat([out[1][3], out[2][3]])), f"truncated step {i}"
        ids = torch.cat([out[1][4]["reset_ids"], out[2][4]["reset_ids"] + h])
        assert torch.equal(xw["reset_ids"], ids), f"reset ids step {i}"
        resets += int(ids.numel())
    for name in ("q", "qd", "ctrl", "ext_force", "time"):
        a = getattr(whole.state, name)
        b = torch.cat([getattr(lo.state, name), getattr(hi.state, name)])
        assert torch.equal(a, b), name
    assert torch.equal(whole.state.contact.in_contact, torch.cat([lo.state.contact.in_contact,
                                                                  hi.state.contact.in_contact]))
    assert torch.equal(whole.terrain_rows, torch.cat([lo.terrain_rows, hi.terrain_rows]))
    assert torch.equal(whole.action_manager.action, torch.cat([lo.action_manager.action, hi.action_manager.action]))
    cw = np.array(list(whole.termination_manager.trigger_counts.values()))
    c2 = np.array(list(lo.termination_manager.trigger_counts.values())) + np.array(
        list(hi.termination_manager.trigger_counts.values()))
    assert np.array_equal(cw, c2)
    assert resets > 0

    # the per-rank statistics kernel vs the torch packing, and shard vectors summing to the whole
    from paper_2601_22074_b200.metrics import StatsPacker

    vecs = []
    for e in (whole, lo, hi):
        rm, tm = e.reward_manager, e.termination_manager
        want = pack_stats(rm.reward, [rm.episodic_sums[k] for k in rm.terms], tm._counts, e.terrain_rows,
                          e.terrain.rows, tm.last_nonfinite)
        got = StatsPacker(e).pack()
        torch.cuda.synchronize()
        np.testing.assert_allclose(got.cpu().numpy(), want.cpu().numpy(), rtol=1e-12, atol=1e-12)
        vecs.append(got.clone())
    np.testing.assert_allclose((vecs[1] + vecs[2]).cpu().numpy(), vecs[0].cpu().numpy(), rtol=1e-12, atol=1e-12)


def test_stats_pack_deterministic_and_reusable():
    """Same inputs -> bit-identical vectors across launches (fixed reduction order; the ticket resets)."""
    from paper_2601_22074_b200.metrics import StatsPacker, build_record
    from paper_2601_22074_b200.policies import random_policy

    env = _env(65536, 0, seed=1)
    for i in range(3):
        env.step(random_policy(env, i, fused=True))
    p = StatsPacker(env)
    a = p.pack().clone()
    b = p.pack().clone()
    torch.cuda.synchronize()
    assert torch.equal(a, b)
    rec = build_record(env, 3, env.reward_manager.reward, None)
    assert sum(rec.terrain_row_histogram) == 65536
    assert rec.reward_mean == pytest.approx(float(env.reward_manager.reward.mean()), abs=1e-9)


@pytest.mark.parametrize("n", [4096, 262144])
def test_fused_step_statistics_equal_the_pack(n):
    """StatsPacker.request: the step kernel reduces the statistics in its tail (bench.py's log-interval
    path); the vector equals a separate ss_stats_pack of the same step's outputs, and the next step
    (no request) leaves it alone."""
    from paper_2601_22074_b200.metrics import StatsPacker
    from paper_2601_22074_b200.policies import random_policy

    env = _env(n, 0, seed=4)
    for i in range(30):
        env.step(random_policy(env, i, fused=True))
    p = StatsPacker(env)
    out = torch.full_like(p.out, -1.0)
    p.request(out)
    env.step(random_policy(env, 30, fused=True))
    want = p.pack().clone()
    torch.cuda.synchronize()
    np.testing.assert_allclose(out.cpu().numpy(), want.cpu().numpy(), rtol=1e-12, atol=1e-9)
    assert float(out[0]) == n and float(out[1:].abs().sum()) > 0
    keep = out.clone()
    env.step(random_policy(env, 31, fused=True))
    torch.cuda.synchronize()
    assert torch.equal(out, keep)
    # and again (the ticket was reset by the kernel)
    p.request(out)
    env.step(random_policy(env, 32, fused=True))
    want = p.pack().clone()
    torch.cuda.synchronize()
    np.testing.assert_allclose(out.cpu().numpy(), want.cpu().numpy(), rtol=1e-12, atol=1e-9)
