"""Learner-side algebra on CPU (the reference has no learner -- parity unpinned): the flat-bucket
all-reduce across 2 gloo ranks equals the gradient of the concatenated batch on one process, GAE matches a
scalar recurrence, advantage normalization uses the job's statistics, and the PPO objective matches a
float64 numpy restatement of the clipped surrogate."""

import os
import socket

import torch
import torch.distributed as dist
import torch.multiprocessing as tmp


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _data(seed, n):
    g = torch.Generator().manual_seed(seed)
    return (torch.randn(n, 6, generator=g), torch.randn(n, 8, generator=g), torch.randn(n, 3, generator=g),
            torch.randn(n, generator=g), torch.randn(n, generator=g), torch.randn(n, generator=g))


def _model():
    from paper_2601_22074_b200.ppo import ActorCritic, PpoCfg

    torch.manual_seed(0)
    cfg = PpoCfg(hidden=(16, 16))
    return ActorCritic(6, 8, 3, cfg), cfg


def _worker(rank, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=2)
    from paper_2601_22074_b200.ppo import FlatGradReducer, ppo_loss

    model, cfg = _model()
    loss = ppo_loss(model, cfg, *_data(rank, 32))
    loss.backward()
    FlatGradReducer(model).reduce()
    if rank == 0:
        torch.save([p.grad.clone() for p in model.parameters()], out)
    dist.destroy_process_group()


def test_flat_bucket_allreduce_equals_concatenated_batch(tmp_path):
    from paper_2601_22074_b200.ppo import ppo_loss

    out = str(tmp_path / "g.pt")
    tmp.spawn(_worker, args=(_port(), out), nprocs=2, join=True)
    got = torch.load(out)
    model, cfg = _model()
    # mean over two equal halves == mean of the two per-rank means
    a, b = _data(0, 32), _data(1, 32)
    loss = 0.5 * (ppo_loss(model, cfg, *a) + ppo_loss(model, cfg, *b))
    loss.backward()
    for g, p in zip(got, model.parameters()):
        assert torch.allclose(g, p.grad, atol=1e-6, rtol=1e-5)


def test_gae_matches_scalar_recurrence():
    from paper_2601_22074_b200.ppo import gae

    g = torch.Generator().manual_seed(3)
    T, n = 7, 3
    r, v = torch.randn(T, n, generator=g), torch.randn(T, n, generator=g)
    d = (torch.rand(T, n, generator=g) < 0.2).float()
    lv = torch.randn(n, generator=g)
    adv, ret = gae(r, v, d, lv, 0.99, 0.95)
    for j in range(n):
        last = 0.0
        for t in reversed(range(T)):
            nv = lv[j] if t == T - 1 else v[t + 1, j]
            delta = r[t, j] + 0.99 * nv * (1 - d[t, j]) - v[t, j]
            last = delta + 0.99 * 0.95 * (1 - d[t, j]) * last
            assert abs(float(adv[t, j]) - float(last)) < 1e-5
    assert torch.allclose(ret, adv + v)


def test_advantage_normalization_single_rank_matches_torch():
    from paper_2601_22074_b200.ppo import normalize_advantages

    a = torch.randn(64, 8, generator=torch.Generator().manual_seed(2))
    want = (a - a.mean()) / (a.std() + 1e-8)
    assert torch.allclose(normalize_advantages(a), want, atol=1e-6)


def _norm_worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2601_22074_b200.ppo import normalize_advantages

    full = torch.randn(32, 6, generator=torch.Generator().manual_seed(5))
    mine = full[rank * 16 : (rank + 1) * 16]
    torch.save(normalize_advantages(mine), os.path.join(out, f"n{rank}.pt"))
    dist.destroy_process_group()


def test_advantage_normalization_uses_job_statistics(tmp_path):
    """Two ranks normalize their halves with the job-wide mean/std: identical to normalizing the whole batch."""
    from paper_2601_22074_b200.ppo import normalize_advantages

    tmp.spawn(_norm_worker, args=(2, _port(), str(tmp_path)), nprocs=2, join=True)
    full = torch.randn(32, 6, generator=torch.Generator().manual_seed(5))
    got = torch.cat([torch.load(tmp_path / "n0.pt"), torch.load(tmp_path / "n1.pt")])
    assert torch.allclose(got, normalize_advantages(full), atol=1e-6)


def test_ppo_loss_matches_a_numpy_restatement():
    """The clipped-surrogate objective (Schulman et al. 2017): -mean(min(r A, clip(r, 1-e, 1+e) A)) +
    c_v mean((R - V)^2) - c_e mean(entropy), with a diagonal Gaussian policy -- restated in float64 numpy
    from the network's own mean / log-std / value outputs, including ratios outside the clip range."""
    import math

    import numpy as np

    from paper_2601_22074_b200.ppo import ppo_loss

    model, cfg = _model()
    obs_p, obs_c, act, old_logp, adv, ret = _data(7, 64)
    old_logp = old_logp * 2.0  # ratios far from 1: both clip branches taken
    loss = float(ppo_loss(model, cfg, obs_p, obs_c, act, old_logp, adv, ret).detach())
    with torch.no_grad():
        mu = model.actor(obs_p).double().numpy()
        ls = model.log_std.double().numpy()
        v = model.critic(obs_c).squeeze(-1).double().numpy()
    a, A, R, lp0 = (x.double().numpy() for x in (act, adv, ret, old_logp))
    logp = np.sum(-((a - mu) ** 2) / (2.0 * np.exp(2.0 * ls)) - ls - 0.5 * math.log(2.0 * math.pi), axis=1)
    ratio = np.exp(logp - lp0)
    assert (ratio > 1 + cfg.clip).any() and (ratio < 1 - cfg.clip).any()
    surr = np.minimum(ratio * A, np.clip(ratio, 1 - cfg.clip, 1 + cfg.clip) * A)
    ent = np.sum(0.5 + 0.5 * math.log(2.0 * math.pi) + ls) * np.ones(len(a))
    want = -surr.mean() + cfg.value_coef * np.mean((R - v) ** 2) - cfg.entropy_coef * ent.mean()
    assert abs(loss - want) < 1e-5 * max(1.0, abs(want))
