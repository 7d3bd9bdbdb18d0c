"""world_size-2 gloo tests of the multi-GPU host logic, on CPU.

The B200 job shards worlds across ranks with world_id_offset = rank * N and
no data-path collective; the only collective is the per-log-interval stats
all-reduce (metrics.build_record). Here: (1) two ranks stepping disjoint
shards reproduce a single-process run bit for bit (the property the sharding
relies on, checked on the oracle), (2) the packed stats all-reduce equals
the single-process statistics.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as tmp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n_total, steps, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import OracleEnv
    from paper_2601_22074_b200.metrics import allreduce_stats, pack_stats, unpack_stats
    from paper_2601_22074_b200.tasks import make_env_cfg
    from paper_2601_22074_b200.terrain import generate_grid

    n = n_total // world
    cfg = make_env_cfg("Velocity-Rough", num_envs=n, seed=5)
    cfg.scene.world_id_offset = rank * n
    env = OracleEnv(cfg, generate_grid(cfg.scene.terrain, cfg.seed).samples)
    env.reset()
    for _ in range(steps):
        _, rew, *_ = env.step(env.random_actions())
    q = torch.from_numpy(env.S["q"].copy())
    gathered = [torch.zeros_like(q) for _ in range(world)]
    dist.all_gather(gathered, q)
    vec = pack_stats(torch.from_numpy(rew), [torch.from_numpy(env.ep_sums[k]) for k in env.rw],
                     torch.tensor(list(env.trigger_counts.values())), torch.from_numpy(env.terrain_rows),
                     env.t_rows, torch.from_numpy(env.last_nonfinite))
    vec = allreduce_stats(vec)
    rec = unpack_stats(vec, list(env.rw), list(env.trigger_counts), env.t_rows, steps)
    if rank == 0:
        np.save(os.path.join(out_dir, "q.npy"), torch.cat(gathered).numpy())
        with open(os.path.join(out_dir, "rec.json"), "w") as fh:
            fh.write(rec.to_json_line())
    dist.destroy_process_group()


def test_two_rank_shards_equal_single_process(tmp_path):
    from oracle import OracleEnv
    from paper_2601_22074_b200.metrics import pack_stats, unpack_stats
    from paper_2601_22074_b200.tasks import make_env_cfg
    from paper_2601_22074_b200.terrain import generate_grid

    n_total, steps = 48, 25
    tmp.spawn(_worker, args=(2, _free_port(), n_total, steps, str(tmp_path)), nprocs=2, join=True)
    cfg = make_env_cfg("Velocity-Rough", num_envs=n_total, seed=5)
    env = OracleEnv(cfg, generate_grid(cfg.scene.terrain, cfg.seed).samples)
    env.reset()
    for _ in range(steps):
        _, rew, *_ = env.step(env.random_actions())
    assert np.array_equal(np.load(tmp_path / "q.npy"), env.S["q"])
    vec = pack_stats(torch.from_numpy(rew), [torch.from_numpy(env.ep_sums[k]) for k in env.rw],
                     torch.tensor(list(env.trigger_counts.values())), torch.from_numpy(env.terrain_rows),
                     env.t_rows, torch.from_numpy(env.last_nonfinite))
    single = unpack_stats(vec, list(env.rw), list(env.trigger_counts), env.t_rows, steps)
    multi = __import__("json").loads(open(tmp_path / "rec.json").read())
    assert multi["termination_counts"] == single.termination_counts
    assert multi["terrain_row_histogram"] == single.terrain_row_histogram
    assert multi["nonfinite_worlds"] == single.nonfinite_worlds
    assert multi["reward_mean"] == pytest.approx(single.reward_mean, abs=1e-9)
    for k, v in single.reward_terms.items():
        assert multi["reward_terms"][k] == pytest.approx(v, abs=1e-9)


def test_bench_self_launch_two_ranks_dry(tmp_path):
    """`bench.py --gpus 2` with no WORLD_SIZE starts 2 ranks itself (torch.distributed.run on 127.0.0.1);
    --dry-cpu runs the same shard / reduce plumbing on gloo + the oracle. The line must report 2 ranks,
    disjoint contiguous shards, and the reduced record of a single 2N-world run."""
    import json
    import subprocess
    import sys

    from oracle import OracleEnv
    from paper_2601_22074_b200.metrics import pack_stats, unpack_stats
    from paper_2601_22074_b200.tasks import make_env_cfg
    from paper_2601_22074_b200.terrain import generate_grid

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env_vars = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    n, steps, warmup = 20, 5, 3
    out = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", "2", "--dry-cpu", "--envs", str(n),
                          "--steps", str(steps), "--warmup", str(warmup)], capture_output=True, text=True,
                         timeout=600, env=env_vars, cwd=str(tmp_path))
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout  # rank 0 alone prints
    got = json.loads(lines[0])
    assert got["n_gpus"] == 2
    assert got["shards"]["world_id_offsets"] == [0, n]
    assert got["config"]["total_envs"] == 2 * n
    cfg = make_env_cfg("Velocity-Rough", num_envs=2 * n, seed=0)
    env = OracleEnv(cfg, generate_grid(cfg.scene.terrain, cfg.seed).samples)
    env.reset()
    for _ in range(steps + warmup):
        _, rew, *_ = env.step(env.random_actions())
    vec = pack_stats(torch.from_numpy(rew), [torch.from_numpy(env.ep_sums[k]) for k in env.rw],
                     torch.tensor(list(env.trigger_counts.values())), torch.from_numpy(env.terrain_rows),
                     env.t_rows, torch.from_numpy(env.last_nonfinite))
    single = unpack_stats(vec, list(env.rw), list(env.trigger_counts), env.t_rows, steps + warmup)
    rec = got["record"]
    assert rec["termination_counts"] == single.termination_counts
    assert rec["terrain_row_histogram"] == single.terrain_row_histogram
    assert rec["nonfinite_worlds"] == single.nonfinite_worlds
    assert rec["reward_mean"] == pytest.approx(single.reward_mean, abs=1e-9)
    for k, v in single.reward_terms.items():
        assert rec["reward_terms"][k] == pytest.approx(v, abs=1e-9)
