"""Line-delimited JSON metrics records (metrics.py of the reference), reduced
over every GPU of a job.

``build_record`` packs all per-log-interval statistics of a rank -- reward
sum, per-term episodic sums, trigger counts, the terrain-row histogram and
the nonfinite count -- into ONE float64 vector on the device, all-reduces it
(SUM) across ranks in a single collective (NCCL on GPUs; gloo works for CPU
tests) and unpacks the job-wide means. With one rank it is exactly the
reference's record (metrics.py:31-45).
"""

from __future__ import annotations

import json
from dataclasses import asdict, dataclass, field

import numpy as np


@dataclass
class MetricsRecord:
    step: int
    reward_mean: float
    steps_per_sec: float | None = None
    reward_terms: dict[str, float] = field(default_factory=dict)
    termination_counts: dict[str, int] = field(default_factory=dict)
    terrain_row_histogram: list[int] = field(default_factory=list)
    nonfinite_worlds: int = 0

    def to_json_line(self) -> str:
        return json.dumps(asdict(self), sort_keys=True, allow_nan=True)


def pack_stats(reward, episodic_sums: list, trigger_counts, terrain_rows, n_rows: int, nonfinite):
    """[n, sum(reward), sum(ep_sum_t)..., counts..., row histogram..., nonfinite] as float64."""
    import torch

    dev = reward.device
    parts = [
        torch.tensor([float(reward.numel())], dtype=torch.float64, device=dev),
        reward.to(torch.float64).sum().reshape(1),
    ]
    parts += [s.to(torch.float64).sum().reshape(1) for s in episodic_sums]
    parts.append(trigger_counts.to(torch.float64).reshape(-1))
    parts.append(torch.bincount(terrain_rows.reshape(-1), minlength=n_rows).to(torch.float64))
    parts.append(nonfinite.to(torch.float64).sum().reshape(1))
    return torch.cat(parts)


def allreduce_stats(vec, group=None):
    """SUM across ranks (one collective per log interval; a no-op without a process group)."""
    import torch.distributed as dist

    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(vec, op=dist.ReduceOp.SUM, group=group)
    return vec


def unpack_stats(vec, term_names, count_names, n_rows: int, step: int, steps_per_sec=None) -> MetricsRecord:
    v = vec.detach().cpu().numpy()
    n = v[0]
    t = len(term_names)
    c = len(count_names)
    reward_terms = {name: round(float(v[2 + i] / n), 10) for i, name in enumerate(term_names)}
    counts = {name: int(round(v[2 + t + i])) for i, name in enumerate(count_names)}
    hist = [int(round(x)) for x in v[2 + t + c : 2 + t + c + n_rows]]
    return MetricsRecord(step=step, reward_mean=round(float(v[1] / n), 10), steps_per_sec=steps_per_sec,
                         reward_terms=reward_terms, termination_counts=counts, terrain_row_histogram=hist,
                         nonfinite_worlds=int(round(v[2 + t + c + n_rows])))


class StatsPacker:
    """The CUDA env's per-rank statistics in ONE kernel launch (``ss_stats_pack``,
    csrc/ss_aux.cu): reads the step's reward, the episodic sums, trigger
    counts, terrain rows and the nonfinite mask straight from the env's device
    buffers and writes the packed vector ``pack_stats`` would build (same
    layout), deterministically. Buffers are allocated once per env."""

    def __init__(self, env):
        import torch

        from . import native

        self.env = env
        rm, tm = env.reward_manager, env.termination_manager
        self.n_rewards = len(rm.terms)
        self.n_counts = int(tm._counts.numel())
        self.n_rows = int(env.terrain.rows)
        dev = env.device
        self.out = torch.zeros(3 + self.n_rewards + self.n_counts + self.n_rows, dtype=torch.float64, device=dev)
        self._maxv = native.SS_STATS_MAXV
        self.partials = torch.zeros(native.SS_STATS_GRID * native.SS_STATS_MAXV, dtype=torch.float64, device=dev)
        self.ticket = torch.zeros(1, dtype=torch.int32, device=dev)
        self._args = native.StatsArgs()
        self._lib = native.lib()

    def request(self, out=None):
        """Have the env's NEXT full control step reduce the statistics itself, fused into the step
        kernel's tail (no extra launch), into ``out`` (default ``self.out``; same layout as ``pack``).
        The vector holds the statistics of that step once it has run."""
        import torch

        env = self.env
        if getattr(self, "_fpartials", None) is None:
            grid = -(-env.num_envs // 32)  # >= the step kernel's grid at any block size
            self._fpartials = torch.zeros(grid * self._maxv, dtype=torch.float64, device=env.device)
            self._fticket = torch.zeros(1, dtype=torch.int32, device=env.device)
        out = self.out if out is None else out
        env._stats_req = (out.data_ptr(), self._fpartials.data_ptr(), self._fticket.data_ptr(), self.n_rows)
        env._stats_req_out = out  # keeps the destination alive until the launch has consumed the request
        return out

    def pack(self, reward=None):
        """Launch the reduction on the current stream; returns the (device) vector."""
        import ctypes

        from . import native

        env = self.env
        rm, tm = env.reward_manager, env.termination_manager
        reward = rm.reward if reward is None else reward
        a = self._args
        a.n_worlds, a.n_rewards, a.n_counts, a.n_rows = env.num_envs, self.n_rewards, self.n_counts, self.n_rows
        a.reward = reward.data_ptr()
        a.ep_sums = rm._sums.data_ptr() if self.n_rewards else None  # one SoA block (T, N)
        a.trigger_counts = tm._counts.data_ptr()
        a.terrain_rows = env.terrain_rows.data_ptr()
        a.nonfinite = tm.last_nonfinite.data_ptr()
        a.partials = self.partials.data_ptr()
        a.ticket = self.ticket.data_ptr()
        a.out = self.out.data_ptr()
        native.LAUNCHES["count"] += 1
        rc = self._lib.ss_stats_pack(ctypes.byref(a), native.current_stream(env._dev_index))
        if rc != 0:
            raise native.NativeError(f"ss_stats_pack failed ({rc}): {self._lib.ss_last_error().decode()}")
        return self.out


def build_record(env, step: int, reward, steps_per_sec: float | None, group=None) -> MetricsRecord:
    """One JSONL record of the job (metrics.py:31-45): this rank's statistics
    packed on the device, ONE all-reduce across ranks, unpacked on the host."""
    rm, tm = env.reward_manager, env.termination_manager
    if getattr(env, "_lib", None) is not None and reward.is_cuda:
        packer = getattr(env, "_stats_packer", None)
        if packer is None:
            packer = env._stats_packer = StatsPacker(env)
        vec = packer.pack(reward)
    else:
        vec = pack_stats(reward, [rm.episodic_sums[k] for k in rm.terms], tm._counts, env.terrain_rows,
                         env.terrain.rows, tm.last_nonfinite)
    vec = allreduce_stats(vec, group)
    return unpack_stats(vec, list(rm.terms), list(tm.trigger_counts), env.terrain.rows, step, steps_per_sec)


class MetricsWriter:
    def __init__(self, path: str):
        self.path = path
        self._fh = open(path, "w")

    def write(self, record: MetricsRecord) -> None:
        self._fh.write(record.to_json_line() + "\n")
        self._fh.flush()

    def close(self) -> None:
        self._fh.close()


__all__ = ["MetricsRecord", "MetricsWriter", "StatsPacker", "allreduce_stats", "build_record", "pack_stats",
           "unpack_stats"]
_ = np
