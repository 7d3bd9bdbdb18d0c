"""Benchmark: env-steps/s of the batched ManagerBasedRlEnv.step on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--envs 4096] [--task Velocity-Rough]
    python bench.py --impl reference ...      # the unmodified reference on the host cores

Workload (BASELINE.json configs[1] restated): Velocity-Rough,
the planar biped on the 5x6 curriculum heightfield, 4096 worlds per GPU,
decimation 4, random actions from the per-world policy.random streams, drawn
inside the timed region like cli.py:163 -- by the step kernel itself
(policies.RandomActions; the same values as random_policy's separate draw,
tests/test_gpu_env_api.py). One step = one control step of every world (4
physics substeps each) = one kernel launch; every --log-every steps that
launch also reduces the job statistics, all-reduced across ranks. Multi-GPU:
one process per GPU (self-launched with torch.distributed.run when WORLD_SIZE
is unset), world_id_offset = rank * N (weak scaling, no collective on the
data path); time = max over ranks.

Timing: W untimed warm-up steps; then K steps, each preceded by an L2 flush
(a 512 MiB write, untimed) and bracketed by CUDA events on the launching
stream; barrier + synchronize around the whole region. The JSON line adds the
roofline of the fused step kernel (and the same step at 262,144 / 1,048,576
worlds), the CPU baseline (the unmodified reference on the host cores), an
end-to-end figure through the public API with host buffers, the 3-D path's
legs and a PPO training leg with its gradient all-reduce (f2).
"""

from __future__ import annotations

import argparse
import json
import multiprocessing as mp
import os
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

METRIC = "env-steps/sec (physics, whole box) at 1/2/4/8 B200 vs host-CPU reference"
UNIT = "env-steps/s"


def _peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as fh:
            j = json.load(fh)
        return float(j["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def _ncu_traffic():
    """dram bytes per launch of the step kernel from the committed ncu capture (or None)."""
    p = os.path.join(ROOT, "profiles", "ncu_step_kernel.json")
    try:
        with open(p) as fh:
            j = json.load(fh)
        return j.get("dram_bytes_per_launch"), j.get("envs")
    except Exception:
        return None, None


# ---------------------------------------------------------------------------
# CPU side: the reference's own implementation on the host cores, partitioned
# over processes through world_id_offset (partition-independent per world,
# reference tests/test_env.py:256-270)

REF_DIR = os.path.join(ROOT, "baseline", "_ref")  # the unmodified reference, pip-installed


def reference_available() -> bool:
    return os.path.isfile(os.path.join(REF_DIR, "stridesim", "env.py"))


def _cpu_worker(conn, kind, task, n_local, offset, seed):
    os.environ.setdefault("OMP_NUM_THREADS", "1")
    if kind == "reference":
        # the unmodified reference through its own public API: make_env_cfg ->
        # ManagerBasedRlEnv -> reset -> step(random_policy(env, i)) (cli.py:155-164)
        sys.path.insert(0, REF_DIR)
        from stridesim.env import ManagerBasedRlEnv
        from stridesim.policies import random_policy
        from stridesim.tasks import make_env_cfg

        cfg = make_env_cfg(task, num_envs=n_local, seed=seed)
        cfg.scene.world_id_offset = offset
        env = ManagerBasedRlEnv(cfg, task)
        env.reset()
        step = lambda i: env.step(random_policy(env, i))  # noqa: E731
    else:
        # the numpy restatement (oracle/, bit-identical to the reference, tests/test_oracle_golden.py)
        sys.path.insert(0, ROOT)
        from oracle import OracleEnv
        from paper_2601_22074_b200.tasks import make_env_cfg
        from paper_2601_22074_b200.terrain import generate_grid

        cfg = make_env_cfg(task, num_envs=n_local, seed=seed)
        cfg.scene.world_id_offset = offset
        env = OracleEnv(cfg, generate_grid(cfg.scene.terrain, cfg.seed).samples)
        env.reset()
        step = lambda i: env.step(env.random_actions())  # noqa: E731
    conn.send("ready")
    i = 0
    while True:
        msg = conn.recv()
        if msg == "stop":
            break
        n_steps = int(msg)
        t0 = time.perf_counter()
        for _ in range(n_steps):
            step(i)
            i += 1
        conn.send(time.perf_counter() - t0)


class CpuBaseline:
    """Persistent worker pool; each run(k) runs k control steps of all worlds.

    kind "reference": the unmodified reference package (baseline/_ref);
    kind "port": the oracle restatement."""

    def __init__(self, task, n_total, seed=0, procs=None, kind=None):
        self.kind = kind or ("reference" if reference_available() else "port")
        procs = procs or min(os.cpu_count() or 1, n_total)
        self.procs = procs
        ctx = mp.get_context("spawn")
        self.conns, self.workers = [], []
        split = np.array_split(np.arange(n_total), procs)
        for part in split:
            a, b = ctx.Pipe()
            w = ctx.Process(target=_cpu_worker, args=(b, self.kind, task, len(part), int(part[0]), seed), daemon=True)
            w.start()
            self.conns.append(a)
            self.workers.append(w)
        for c in self.conns:
            assert c.recv() == "ready"

    def run(self, n_steps: int) -> float:
        """Wall seconds for n_steps control steps of all worlds (the slowest worker)."""
        t0 = time.perf_counter()
        for c in self.conns:
            c.send(n_steps)
        for c in self.conns:
            c.recv()
        return time.perf_counter() - t0

    def close(self):
        for c in self.conns:
            c.send("stop")
        for w in self.workers:
            w.join(timeout=10)


def cpu_model_name() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def _describe(kind: str) -> str:
    return ("the unmodified reference (stridesim 0.1.0 from baseline/_ref, its own make_env_cfg / "
            "ManagerBasedRlEnv / random_policy)" if kind == "reference"
            else "the numpy oracle port of the reference (oracle/, bit-identical to it)")


def measure_cpu(task, n, seconds=10.0, procs=None, kind=None):
    pool = CpuBaseline(task, n, procs=procs, kind=kind)
    try:
        pool.run(3)
        steps, el = 0, 0.0
        while el < seconds:
            el += pool.run(5)
            steps += 5
    finally:
        pool.close()
    return {"value": n * steps / el, "unit": UNIT, "cores": pool.procs, "kind": pool.kind,
            "sample": f"{task} N={n} split over {pool.procs} processes (world_id_offset), {steps} control steps "
                      f"({el:.1f} s wall), random actions, {_describe(pool.kind)}, CPU {cpu_model_name()}"}


def bench_config(task: str, n: int, world: int) -> dict:
    """The workload record, key- and value-identical in both arms."""
    sys.path.insert(0, ROOT)
    from paper_2601_22074_b200.tasks import make_env_cfg

    cfg = make_env_cfg(task, num_envs=n)
    dec = cfg.decimation if cfg.decimation is not None else cfg.scene.model.decimation
    return {"workload": f"{task} (planar biped restatement of BASELINE configs[1], SURVEY 0.1)",
            "task": task, "envs_per_gpu": n, "total_envs": n * world, "decimation": int(dec),
            "parallelism": f"dp{world} (world shards, world_id_offset = rank * envs_per_gpu)",
            "l2": "flushed between timed iterations (GPU arm: 512 MiB device write before each step)"}


# ---------------------------------------------------------------------------
# clocks during the timed region


class Clocks:
    def __init__(self, index: int):
        self.path = os.path.join(ROOT, "gpurun_out", f"clocks_rank{index}.csv")
        os.makedirs(os.path.dirname(self.path), exist_ok=True)
        # the recipe's clocks line at its 200 ms period, reduced to the fields the JSON needs (every throttle
        # reason is a bit of clocks_event_reasons.active): a running sampler perturbs the ~21 us headline step
        # -- 20-step windows started together with the full line at 100 ms measured up to 5x slower in 5 of 12
        # trials, and any sampler adds ~0.3-1 us per step on average (tools/sampler_ab.py) -- so it runs with
        # few queries, at the recipe's period, and is started ahead of the warm-up
        q = "index,clocks.sm,clocks.max.sm,clocks_event_reasons.active"
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(index), f"--query-gpu={q}", "--format=csv,noheader,nounits",
                                          "-lms", "200"], stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
        # nvidia-smi can take a while to start on a fresh box: wait (bounded) for its first sample so the
        # sampler is live when the timed region begins
        t0 = time.time()
        while self.proc is not None and time.time() - t0 < 5.0 and self._lines() == 0:
            time.sleep(0.05)

    def _lines(self) -> int:
        try:
            with open(self.path) as fh:
                return sum(1 for _ in fh)
        except OSError:
            return 0

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        n0, t0 = self._lines(), time.time()
        while time.time() - t0 < 2.0 and self._lines() < n0 + 2:  # at least two samples after the region
            time.sleep(0.05)
        self.proc.terminate()
        self.proc.wait()
        sm, mx, reasons, masks = [], None, set(), set()
        # NVML clocks-event reason bits (nvmlClocksEventReason*)
        names = {0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
                 0x80: "hw_power_brake_slowdown"}
        for line in open(self.path):
            f = [x.strip() for x in line.split(",")]
            if len(f) < 4:
                continue
            try:
                sm.append(float(f[1]))
                mx = float(f[2])
                bits = int(f[3], 16)
            except ValueError:
                continue
            masks.add(f[3])
            reasons.update(nm for b, nm in names.items() if bits & b)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm), "event_reason_masks": sorted(masks)}


# ---------------------------------------------------------------------------


def dist_setup(gpus, backend="nccl"):
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if backend == "nccl":
        import torch

        torch.cuda.set_device(local)
    if world > 1:
        import torch
        import torch.distributed as dist

        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        if backend == "nccl":
            # communicator setup (rank count, NVLink / NVLS transport) logged -- to stderr, so stdout
            # carries nothing but rank 0's JSON line
            os.environ.setdefault("NCCL_DEBUG", "INFO")
            os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    return rank, world, local


def barrier(world):
    if world > 1:
        import torch.distributed as dist

        dist.barrier()


def allmax(x: float, world: int) -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist

    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def timed_steps(env, steps: int, flush, stream, policy, after=None, before=None) -> float:
    """Seconds of GPU time for `steps` env steps, each preceded by an L2 flush
    (untimed) and bracketed by CUDA events on the launching stream. `before(i)`
    / `after(i)` run inside step i's bracket (the per-log-interval statistics:
    fused into the step, then the all-reduce)."""
    import torch

    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    torch.cuda.synchronize()
    for i in range(steps):
        flush.fill_(float(i))  # evict L2 (126 MB) between timed iterations (untimed)
        e0, e1 = evs[i]
        e0.record(stream)
        if before is not None:
            before(i)
        env.step(policy(i))
        if after is not None:
            after(i)
        e1.record(stream)
        if i >= 2:
            # bound the host's lead to two iterations: the flush of the next
            # iteration gives the host time to enqueue the step before the GPU
            # reaches e0, so the events time GPU work only
            evs[i - 2][1].synchronize()
    torch.cuda.synchronize()
    return sum(e0.elapsed_time(e1) for e0, e1 in evs) / 1e3


def at_scale(args, flush, stream) -> dict:
    """The same step at world counts past the L2 (the roofline
    fraction is quoted where the working set streams from HBM): --scale-envs
    (262,144) and 4x that; the first is the line's `at_scale`, both are listed
    in `at_scale.points`."""
    pts = [_at_scale_point(args, flush, stream, n) for n in (args.scale_envs, 4 * args.scale_envs)]
    out = dict(pts[0])
    out["points"] = [{k: p[k] for k in ("envs", "value", "ms_per_step", "achieved_gbs", "frac")} for p in pts]
    return out


def _at_scale_point(args, flush, stream, n) -> dict:
    from paper_2601_22074_b200.env import ManagerBasedRlEnv
    from paper_2601_22074_b200.policies import random_policy
    from paper_2601_22074_b200.tasks import make_env_cfg
    from paper_2601_22074_b200.traffic import step_bytes_per_world

    env = ManagerBasedRlEnv(make_env_cfg(args.task, num_envs=n, seed=args.seed), args.task)
    env.reset()
    for i in range(5):
        env.step(random_policy(env, i, fused=True))
    steps = 20
    t = timed_steps(env, steps, flush, stream, lambda i: random_policy(env, 5 + i, fused=True))
    per_world = step_bytes_per_world(env, fused_policy=True)["total"]
    peak, _ = _peaks()
    gbs = per_world * n * steps / t / 1e9
    out = {"envs": n, "value": n * steps / t, "unit": UNIT, "ms_per_step": 1e3 * t / steps,
           "achieved_gbs": gbs, "frac": gbs / peak, "bytes_per_env_step": per_world}
    del env
    import torch

    torch.cuda.empty_cache()
    return out


def sim3d_leg(args, flush, stream) -> dict:
    """The 3-D path: G1-like humanoid (29 dof, free base) velocity tracking on a rough
    heightfield with the height scan, 4096 worlds, decimation 4, Newton contact solver; one fused launch
    per control step (s3_env_step). Random actions are pre-drawn on the device (inputs resident in HBM).
    Parity is against oracle/sim3d.py (unpinned w.r.t. the reference, which has no 3-D engine)."""
    import torch

    from paper_2601_22074_b200.sim3d import native as native3
    from paper_2601_22074_b200.sim3d import robots
    from paper_2601_22074_b200.sim3d.task import VelocityEnv3D, VelocityTaskCfg

    n = args.envs
    out = {"workload": f"G1-like 3-D humanoid velocity tracking on the 5x6 terrain-curriculum heightfield (levels, "
                       f"height scan, friction randomisation, pushes; mjlab's penalties incl. angular momentum, joint "
                       f"limits, foot slip over per-foot contact sensors), {n} worlds/GPU, decimation 4 (SURVEY 8 f4)",
           "unit": UNIT}
    for dtype in ("f32", "f64"):
        m = robots.g1_like(rough="curriculum", seed=args.seed)
        cfg = VelocityTaskCfg(default_qpos=robots.default_qpos(m, robots.G1_DEFAULT_JOINTS), height_scan=True,
                              curriculum=(5, 6, 8.0))
        env = VelocityEnv3D(m, cfg, n, seed=args.seed, world_offset=int(os.environ.get("RANK", "0")) * n, dtype=dtype)
        env.reset()
        steps = 20
        g = torch.Generator(device="cuda")
        g.manual_seed(args.seed)
        acts = torch.rand(steps + 5, n, m.nu, generator=g, device="cuda", dtype=env.dm.tdtype) * 2 - 1
        for i in range(5):
            env.step(acts[i])
        l0 = native3.LAUNCHES["count"]
        t = timed_steps(env, steps, flush, stream, lambda i: acts[5 + i])
        launches = native3.LAUNCHES["count"] - l0
        out[dtype] = {"value": n * steps / t, "ms_per_step": 1e3 * t / steps, "gpu_launches": launches,
                      "warps_per_block_max": env.dm.layout.warps_per_block,
                      "smem_bytes_per_world": env.dm.layout.elems_per_world * (4 if dtype == "f32" else 8),
                      "terminated_frac_last": float(env.terminated.float().mean().item())}
        del env
    # BASELINE configs[2]: BeyondMimic-style motion imitation (reference-motion command), 8192 worlds/GPU
    from paper_2601_22074_b200.sim3d.motion import synthetic_walk_clip
    from paper_2601_22074_b200.sim3d.task import MotionTrackingCfg

    nm = 2 * n
    out["motion"] = {"workload": f"G1-like 3-D motion imitation (BeyondMimic-style reference-motion command, synthetic "
                                 f"10 s walking clip, RSI with adaptive start-time sampling, relative body pose / "
                                 f"velocity rewards over 14 tracked bodies, self-collision sensor), flat, {nm} "
                                 f"worlds/GPU, decimation 4"}
    for dtype in ("f32", "f64"):
        m = robots.g1_like(seed=args.seed)
        dq = robots.default_qpos(m, robots.G1_DEFAULT_JOINTS)
        Q, V, fdt = synthetic_walk_clip(m, dq)
        cfg = MotionTrackingCfg(default_qpos=dq, motion_qpos=Q, motion_qvel=V, motion_dt=fdt)
        env = VelocityEnv3D(m, cfg, nm, seed=args.seed, world_offset=int(os.environ.get("RANK", "0")) * nm,
                            dtype=dtype)
        env.reset()
        steps = 10
        g = torch.Generator(device="cuda")
        g.manual_seed(args.seed + 1)
        acts = torch.rand(steps + 3, nm, m.nu, generator=g, device="cuda", dtype=env.dm.tdtype) * 2 - 1
        for i in range(3):
            env.step(acts[i])
        t = timed_steps(env, steps, flush, stream, lambda i: acts[3 + i])
        out["motion"][dtype] = {"value": nm * steps / t, "ms_per_step": 1e3 * t / steps}
        del env
    # BASELINE configs[3]: arm cube lift with dense contacts + a palm depth camera rendered every step
    from paper_2601_22074_b200.sim3d.sensors import DepthCamera
    from paper_2601_22074_b200.sim3d.task import LiftTaskCfg

    out["lift"] = {"workload": f"fixed-base 6-dof arm + claw, free cube (2 kinematic trees), cube lift, {n} worlds/GPU, "
                               "decimation 4, + 32x24 palm depth camera rendered every control step"}
    for dtype in ("f32", "f64"):
        m = robots.arm_cube_like()
        cfg = LiftTaskCfg.for_model(m, robots.default_qpos(m, robots.ARM_DEFAULT_JOINTS))
        env = VelocityEnv3D(m, cfg, n, seed=args.seed, world_offset=int(os.environ.get("RANK", "0")) * n, dtype=dtype)
        env.data.enable_geom_frames()
        palm = [g for g in range(m.ngeom) if m.geom_bodyid[g] == m.body_names.index("hand")][0]
        cam = DepthCamera(env.dm, palm, width=32, height=24, fovy=1.2, max_dist=1.0)
        env.reset()

        class _WithDepth:
            def step(self, a, env=env, cam=cam):
                env.step(a)
                cam.render(env.data)

        steps = 10
        g = torch.Generator(device="cuda")
        g.manual_seed(args.seed + 2)
        acts = torch.rand(steps + 3, n, m.nu, generator=g, device="cuda", dtype=env.dm.tdtype) * 2 - 1
        for i in range(3):
            _WithDepth().step(acts[i])
        t = timed_steps(_WithDepth(), steps, flush, stream, lambda i: acts[3 + i])
        t_env = timed_steps(env, steps, flush, stream, lambda i: acts[3 + i])
        out["lift"][dtype] = {"value": n * steps / t, "ms_per_step": 1e3 * t / steps,
                              "env_only_ms_per_step": 1e3 * t_env / steps}
        del env, cam
    out["kernel"] = "s3::env_kernel (warp per world, shared-memory resident; one launch per control step)"
    # the kernel is latency/issue bound with ~0 DRAM traffic (per-world data lives in shared memory), so its
    # evidence is the committed ncu capture, not an HBM roofline
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_sim3d_env_kernel.json")) as fh:
            prof = json.load(fh)
        out["roofline"] = {"bound": "latency (serial per-world factorization/solves in shared memory)",
                           "dram_throughput_frac": prof["f32"]["dram_throughput_frac"],
                           "issue_slots_busy_frac": prof["f32"]["issue_slots_busy_frac"],
                           "executed_ipc_active": prof["f32"]["executed_ipc_active"],
                           "achieved_occupancy_frac": prof["f32"]["achieved_occupancy_frac"],
                           "source": "profiles/ncu_sim3d_env_kernel.json (f32, 4096 worlds)"}
    except (OSError, KeyError, ValueError):
        out["roofline"] = None
    out["parity"] = "oracle/sim3d.py (tests/test_gpu_sim3d*.py); unpinned w.r.t. the reference (no 3-D engine)"
    if not args.no_cpu:
        out["cpu_baseline"] = sim3d_cpu(args.seed)
    return out


def ppo_leg(args, rank: int, world: int) -> dict:
    """BASELINE configs[4]'s "incl. PPO gradient allreduce": the on-device PPO learner (ppo.py) on this
    rank's Velocity-Rough shard -- every minibatch's gradients reduced across ranks as ONE flat bucket
    (NCCL; the minibatch step is one CUDA graph at one rank). Whole-job training env-steps/s over a few
    iterations (collect + update), time = max over ranks."""
    import torch

    from paper_2601_22074_b200.env import ManagerBasedRlEnv
    from paper_2601_22074_b200.ppo import PpoCfg, PpoTrainer
    from paper_2601_22074_b200.tasks import make_env_cfg

    n = args.envs
    cfg = make_env_cfg(args.task, num_envs=n, seed=args.seed)
    cfg.scene.world_id_offset = rank * n
    env = ManagerBasedRlEnv(cfg, args.task)
    tr = PpoTrainer(env, PpoCfg(), seed=args.seed)
    tr.collect()
    tr.update()  # warm-up (graph capture at one rank)
    torch.cuda.synchronize()
    barrier(world)
    iters = 3
    t0 = time.perf_counter()
    st = None
    for _ in range(iters):
        tr.collect()
        st = tr.update()
    torch.cuda.synchronize()
    t = allmax(time.perf_counter() - t0, world)
    steps = iters * tr.cfg.steps_per_env * n * world
    out = {"workload": f"PPO on {args.task}, {n} worlds per GPU, {tr.cfg.steps_per_env} steps x {world} GPU(s) "
                       f"per iteration, MLPs {'-'.join(str(h) for h in tr.cfg.hidden)}",
           "unit": UNIT, "train_env_steps_per_s": steps / t, "iterations": iters,
           "allreduces_per_iter": st["allreduces"], "grad_bucket_floats": tr.reducer.numel,
           "cuda_graph": tr._graph is not None, "collective": "NCCL all_reduce" if world > 1 else "none (1 rank)",
           "parity": "unpinned (the reference has no learner, SPEC.md:509)"}
    del tr, env
    return out


def sim3d_cpu(seed, worlds=4, steps=2) -> dict:
    """The 3-D oracle (numpy, one core) on a bounded sample of the same task."""
    from oracle import sim3d as O
    from paper_2601_22074_b200.sim3d import robots
    from paper_2601_22074_b200.sim3d.task import VelocityTaskCfg

    m = robots.g1_like(rough=True, seed=seed)
    O.set_const(m)
    cfg = VelocityTaskCfg(default_qpos=robots.default_qpos(m, robots.G1_DEFAULT_JOINTS), height_scan=True)
    ref = O.TaskOracle(m, cfg, worlds, seed=seed)
    ref.reset()
    rng = np.random.default_rng(seed)
    t0 = time.perf_counter()
    for _ in range(steps):
        ref.step(rng.uniform(-1, 1, size=(worlds, m.nu)))
    el = time.perf_counter() - t0
    return {"value": worlds * steps / el, "unit": UNIT, "cores": 1, "kind": "port",
            "sample": f"{worlds} worlds x {steps} control steps of the 3-D oracle (numpy float64, 1 process)"}


def run_ours(args):
    import torch

    import __graft_entry__

    rank, world, local = dist_setup(args.gpus)
    if world == 1 and args.gpus > 1:
        raise SystemExit("--gpus N > 1 needs one process per GPU (bench.py self-launches them when WORLD_SIZE is unset)")
    if rank == 0:
        __graft_entry__.build()
    barrier(world)
    from paper_2601_22074_b200 import native
    from paper_2601_22074_b200.env import ManagerBasedRlEnv
    from paper_2601_22074_b200.metrics import allreduce_stats, build_record, unpack_stats
    from paper_2601_22074_b200.policies import random_policy
    from paper_2601_22074_b200.tasks import make_env_cfg
    from paper_2601_22074_b200.traffic import step_bytes_per_world

    n = args.envs
    cfg = make_env_cfg(args.task, num_envs=n, seed=args.seed)
    cfg.scene.world_id_offset = rank * n  # rank r owns worlds [r*N, (r+1)*N) (env.py:67-69, :114)
    env = ManagerBasedRlEnv(cfg, args.task)
    env.reset()
    stream = torch.cuda.current_stream()
    flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")

    # clocks sampler: started ahead of the warm-up so its start-up queries are over when the timed region begins
    clocks = Clocks(local)
    time.sleep(0.5)
    # the benchmark loop of the reference (cli.py:163): env.step(random_policy(env));
    # fused=True draws the same actions (stream policy.random) inside the step kernel
    for i in range(args.warmup):
        env.step(random_policy(env, i, fused=True))
    build_record(env, 0, env.reward_manager.reward, None)  # warm the stats kernel and the collective
    env._stats_packer.request()  # and the fused statistics tail of the step kernel
    env.step(random_policy(env, args.warmup, fused=True))
    torch.cuda.synchronize()

    # every log interval (cli.py:118, --log-every 10) the job's statistics are
    # reduced across ranks inside the timed step: the step kernel itself reduces
    # this rank's reward / episodic sums / trigger counts / terrain-row
    # histogram / nonfinite count into one vector in its tail (StatsPacker.request,
    # no extra launch), one all_reduce (NCCL) sums it over ranks; the records are
    # unpacked on the host after the timed region
    vecs = []
    n_rec = args.steps // args.log_every if args.log_every > 0 else 0
    rec_bufs = [torch.zeros_like(env._stats_packer.out) for _ in range(n_rec)]

    def log_request(i):
        if args.log_every > 0 and (i + 1) % args.log_every == 0:
            env._stats_packer.request(rec_bufs[len(vecs)])

    def log_interval(i):
        if args.log_every > 0 and (i + 1) % args.log_every == 0:
            vecs.append((i + 1, allreduce_stats(rec_bufs[len(vecs)])))

    barrier(world)
    launches0 = native.LAUNCHES["count"]
    t_step = timed_steps(env, args.steps, flush, stream, lambda i: random_policy(env, args.warmup + i, fused=True),
                         after=log_interval, before=log_request)
    barrier(world)
    launches = native.LAUNCHES["count"] - launches0
    t_max = allmax(t_step, world)
    value = n * world * args.steps / t_max
    rm, tm = env.reward_manager, env.termination_manager
    records = [unpack_stats(v, list(rm.terms), list(tm.trigger_counts), env.terrain.rows, st).__dict__
               for st, v in vecs]

    # roofline of the dominant kernel (the fused step), timed on its own
    # (the log-interval reduction excluded) with the same flush protocol
    t_kernel = timed_steps(env, args.steps, flush, stream,
                           lambda i: random_policy(env, args.warmup + args.steps + i, fused=True))
    per_world = step_bytes_per_world(env, fused_policy=True)
    peak, peak_kind = _peaks()
    achieved = per_world["total"] * n / (t_kernel / args.steps) / 1e9
    traffic, traffic_envs = _ncu_traffic()
    if traffic is not None and traffic_envs not in (None, n):
        traffic = None

    # end-to-end through the public API with host buffers (gym VectorEnv-style
    # step_async / step_wait): each step's actions are copied from pinned host
    # memory to the device by a copy engine ahead of the step kernel; its
    # results (obs groups, reward, terminated, truncated: the whole output
    # arena) are snapshotted on the device and copied into pinned host memory
    # by a second copy engine, overlapping the next step's kernel; step_wait()
    # blocks until a step's results are in host memory. Every step's inputs
    # and outputs cross PCIe inside the timed region; the last step is waited
    # for before the clock stops.
    A = env.action_manager.total_dim
    rng = np.random.default_rng(rank)
    e2e_steps = 0 if args.no_e2e else max(args.steps, 200)  # tens of us each: a longer sample smooths jitter
    host_actions = torch.from_numpy(rng.uniform(-1, 1, size=(e2e_steps, n, A))).pin_memory()
    checksum = 0.0
    # warm-up (untimed): three full passes over the pinned host buffers the timed pass will use -- the
    # pipe reaches its steady rate only after a few hundred steps (tools/e2e_ab.py: 200-step passes at
    # 39 / 34 / 32 / 32 us per step), as a training loop's reused buffers are past after its first iterations
    from paper_2601_22074_b200.env import PIPE_SLOTS

    for _ in range(3):
        for i in range(e2e_steps):
            env.step_async(host_actions[i])
            if i >= PIPE_SLOTS - 1:
                env.step_wait()
        for _ in range(min(PIPE_SLOTS - 1, e2e_steps)):
            env.step_wait()
    barrier(world)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for i in range(e2e_steps):
        env.step_async(host_actions[i])
        if i >= PIPE_SLOTS - 1:
            checksum += float(env.step_wait()["reward"][0])
    host_views = None
    for _ in range(min(PIPE_SLOTS - 1, e2e_steps)):
        host_views = env.step_wait()
    e2e_t = allmax(time.perf_counter() - t0, world)
    assert host_views is None or (host_views["reward"].shape == (n,) and host_views["reward"].device.type == "cpu")
    e2e = None if not e2e_steps else {
        "value": n * world * e2e_steps / e2e_t, "unit": UNIT, "steps": e2e_steps, "h2d_bytes_per_step": n * A * 8,
        "d2h_bytes_per_step": int(env.step_outputs.numel()),
        "path": "pinned host actions -> env.step_async (H2D cudaMemcpyAsync on a copy-engine stream, the step "
                "kernel waits on it; the output arena is snapshotted D2D and copied to pinned host memory on a "
                "second copy-engine stream -- two consecutive steps' arenas per copy once both are submitted -- "
                "overlapping the next steps) -> env.step_wait (results in host memory)"}

    scale = at_scale(args, flush, stream) if (world == 1 and args.scale_envs > 0) else None
    s3 = None if args.no_sim3d else sim3d_leg(args, flush, stream)
    ppo = None if args.no_ppo else ppo_leg(args, rank, world)
    # the headline region lasts ~1 ms (shorter than nvidia-smi's 100 ms period): the sampler runs from just
    # before it through the e2e, at-scale and 3-D legs, so its samples are of the GPU under this load
    clk = clocks.stop()
    clk["window"] = "warm-up and headline timed region through the e2e, at-scale and 3-D legs"
    if s3 is not None:
        for blk in (s3, s3["motion"], s3["lift"]):
            for k in ("f32", "f64"):
                blk[k]["value"] = blk[k]["value"] * world  # whole job: every rank steps its shard (weak scaling)
                blk[k]["ms_per_step"] = allmax(blk[k]["ms_per_step"], world)

    offsets = [rank * n]
    if world > 1:
        import torch.distributed as dist

        got = [None] * world
        dist.all_gather_object(got, rank * n)
        offsets = got
    if rank == 0:
        cpu = None
        if world == 1 and not args.no_cpu:
            cpu = measure_cpu(args.task, n, seconds=args.cpu_seconds)
        line = {
            "metric": METRIC,
            "value": value,
            "unit": UNIT,
            "n_gpus": world,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": 1e3 * t_max / args.steps,
            "higher_is_better": True,
            "scaling": "weak",
            "vs_baseline": None,
            "dtype": "f64",
            "data": "synthetic (random actions from the per-world device streams; random-init env, no checkpoint)",
            "config": bench_config(args.task, n, world),
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "peak_kind": peak_kind, "traffic": traffic,
                         "algorithmic_bytes_per_env_step": per_world["total"],
                         "kernel": "ss_step_jit (fused control step, per-env NVRTC specialization)"
                         if env.use_jit else "step_kernel<4,2> (fused control step, generic)",
                         "kernel_ms": 1e3 * t_kernel / args.steps},
            "policy": "random_policy fused into the step kernel (policies.RandomActions: same stream and values)",
            "stats_allreduce": {"every_steps": args.log_every, "per_interval": "the job statistics reduced in the step "
                                "kernel's tail (fused, no extra launch) + 1 all_reduce "
                                f"({'NCCL' if world > 1 else 'no-op at 1 rank'}) of {int(env._stats_packer.out.numel())} "
                                "float64, inside the timed step", "records": len(records),
                                "last": records[-1] if records else None},
            "shards": {"world_id_offsets": offsets, "envs_per_rank": n},
            "at_scale": scale,
            "sim3d": s3,
            "ppo": ppo,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": launches,
            "clocks": clk,
        }
    if world > 1:
        import torch.distributed as dist

        dist.barrier()
        dist.destroy_process_group()
    if rank == 0:
        print(json.dumps(line), flush=True)  # last: after the communicator's teardown messages


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    # the whole job of our arm: envs per GPU x GPUs (weak scaling), on the host cores
    world = int(os.environ.get("WORLD_SIZE", str(max(1, args.gpus))))
    n = args.envs * world
    runs = {}
    for kind in (["reference", "port"] if reference_available() else ["port"]):
        pool = CpuBaseline(args.task, n, kind=kind)
        try:
            pool.run(max(1, args.warmup))
            el = pool.run(args.steps)
        finally:
            pool.close()
        runs[kind] = {"value": n * args.steps / el, "unit": UNIT, "cores": pool.procs, "kind": kind,
                      "ms_per_step": 1e3 * el / args.steps,
                      "sample": f"{args.task} N={n} over {pool.procs} host processes (world_id_offset shards), "
                                f"{args.steps} control steps after {max(1, args.warmup)} warm-up steps, random "
                                f"actions, {_describe(kind)}, CPU {cpu_model_name()}"}
    head = runs.get("reference") or runs["port"]
    v = head["value"]
    line = {
        "metric": METRIC,
        "value": v,
        "unit": UNIT,
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": head["ms_per_step"],
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic (random actions from the per-world streams)",
        "config": bench_config(args.task, args.envs, world),
        "impl": "reference",
        "cpu_baseline": {k: head[k] for k in ("value", "unit", "cores", "kind", "sample")},
        "beside": {k: r for k, r in runs.items() if r is not head},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def run_dry(args):
    """--dry-cpu: the multi-rank plumbing of run_ours on CPU (gloo), for tests:
    each rank steps its world shard (oracle env, world_id_offset = rank * N)
    and the job's stats are reduced with the same pack / all_reduce / unpack
    path; rank 0 prints the shard offsets and the reduced record."""
    rank, world, _ = dist_setup(args.gpus, backend="gloo")
    import torch

    from oracle import OracleEnv
    from paper_2601_22074_b200.metrics import allreduce_stats, pack_stats, unpack_stats
    from paper_2601_22074_b200.tasks import make_env_cfg
    from paper_2601_22074_b200.terrain import generate_grid

    n = args.envs
    cfg = make_env_cfg(args.task, num_envs=n, seed=args.seed)
    cfg.scene.world_id_offset = rank * n
    env = OracleEnv(cfg, generate_grid(cfg.scene.terrain, cfg.seed).samples)
    env.reset()
    steps = args.warmup + args.steps
    for _ in range(steps):
        _, rew, *_ = env.step(env.random_actions())
    vec = pack_stats(torch.from_numpy(rew), [torch.from_numpy(env.ep_sums[k]) for k in env.rw],
                     torch.tensor(list(env.trigger_counts.values())), torch.from_numpy(env.terrain_rows),
                     env.t_rows, torch.from_numpy(env.last_nonfinite))
    vec = allreduce_stats(vec)
    rec = unpack_stats(vec, list(env.rw), list(env.trigger_counts), env.t_rows, steps)
    offsets = [rank * n]
    if world > 1:
        import torch.distributed as dist

        offsets = [None] * world
        dist.all_gather_object(offsets, rank * n)
    if rank == 0:
        print(json.dumps({"dry": True, "n_gpus": world, "config": bench_config(args.task, n, world),
                          "shards": {"world_id_offsets": offsets, "envs_per_rank": n}, "steps": steps,
                          "record": rec.__dict__}), flush=True)
    if world > 1:
        import torch.distributed as dist

        dist.destroy_process_group()


def self_launch(argv) -> int:
    """bench.py --gpus N with no WORLD_SIZE in the environment: start N ranks
    (one process per GPU) through torch.distributed.run on this node and
    relay their output (rank 0 prints the JSON line)."""
    import socket

    sock = socket.socket()
    sock.bind(("127.0.0.1", 0))
    port = sock.getsockname()[1]
    sock.close()
    gpus = None
    for i, a in enumerate(argv):
        if a == "--gpus":
            gpus = int(argv[i + 1])
        elif a.startswith("--gpus="):
            gpus = int(a.split("=", 1)[1])
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")  # communicator setup (rank count, NVLS / NVLink transport) ...
    env.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")  # ... on stderr: stdout is the JSON line
    env.setdefault("OMP_NUM_THREADS", "1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__), *argv]
    return subprocess.call(cmd, env=env)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--envs", type=int, default=4096)
    ap.add_argument("--task", default="Velocity-Rough")
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--log-every", type=int, default=10,
                    help="steps between stats all-reduces inside the timed loop (cli.py --log-every; 0 disables)")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-e2e", action="store_true", help="skip the end-to-end leg (profiling runs)")
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--no-sim3d", action="store_true", help="skip the 3-D (SURVEY 8 f4) leg")
    ap.add_argument("--no-ppo", action="store_true", help="skip the PPO training leg (SURVEY 8 f2)")
    ap.add_argument("--dry-cpu", action="store_true", help="multi-rank plumbing on CPU (gloo + oracle), for tests")
    ap.add_argument("--scale-envs", type=int, default=262144,
                    help="also time the step at this many worlds (HBM-bound regime); 0 disables")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "ours" and args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        if not args.dry_cpu:
            import torch

            if torch.cuda.device_count() < args.gpus:
                raise SystemExit(f"--gpus {args.gpus}: only {torch.cuda.device_count()} CUDA devices visible")
        raise SystemExit(self_launch(sys.argv[1:]))
    if args.impl == "reference":
        run_reference(args)
    elif args.dry_cpu:
        run_dry(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
