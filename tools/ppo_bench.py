"""PPO training throughput on the B200 env (BASELINE configs[4]: env scaling
incl. the PPO gradient all-reduce). One process per GPU under torchrun;
env-steps/s of collection+update, the all-reduce time share, mean reward."""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2601_22074_b200.env import ManagerBasedRlEnv  # noqa: E402
from paper_2601_22074_b200.ppo import PpoCfg, PpoTrainer  # noqa: E402
from paper_2601_22074_b200.tasks import make_env_cfg  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--envs", type=int, default=4096)
ap.add_argument("--iters", type=int, default=10)
ap.add_argument("--task", default="Velocity-Rough",
                help="planar task id, or G1-3D / G1-3D-Rough for the fused 3-D G1 velocity task (float32)")
args = ap.parse_args()
rank, world = int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))
torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", 0)))
if world > 1:
    dist.init_process_group("nccl", device_id=torch.device("cuda", torch.cuda.current_device()))
if args.task.startswith("G1-3D"):
    from paper_2601_22074_b200.sim3d import robots
    from paper_2601_22074_b200.sim3d.rl import ManagerView
    from paper_2601_22074_b200.sim3d.task import VelocityEnv3D, VelocityTaskCfg

    rough = args.task.endswith("Rough")
    m = robots.g1_like(rough=rough)
    tcfg = VelocityTaskCfg(default_qpos=robots.default_qpos(m, robots.G1_DEFAULT_JOINTS), height_scan=rough)
    env = ManagerView(VelocityEnv3D(m, tcfg, args.envs, world_offset=rank * args.envs, dtype="f32"))
else:
    cfg = make_env_cfg(args.task, num_envs=args.envs)
    cfg.scene.world_id_offset = rank * args.envs
    env = ManagerBasedRlEnv(cfg, args.task)
tr = PpoTrainer(env, PpoCfg())
tr.collect()
tr.update()
torch.cuda.synchronize()
t_col = t_upd = 0.0
rewards = []
for it in range(args.iters):
    t0 = time.perf_counter()
    tr.collect()
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    st = tr.update()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    t_col += t1 - t0
    t_upd += t2 - t1
    rewards.append(float(tr.buf["rew"].mean()))
steps = args.iters * tr.cfg.steps_per_env * args.envs * world
if rank == 0:
    print(json.dumps({"task": args.task, "envs_per_gpu": args.envs, "gpus": world,
                      "train_env_steps_per_s": steps / (t_col + t_upd),
                      "collect_env_steps_per_s": steps / t_col, "collect_s": t_col, "update_s": t_upd,
                      "grad_bucket_floats": tr.reducer.numel, "allreduces_per_iter": st["allreduces"],
                      "mean_reward_first_last": [rewards[0], rewards[-1]]}))
if world > 1:
    dist.destroy_process_group()
