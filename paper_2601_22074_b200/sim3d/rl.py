"""Adapter exposing a fused 3-D env (task.VelocityEnv3D) through the manager-style surface the
on-device PPO learner uses (ppo.PpoTrainer: observation_manager.group_dim / groups,
action_manager.total_dim, reset() -> {"policy": obs}, step(a) -> (obs dict, reward, terminated,
truncated, extras)). BASELINE configs[4]'s "incl. PPO gradient allreduce" on the 3-D G1."""

from __future__ import annotations

import torch


class _Obs:
    def __init__(self, dim: int):
        self.groups = {"policy": dim}

    def group_dim(self, group: str) -> int:
        return self.groups[group]


class _Act:
    def __init__(self, dim: int):
        self.total_dim = dim


class ManagerView:
    def __init__(self, env):
        self.env = env
        self.num_envs = env.num_envs
        self.device = env.dm.device
        self.observation_manager = _Obs(env.obs_dim)
        self.action_manager = _Act(env.model.nu)

    def reset(self):
        return {"policy": self.env.reset()}

    def step(self, actions: torch.Tensor):
        obs, rew, term, trunc = self.env.step(actions.to(self.env.dm.tdtype))
        return {"policy": obs}, rew, term.bool(), trunc.bool(), {}
