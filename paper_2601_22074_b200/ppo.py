"""On-device PPO learner with a single flat gradient all-reduce per minibatch.

SURVEY §8f row 2 / BASELINE configs[4] ("... incl. PPO gradient
allreduce"). The reference has no learner (mjlab uses RSL-RL,
PAPER.md:240), so this is an addition without an oracle: parity is unpinned,
the tests check the distributed gradient algebra instead.

Design: rollouts stay on the GPU (observations come straight from the env's
output buffers, cast to float32 once); the actor-critic is two small MLPs
(cuBLAS GEMMs -- library code, not the hot path of this repo -- in bf16 on the
tensor cores during the update, distribution math in float32); parameters
and gradients live in two flat float32 buffers, so after each minibatch
backward the gradients already form ONE contiguous bucket, reduced in place
with a single all_reduce (NCCL over NVLink between GPUs, gloo in CPU tests),
i.e. one latency-bound collective of ~1.4 MB per minibatch instead of one per
parameter tensor; fused Adam.
"""

from __future__ import annotations

from dataclasses import dataclass

import torch
import torch.distributed as dist
from torch import nn


@dataclass
class PpoCfg:
    hidden: tuple[int, ...] = (512, 256, 128)
    steps_per_env: int = 24
    epochs: int = 5
    minibatches: int = 4
    lr: float = 1e-3
    gamma: float = 0.99
    lam: float = 0.95
    clip: float = 0.2
    value_coef: float = 1.0
    entropy_coef: float = 0.01
    max_grad_norm: float = 1.0
    init_std: float = 1.0
    cuda_graph: bool = True  # capture the minibatch step (forward, backward, all-reduce, clip, Adam) once


def _mlp(n_in: int, hidden, n_out: int) -> nn.Sequential:
    layers, d = [], n_in
    for h in hidden:
        layers += [nn.Linear(d, h), nn.ELU()]
        d = h
    layers.append(nn.Linear(d, n_out))
    return nn.Sequential(*layers)


class ActorCritic(nn.Module):
    def __init__(self, n_policy_obs: int, n_critic_obs: int, n_actions: int, cfg: PpoCfg):
        super().__init__()
        self.actor = _mlp(n_policy_obs, cfg.hidden, n_actions)
        self.critic = _mlp(n_critic_obs, cfg.hidden, 1)
        self.log_std = nn.Parameter(torch.full((n_actions,), float(torch.log(torch.tensor(cfg.init_std)))))

    def dist(self, obs_p):
        mean = self.actor(obs_p).float()  # distribution math in float32 (the GEMMs may run in bf16)
        # validate_args=False: argument validation is a data-dependent check that
        # synchronizes the device on every call
        return torch.distributions.Normal(mean, self.log_std.exp().expand_as(mean), validate_args=False)

    def value(self, obs_c):
        return self.critic(obs_c).squeeze(-1).float()


class FlatGradReducer:
    """All gradients of a module in one contiguous bucket, one collective.

    At construction the module's parameters and gradients are re-pointed into
    two flat float32 buffers (``flat_param`` / ``bucket``; each ``p.data`` /
    ``p.grad`` becomes a view), so backward accumulates straight into the
    bucket: ``reduce`` is a single in-place all_reduce (no gather / scatter
    copies), ``zero_grad`` one fill, the gradient norm one reduction."""

    def __init__(self, module: nn.Module, group=None):
        self.params = [p for p in module.parameters() if p.requires_grad]
        self.numel = sum(p.numel() for p in self.params)
        self.group = group
        dev = self.params[0].device
        self.flat_param = torch.empty(self.numel, dtype=torch.float32, device=dev)
        self.bucket = torch.zeros(self.numel, dtype=torch.float32, device=dev)
        off = 0
        for p in self.params:
            n = p.numel()
            self.flat_param[off : off + n].copy_(p.data.reshape(-1))
            p.data = self.flat_param[off : off + n].view_as(p)
            g = self.bucket[off : off + n].view_as(p)
            if p.grad is not None:
                g.copy_(p.grad)
            p.grad = g
            off += n

    @property
    def world(self) -> int:
        return dist.get_world_size(self.group) if dist.is_available() and dist.is_initialized() else 1

    def zero_grad(self) -> None:
        self.bucket.zero_()

    def reduce(self) -> None:
        if self.world > 1:
            dist.all_reduce(self.bucket, op=dist.ReduceOp.SUM, group=self.group)
            self.bucket.div_(self.world)

    def clip_(self, max_norm: float) -> None:
        """clip_grad_norm_ over the bucket: one norm, one scale, no host sync."""
        norm = torch.linalg.vector_norm(self.bucket)
        self.bucket.mul_(torch.clamp(max_norm / (norm + 1e-6), max=1.0))


def broadcast_parameters(module: nn.Module, group=None) -> None:
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        for p in module.parameters():
            dist.broadcast(p.data, src=0, group=group)


def gae(rewards, values, dones, last_value, gamma: float, lam: float):
    """Generalized advantage estimation over a (T, N) rollout."""
    T = rewards.shape[0]
    adv = torch.zeros_like(rewards)
    last = torch.zeros_like(last_value)
    for t in reversed(range(T)):
        next_v = last_value if t == T - 1 else values[t + 1]
        nonterm = 1.0 - dones[t]
        delta = rewards[t] + gamma * next_v * nonterm - values[t]
        last = delta + gamma * lam * nonterm * last
        adv[t] = last
    return adv, adv + values


def normalize_advantages(adv, group=None):
    """(adv - mean) / std with the mean and variance of the WHOLE job: data-parallel ranks all-reduce
    [sum, sum of squares, count] (one 3-float collective) so every rank normalizes identically."""
    st = torch.stack([adv.sum(), (adv * adv).sum(), torch.tensor(float(adv.numel()), device=adv.device)])
    st = st.double()
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(st, op=dist.ReduceOp.SUM, group=group)
    n = st[2]
    mean = st[0] / n
    var = (st[1] - n * mean * mean) / (n - 1).clamp(min=1.0)  # unbiased, like torch.std
    return ((adv.double() - mean) / (var.clamp(min=0.0).sqrt() + 1e-8)).to(adv.dtype)


def ppo_loss(model: ActorCritic, cfg: PpoCfg, obs_p, obs_c, actions, old_logp, adv, ret):
    d = model.dist(obs_p)
    logp = d.log_prob(actions).sum(-1)
    ratio = torch.exp(logp - old_logp)
    s1 = ratio * adv
    s2 = torch.clamp(ratio, 1.0 - cfg.clip, 1.0 + cfg.clip) * adv
    v = model.value(obs_c)
    return -torch.min(s1, s2).mean() + cfg.value_coef * (ret - v).pow(2).mean() - cfg.entropy_coef * d.entropy().sum(-1).mean()


class PpoTrainer:
    """Collect `steps_per_env` control steps from a ManagerBasedRlEnv, then update."""

    def __init__(self, env, cfg: PpoCfg | None = None, group=None, seed: int = 0):
        self.env = env
        self.cfg = cfg or PpoCfg()
        om = env.observation_manager
        self.n_p = om.group_dim("policy")
        self.n_c = om.group_dim("critic") if "critic" in om.groups else self.n_p
        self.n_a = env.action_manager.total_dim
        torch.manual_seed(seed)
        self.model = ActorCritic(self.n_p, self.n_c, self.n_a, self.cfg).to(env.device)
        broadcast_parameters(self.model, group)
        self.reducer = FlatGradReducer(self.model, group)  # parameters / gradients -> flat buffers
        fused = env.device.type == "cuda"
        # one rank only: the multi-rank step keeps eager launches (collective capture not exercised here)
        self.use_graph = fused and self.cfg.cuda_graph and self.reducer.world == 1
        self.opt = torch.optim.Adam(self.model.parameters(), lr=self.cfg.lr, fused=fused,
                                    capturable=self.use_graph)
        self.amp = fused  # bf16 GEMMs on the tensor cores in the update's forward / backward
        self._graph = None
        T, n = self.cfg.steps_per_env, env.num_envs
        dev = env.device
        self.buf = {
            "obs_p": torch.zeros((T, n, self.n_p), device=dev),
            "obs_c": torch.zeros((T, n, self.n_c), device=dev),
            "act": torch.zeros((T, n, self.n_a), device=dev),
            "logp": torch.zeros((T, n), device=dev),
            "val": torch.zeros((T, n), device=dev),
            "rew": torch.zeros((T, n), device=dev),
            "done": torch.zeros((T, n), device=dev),
        }
        self.obs = None

    def _split(self, obs):
        p = obs["policy"].float()
        c = obs["critic"].float() if "critic" in obs else p
        return p, c

    @torch.no_grad()
    def collect(self) -> None:
        env, b = self.env, self.buf
        if self.obs is None:
            self.obs = env.reset()
        for t in range(self.cfg.steps_per_env):
            p, c = self._split(self.obs)
            d = self.model.dist(p)
            a = d.sample()
            b["obs_p"][t], b["obs_c"][t], b["act"][t] = p, c, a
            b["logp"][t] = d.log_prob(a).sum(-1)
            b["val"][t] = self.model.value(c)
            self.obs, rew, term, trunc, _ = env.step(a.double())
            # episode boundary for GAE; a time-limit truncation is not a terminal state, so its reward
            # bootstraps gamma * V (the value of the state the last action was taken in, the pre-reset
            # estimate available once the env has auto-reset; rsl_rl's time_outs treatment)
            b["rew"][t] = rew.float() + self.cfg.gamma * b["val"][t] * (trunc & ~term).float()
            b["done"][t] = (term | trunc).float()

    def _minibatch_step(self) -> None:
        """One minibatch: forward (bf16 GEMMs), backward into the flat bucket, the bucket's single
        all-reduce, clip, Adam -- on the static buffers (self._mb_idx selects the samples)."""
        cfg, fl, idx = self.cfg, self._flat, self._mb_idx
        with torch.autocast("cuda", dtype=torch.bfloat16, enabled=self.amp):
            loss = ppo_loss(self.model, cfg, fl["obs_p"][idx], fl["obs_c"][idx], fl["act"][idx], fl["logp"][idx],
                            self._adv[idx], self._ret[idx])
        self.reducer.zero_grad()
        loss.backward()
        self.reducer.reduce()
        self.reducer.clip_(cfg.max_grad_norm)
        self.opt.step()
        self._mb_loss.copy_(loss.detach())

    def _ensure_static(self, T: int, n: int, mb: int) -> None:
        if getattr(self, "_flat", None) is not None:
            return
        b = self.buf
        self._flat = {k: v.reshape(T * n, *v.shape[2:]) for k, v in b.items()}  # views of the rollout buffers
        dev = b["rew"].device
        self._adv = torch.zeros(T * n, device=dev)
        self._ret = torch.zeros(T * n, device=dev)
        self._mb_idx = torch.zeros(mb, dtype=torch.int64, device=dev)
        self._mb_loss = torch.zeros((), device=dev)

    def _capture(self) -> None:
        """Record the minibatch step as one CUDA graph (after warm-up iterations on a side stream, as
        graph capture requires): a minibatch then costs one graph launch instead of ~100 kernel launches
        from Python -- the update was launch-bound."""
        saved = self.reducer.flat_param.clone()  # the warm-up steps must not train: restore after them
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            for _ in range(3):
                self._minibatch_step()
        torch.cuda.current_stream().wait_stream(s)
        self._graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self._graph):
            self._minibatch_step()
        # back to the state before the warm-up: the parameters, and Adam's moments and step (created by
        # the warm-up -- the graph is recorded at the first update -- so zero is their initial value)
        self.reducer.flat_param.copy_(saved)
        for p, st in self.opt.state.items():
            for k, v in st.items():
                if torch.is_tensor(v):
                    v.zero_()

    def update(self) -> dict:
        cfg, b = self.cfg, self.buf
        T, n = b["rew"].shape
        mb = (T * n) // cfg.minibatches
        self._ensure_static(T, n, mb)
        with torch.no_grad():
            _, c = self._split(self.obs)
            adv, ret = gae(b["rew"], b["val"], b["done"], self.model.value(c), cfg.gamma, cfg.lam)
            adv = normalize_advantages(adv, self.reducer.group)
            self._adv.copy_(adv.reshape(-1))
            self._ret.copy_(ret.reshape(-1))
        stats = {"loss": 0.0, "allreduces": 0}
        for _ in range(cfg.epochs):
            perm = torch.randperm(T * n, device=self._adv.device)
            for m in range(cfg.minibatches):
                self._mb_idx.copy_(perm[m * mb : (m + 1) * mb])
                if self.use_graph:
                    if self._graph is None:
                        self._capture()
                    self._graph.replay()
                else:
                    self._minibatch_step()
                stats["allreduces"] += 1
        stats["loss"] = float(self._mb_loss) if stats["allreduces"] else 0.0  # one host sync per update
        return stats
