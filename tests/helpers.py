"""Shared test helpers: golden fixtures, config rebuild, specs."""

import json
import os

import numpy as np

from paper_2601_22074_b200 import config as C
from paper_2601_22074_b200.terrain import generate_grid

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def golden(name: str):
    return np.load(os.path.join(GOLDEN, name), allow_pickle=False)


def cfg_from_golden(g) -> C.EnvCfg:
    return C.from_dict(C.EnvCfg, json.loads(str(g["cfg_json"])))


def spec_from_json(s) -> C.ModelSpec:
    return C.from_dict(C.ModelSpec, json.loads(str(s)))


def samples_for(cfg):
    return generate_grid(cfg.scene.terrain, cfg.seed).samples


def pendulum_spec(**over) -> C.ModelSpec:
    kw = dict(name="pendulum", base_mass=8.0, base_inertia=0.15,
              joints=[C.JointSpec(name="leg", parent=-1, attach_offset=(0.0, 0.0), link_length=0.5,
                                  link_mass=0.5, rotor_inertia=0.02, damping=0.2)],
              feet=[0])
    kw.update(over)
    return C.ModelSpec(**kw)


def two_leg_spec() -> C.ModelSpec:
    joints = []
    for side, hx in (("l", -0.1), ("r", 0.1)):
        h = len(joints)
        joints.append(C.JointSpec(name=f"{side}_hip", parent=-1, attach_offset=(hx, 0.0), link_length=0.25))
        joints.append(C.JointSpec(name=f"{side}_knee", parent=h, attach_offset=(0.0, -0.25), link_length=0.25))
    return C.ModelSpec(name="biped", joints=joints, feet=[1, 3])


def sync_from_oracle(env, ref, world_start=None):
    """Teacher forcing: copy every floating-point state array of the oracle env
    into the GPU env (discrete state -- counters, RNG counters, flags -- evolves
    identically on both sides as long as the flags match, which the tests
    assert). After this the next step starts from bit-identical state.

    With ``world_start`` the oracle holds only worlds [world_start,
    world_start + ref.n) of the GPU env (built with world_id_offset =
    world_start, partition-independent per SPEC.md:113): every array is
    written into that slice of its world axis."""
    import torch

    dev = env.device
    N = env.num_envs

    def put(dst, src):
        if world_start is not None:
            axes = [i for i, s in enumerate(dst.shape) if s == N]
            assert len(axes) == 1, (tuple(dst.shape), N)
            dst = dst.narrow(axes[0], world_start, ref.n)
        dst.copy_(torch.as_tensor(np.array(src, copy=True), device=dev).to(dst.dtype).reshape(dst.shape))

    S = ref.S
    st = env.state
    put(st.q, S["q"])
    put(st.qd, S["qd"])
    put(st.ctrl, S["ctrl"])
    put(st.ext_force, S["ext"])
    put(st.time, S["time"])
    c = st.contact
    put(c.normal_force, S["fn"])
    put(c.tangent_force, S["ft"])
    put(c.foot_pos, S["fpos"])
    put(c.foot_vel, S["fvel"])
    put(c.in_contact, S["fin"])
    cs, z = env.contact_sensor, ref.sens
    put(cs.in_contact, z["in"])
    put(cs.normal_force, z["normal"])
    put(cs.tangent_force, z["tangent"])
    put(cs.force_history, z["hist"])
    put(cs.current_air_time, z["air"])
    put(cs.last_air_time, z["last_air"])
    put(cs.current_contact_time, z["contact"])
    put(cs.last_touchdown_step, z["td"])
    rm = env.reward_manager
    for name in rm.terms:
        put(rm.episodic_sums[name], ref.ep_sums[name])
        put(rm.episodic_raw[name], ref.ep_raw[name])
    put(env.prev_lin_vel_b, ref.prev_lin_vel_b)
    put(env.episode_start_x, ref.episode_start_x)
    put(env.commanded_distance, ref.commanded_distance)
    put(env.command_manager.command, ref.command)
    put(env.command_manager.ranges, ref.ranges)
    am = env.action_manager
    put(am.action, ref.action)
    put(am.prev_action, ref.prev_action)
    put(am.targets, ref.targets)
    for name in env.model.field_names():
        f = env.model.field(name)
        v = ref.m.fields[name][0]
        if f.expanded:
            shape = tuple(f.value.shape)
            if world_start is not None:
                shape = tuple(ref.n if s == N else s for s in shape)
            put(f.value, np.broadcast_to(v, shape))
    for k, el in ref.ev_elapsed.items():
        put(env.event_manager._elapsed[k], el)
        put(env.event_manager._target[k], ref.ev_target[k])
    # observation rings: same head convention for delay rings; history is a
    # ring with the newest entry at hist_head (the oracle shifts physically)
    for g, (gc, terms) in ref.groups.items():
        for mine, t in zip(env.observation_manager.groups[g], terms):
            if mine._dring is not None:
                put(mine._dring, np.transpose(t["dring"], (0, 2, 1)))
            if mine._hring is not None:
                H = mine.cfg.history
                for i in range(H):
                    slot = (mine.hist_head + 1 + i) % H
                    put(mine._hring[slot], t["hring"][i].T)
