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
