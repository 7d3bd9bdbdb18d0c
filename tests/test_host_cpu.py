"""CPU-only checks: the C-ABI library, config/spec host logic, host RNG."""

import json
import re

import numpy as np
import pytest

from helpers import golden, pendulum_spec, two_leg_spec
from paper_2601_22074_b200 import config as C


def test_library_loads_and_exports_every_declared_symbol():
    from paper_2601_22074_b200 import native

    so = native.lib()
    text = open(native.HEADER).read()
    declared = set(re.findall(r"^\s*(?:int|size_t|const char\*)\s+(ss_\w+)\s*\(", text, flags=re.M))
    assert declared == set(native.EXPORTED), declared ^ set(native.EXPORTED)
    for name in declared:
        assert hasattr(so, name), name
    assert so.ss_abi_version() == native.SS_ABI_VERSION


def test_header_struct_layouts_match_the_library():
    import ctypes

    from paper_2601_22074_b200 import native

    so = native.lib()
    assert so.ss_sizeof(0) == ctypes.sizeof(native.EnvDesc)
    assert so.ss_sizeof(1) == ctypes.sizeof(native.Uniforms)
    assert so.ss_sizeof(2) == ctypes.sizeof(native.RngDrawArgs)
    assert ctypes.sizeof(native.EnvDesc) < 32764  # fits a kernel parameter block


@pytest.mark.parametrize("task,fixture", [("Velocity-Flat", "rollout_flat.npz"), ("Velocity-Rough", "rollout_rough.npz")])
def test_task_configs_identical_to_reference(task, fixture):
    from paper_2601_22074_b200.tasks import make_env_cfg

    g = golden(fixture)
    ref = json.loads(str(g["cfg_json"]))
    mine = make_env_cfg(task, num_envs=ref["scene"]["num_envs"], seed=ref["seed"])
    assert C.to_dict(mine) == ref
    assert C.config_hash(mine) == str(g["config_hash"])


def test_unknown_task_rejected():
    from paper_2601_22074_b200.tasks import TaskError, make_env_cfg

    with pytest.raises(TaskError, match="Velocity-Flat"):
        make_env_cfg("Velocity-Flight")


def test_config_round_trip_preserves_variants():
    from paper_2601_22074_b200.tasks import make_env_cfg

    cfg = make_env_cfg("Velocity-Rough")
    cfg.actions["joint_targets"].actuators = {"x": C.DelayedCfg(inner=C.DcMotorCfg(kp=3.0))}
    back = C.from_dict(C.EnvCfg, json.loads(json.dumps(C.to_dict(cfg))))
    assert C.to_dict(back) == C.to_dict(cfg)
    assert isinstance(back.actions["joint_targets"].actuators["x"].inner, C.DcMotorCfg)
    assert isinstance(back.scene.terrain.sub_terrains[1], C.PyramidStairsCfg)


@pytest.mark.parametrize("mutate,msg", [
    (lambda s: setattr(s.joints[0], "link_length", 0.0), "link_length"),
    (lambda s: setattr(s.joints[0], "pos_limits", (1.0, -1.0)), "pos_limits"),
    (lambda s: setattr(s, "base_mass", 0.0), "base_mass"),
    (lambda s: setattr(s, "physics_dt", -1.0), "physics_dt"),
    (lambda s: setattr(s, "feet", [0]), "not a chain tip"),
])
def test_spec_validation(mutate, msg):
    s = two_leg_spec()
    mutate(s)
    with pytest.raises(C.SpecError, match=msg):
        s.validate()


def test_spec_yaml_round_trip(tmp_path):
    s = two_leg_spec()
    p = str(tmp_path / "s.yaml")
    C.save_model_spec(s, p)
    back = C.load_model_spec(p)
    assert C.to_dict(back) == C.to_dict(s)


def test_host_streams_match_reference_draws():
    from paper_2601_22074_b200.rng import HostStreams, purpose_base, purpose_id

    g = golden("rng.npz")
    hs = HostStreams(7, 100 + np.arange(6))
    assert np.array_equal(hs.uniform("a.b", -2.0, 3.0, None, 5), g["u_all"])
    assert np.array_equal(hs.uniform("a.b", 0.0, 1.0, np.array([1, 4]), 3), g["u_sel"])
    assert purpose_id("policy.random") == int.from_bytes(
        __import__("hashlib").sha256(b"policy.random").digest()[:8], "little")
    assert 0 <= purpose_base(0, "x") < 2**64


def test_traffic_model_constants():
    from paper_2601_22074_b200 import traffic

    assert traffic.F64 == 8 and traffic.U8 == 1


def test_pendulum_spec_valid():
    pendulum_spec().validate()


def test_jit_staging_layout_decisions(monkeypatch):
    """The specialized kernel's shared-memory staging (jit.staging_layout): the biped keeps the model
    fields in static shared memory beside the observation rows; a 12-joint model also moves its action /
    target vectors and episodic sums there and needs the dynamic block (> 48 KB); block 128 (large N)
    drops the biped's field columns (they no longer fit beside 128 observation rows)."""
    from paper_2601_22074_b200 import jit, native

    def desc(k, a, rewards, groups):
        d = native.EnvDesc()
        d.model.n_joints, d.n_actuators, d.action_dim, d.n_rewards = k, 1, a, rewards
        d.n_groups = len(groups)
        for g, dim in enumerate(groups):
            d.group[g].dim = dim
        return d

    for var in ("SS_PARAM_SMEM", "SS_ACT_SMEM", "SS_DYN_SMEM_MAX", "SS_STAGE_OBS"):
        monkeypatch.delenv(var, raising=False)
    biped = desc(4, 4, 7, (19, 28))
    L = jit.staging_layout(biped, 64, jit.obs_staged(biped, 64), 47)
    assert (L["param"], L["act"], L["dyn"]) == (1, 0, 0)
    L = jit.staging_layout(biped, 128, jit.obs_staged(biped, 128), 47)
    assert (L["param"], L["act"], L["dyn"]) == (0, 0, 0)
    quad = desc(12, 12, 7, (43, 51))
    L = jit.staging_layout(quad, 64, jit.obs_staged(quad, 64), 94)
    assert L["param"] == 1 and L["act"] == 1 and 48 * 1024 < L["dyn"] <= 112 * 1024
    assert L["obs_off"] == 0 < L["param_off"] < L["act_off"]
    monkeypatch.setenv("SS_ACT_SMEM", "0")
    L = jit.staging_layout(quad, 64, jit.obs_staged(quad, 64), 94)
    assert (L["act"], L["dyn"]) == (0, 0)
