"""Generate golden vectors by running the UNMODIFIED reference (stridesim).

Run in the build container (the reference only exists there):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Writes tests/golden/*.npz (+ the EnvCfg of each rollout as JSON inside the
archive). The CPU test-suite pins the numpy oracle to these files; the GPU
suite compares the CUDA path against the oracle (and these files) on the box,
where /root/reference does not exist.
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
if REF not in sys.path:
    sys.path.insert(0, REF)

import stridesim  # noqa: E402
from stridesim.actuators import DcMotorCfg, DelayedCfg, IdealPdCfg  # noqa: E402
from stridesim.config import config_hash, to_dict  # noqa: E402
from stridesim.env import ManagerBasedRlEnv  # noqa: E402
from stridesim.managers import CurriculumTermCfg, EventTermCfg, NoiseCfg, ObsGroupCfg, ObsTermCfg  # noqa: E402
from stridesim.policies import random_policy  # noqa: E402
from stridesim.rng import StreamPack  # noqa: E402
from stridesim.sim import BatchState, JointSpec, ModelSpec, StepPipeline, compile_model  # noqa: E402
from stridesim.tasks import make_env_cfg  # noqa: E402
from stridesim.terrain import generate_grid  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def quad_spec() -> ModelSpec:
    """Go1-sized planar quadruped surrogate: 4 legs x (hip, knee, ankle)."""
    joints = []
    feet = []
    for leg, hx in (("fl", 0.25), ("fr", 0.2), ("rl", -0.2), ("rr", -0.25)):
        h = len(joints)
        joints.append(JointSpec(f"{leg}_hip", -1, (hx, 0.0), 0.12, 0.4, 0.05, 0.05, (-1.2, 1.2)))
        joints.append(JointSpec(f"{leg}_knee", h, (0.0, -0.12), 0.12, 0.3, 0.05, 0.05, (-2.0, 0.5)))
        joints.append(JointSpec(f"{leg}_ankle", h + 1, (0.0, -0.12), 0.06, 0.1, 0.05, 0.05, (-1.0, 1.0)))
        feet.append(h + 2)
    return ModelSpec(name="quad12", base_mass=10.0, base_inertia=0.3, joints=joints, feet=feet)


def humanoid_spec() -> ModelSpec:
    """G1-sized surrogate: 2 legs x (hip, knee, ankle) + 2 arms x (shoulder, elbow)."""
    joints = []
    feet = []
    for side, hx in (("l", -0.08), ("r", 0.08)):
        h = len(joints)
        joints.append(JointSpec(f"{side}_hip", -1, (hx, 0.0), 0.3, 1.5, 0.1, 0.1, (-1.6, 1.6)))
        joints.append(JointSpec(f"{side}_knee", h, (0.0, -0.3), 0.3, 1.0, 0.1, 0.1, (-2.2, 0.4)))
        joints.append(JointSpec(f"{side}_ankle", h + 1, (0.0, -0.3), 0.08, 0.3, 0.05, 0.05, (-1.0, 1.0)))
        feet.append(h + 2)
    for side, hx in (("l", -0.15), ("r", 0.15)):
        s = len(joints)
        joints.append(JointSpec(f"{side}_shoulder", -1, (hx, 0.45), 0.25, 0.8, 0.05, 0.05, (-2.5, 2.5)))
        joints.append(JointSpec(f"{side}_elbow", s, (0.0, -0.25), 0.25, 0.5, 0.05, 0.05, (-2.5, 0.5)))
    return ModelSpec(name="humanoid10", base_mass=20.0, base_inertia=0.6, joints=joints, feet=feet)


def rollout(cfg, steps: int, task: str = "", policy="random"):
    env = ManagerBasedRlEnv(cfg, task)
    obs0 = env.reset()
    rec = {k: [] for k in ("q", "qd", "ctrl", "reward", "terminated", "truncated", "actions")}
    groups = list(obs0)
    for g in groups:
        rec[f"obs0/{g}"] = obs0[g].copy()
        rec[f"obs/{g}"] = []
    for i in range(steps):
        if policy == "random":
            a = random_policy(env, i)
        else:
            a = np.full((env.num_envs, env.action_manager.total_dim), np.sin(0.37 * i))
        obs, rew, term, trunc, extras = env.step(a)
        rec["actions"].append(np.asarray(a).copy())
        rec["q"].append(env.state.q.copy())
        rec["qd"].append(env.state.qd.copy())
        rec["ctrl"].append(env.state.ctrl.copy())
        rec["reward"].append(rew.copy())
        rec["terminated"].append(term.copy())
        rec["truncated"].append(trunc.copy())
        for g in groups:
            rec[f"obs/{g}"].append(obs[g].copy())
    out = {k: np.asarray(v) for k, v in rec.items()}
    out["trigger_counts"] = np.array([env.termination_manager.trigger_counts[k]
                                      for k in env.termination_manager.trigger_counts], dtype=np.int64)
    out["terrain_rows"] = env.terrain_rows.copy()
    out["sensor_last_air"] = env.contact_sensor.last_air_time.copy()
    out["ranges"] = env.command_manager.ranges.copy()
    out["ep_sums"] = np.stack([env.reward_manager.episodic_sums[k] for k in env.reward_manager.episodic_sums])
    for name in env.model.field_names():
        out[f"field/{name}"] = np.asarray(env.model.field(name).value).copy()
    out["cfg_json"] = np.array(json.dumps(to_dict(cfg)))
    out["config_hash"] = np.array(config_hash(cfg))
    out["sim_step"] = np.array(env.state.sim_step)
    return out


def soup_cfg(n: int, seed: int):
    """Velocity-Rough plus every optional manager feature the reference has."""
    cfg = make_env_cfg("Velocity-Rough", num_envs=n, seed=seed)
    cfg.actions["joint_targets"].actuators = {
        "hips": DelayedCfg(inner=IdealPdCfg(joint_patterns=[".*_hip"], kp=45.0, kd=1.5, effort_limit=28.0),
                           latency_range=(0.0, 0.015)),
        "knees": DcMotorCfg(joint_patterns=[".*_knee"], kp=40.0, kd=2.0, effort_limit=30.0,
                            saturation_effort=40.0, velocity_limit=15.0),
    }
    pol = cfg.observations["policy"].terms
    pol["base_lin_vel"].delay_steps = 2
    pol["joint_pos_rel"].history = 3
    pol["joint_vel"].clip = (-5.0, 5.0)
    pol["joint_vel"].scale = 0.5
    pol["base_lin_acc"] = ObsTermCfg(func="base_lin_acc", noise=NoiseCfg("gaussian", 0.05), delay_steps=1,
                                     history=2)
    pol["sim_time"] = ObsTermCfg(func="sim_time", history=4)
    cfg.observations["critic"].terms["base_height"] = ObsTermCfg(func="base_height", scale=2.0)
    cfg.observations["aux"] = ObsGroupCfg(terms={
        "feet": ObsTermCfg(func="foot_contact_forces", clip=(-100.0, 100.0), scale=0.01, delay_steps=3),
        "scan": ObsTermCfg(func="height_scan", noise=NoiseCfg("uniform", 0.02), history=2),
    }, enable_noise=True)
    cfg.events["interval_push"].interval_range = (0.2, 0.5)
    cfg.events["reset_friction"] = EventTermCfg(func="randomize_model_field", mode="reset",
                                                params={"field": "friction", "distribution": "gaussian",
                                                        "rng_range": (1.0, 0.1), "operation": "set"})
    cfg.events["interval_damping"] = EventTermCfg(func="randomize_model_field", mode="interval",
                                                  interval_range=(0.3, 0.6),
                                                  params={"field": "damping", "distribution": "uniform",
                                                          "rng_range": (0.05, 0.0), "operation": "add"})
    cfg.curriculum["command_widen"].params["threshold"] = 0.2
    cfg.curriculum["fade"] = CurriculumTermCfg(func="reward_weight_schedule",
                                               params={"term": "foot_slip_penalty", "start_weight": -0.1,
                                                       "end_weight": -0.5, "start_step": 5, "end_step": 40})
    cfg.episode_length_s = 0.8
    return cfg


def mlp_cfg(n: int, seed: int):
    """Velocity-Flat with an MLP actuator on the knees (actuators.py:124-180, 302-316)."""
    from stridesim.actuators import MlpActuatorCfg, save_mlp_weights

    path = os.path.join(OUT, "mlp_knee.ssmlp")
    r = np.random.default_rng(11)
    layers = [(r.normal(0, 0.8, (16, 4)), r.normal(0, 0.1, 16), "tanh"),
              (r.normal(0, 0.5, (16, 16)), r.normal(0, 0.1, 16), "relu"),
              (r.normal(0, 2.0, (1, 16)), r.normal(0, 0.1, 1), "identity")]
    save_mlp_weights(path, layers)
    cfg = make_env_cfg("Velocity-Flat", num_envs=n, seed=seed)
    cfg.actions["joint_targets"].actuators = {
        "hips": IdealPdCfg(joint_patterns=[".*_hip"], kp=40.0, kd=2.0, effort_limit=30.0),
        "knees": MlpActuatorCfg(joint_patterns=[".*_knee"], weights_path="tests/golden/mlp_knee.ssmlp",
                                error_history=2, velocity_history=2, effort_limit=25.0),
    }
    return cfg


def physics_cases():
    out = {}
    rng = np.random.default_rng(2601)
    terrain = generate_grid(make_env_cfg("Velocity-Rough").scene.terrain, 0)
    for name, spec in (("biped", make_env_cfg("Velocity-Flat").scene.model), ("quad", quad_spec()),
                       ("humanoid", humanoid_spec())):
        for tname, ter in (("flat", None), ("rough", terrain)):
            n = 64
            model = compile_model(spec, n)
            st = BatchState(model)
            q = rng.uniform(-0.6, 0.6, size=(n, model.nq))
            q[:, 0] = rng.uniform(0.0, 200.0, size=n) if ter is not None else q[:, 0]
            q[:, 1] = rng.uniform(0.2, 0.6, size=n) + (ter.heights(q[:, 0]) if ter is not None else 0.0)
            st.q[:] = q
            st.qd[:] = rng.uniform(-1.5, 1.5, size=(n, model.nq))
            st.ctrl[:] = rng.uniform(-5.0, 5.0, size=(n, model.num_joints))
            st.ext_force[:] = rng.uniform(-20.0, 20.0, size=(n, 2))
            key = f"{name}_{tname}"
            out[f"{key}/q0"] = st.q.copy()
            out[f"{key}/qd0"] = st.qd.copy()
            out[f"{key}/ctrl"] = st.ctrl.copy()
            out[f"{key}/ext0"] = st.ext_force.copy()
            pipe = StepPipeline(model, ter)
            qs, qds = [], []
            for _ in range(20):
                pipe.substep(st)
                qs.append(st.q.copy())
                qds.append(st.qd.copy())
            out[f"{key}/q"] = np.asarray(qs)
            out[f"{key}/qd"] = np.asarray(qds)
            out[f"{key}/fn"] = st.contact.normal_force.copy()
            out[f"{key}/ft"] = st.contact.tangent_force.copy()
            out[f"{key}/fin"] = st.contact.in_contact.copy()
            out[f"{key}/fpos"] = st.contact.foot_pos.copy()
            out[f"{key}/fvel"] = st.contact.foot_vel.copy()
            out[f"{key}/spec_json"] = np.array(json.dumps(to_dict(spec)))
    return out


def rng_cases():
    out = {}
    sp = StreamPack(7, 100 + np.arange(6))
    out["u_all"] = sp.uniform("a.b", -2.0, 3.0, None, 5)
    out["u_sel"] = sp.uniform("a.b", 0.0, 1.0, np.array([1, 4]), 3)
    out["u_rowlo"] = sp.uniform("c", np.arange(6.0), np.arange(6.0) + 2.0, None, 2)
    out["n_all"] = sp.normal("d", 0.5, None, 3)
    out["n_sel"] = sp.normal("d", 2.0, np.array([0, 5]), 2)
    out["i_all"] = sp.integers("e", -3, 4, None, 7)
    return out


def capture_cases():
    """SSCAPT v1 dumps written by the reference itself (capture.py:81-104):
    the replay case of tests/test_env.py:182-213 (Velocity-Flat, 2 worlds,
    seed 5, six zero-action steps, env.dump_capture) and an automatic
    nonfinite dump (env.py:240-241, :276-298) of a Velocity-Rough run whose
    world 1 gets an infinite velocity after three random-policy steps."""
    import shutil
    import tempfile

    cfg = make_env_cfg("Velocity-Flat", num_envs=2, seed=5)
    env = ManagerBasedRlEnv(cfg, "Velocity-Flat")
    env.reset()
    for _ in range(6):
        env.step(np.zeros((2, 4)))
    env.dump_capture(os.path.join(OUT, "capture_flat.bin"))

    tmp = tempfile.mkdtemp()
    cfg = make_env_cfg("Velocity-Rough", num_envs=3, seed=9)
    cfg.capture_len = 10
    cfg.capture_dir = tmp
    env = ManagerBasedRlEnv(cfg, "Velocity-Rough")
    env.reset()
    for i in range(3):
        env.step(random_policy(env, i))
    env.state.qd[1, 0] = np.inf
    env.step(random_policy(env, 3))
    assert len(env.dump_paths) == 1
    shutil.copy(env.dump_paths[0], os.path.join(OUT, "capture_nan.bin"))
    shutil.rmtree(tmp)


def main():
    if "--only-capture" in sys.argv:
        capture_cases()
        return
    capture_cases()
    t = generate_grid(make_env_cfg("Velocity-Rough").scene.terrain, 0)
    np.savez_compressed(os.path.join(OUT, "terrain_rough_seed0.npz"), samples=t.samples,
                        difficulty=t.difficulty, type_index=t.type_index)
    np.savez_compressed(os.path.join(OUT, "physics.npz"), **physics_cases())
    np.savez_compressed(os.path.join(OUT, "rng.npz"), **rng_cases())
    np.savez_compressed(os.path.join(OUT, "rollout_flat.npz"),
                        **rollout(make_env_cfg("Velocity-Flat", num_envs=8, seed=0), 40, "Velocity-Flat"))
    np.savez_compressed(os.path.join(OUT, "rollout_rough.npz"),
                        **rollout(make_env_cfg("Velocity-Rough", num_envs=16, seed=7), 60, "Velocity-Rough"))
    np.savez_compressed(os.path.join(OUT, "rollout_soup.npz"), **rollout(soup_cfg(12, 123), 60))
    cwd = os.getcwd()
    os.chdir(os.path.dirname(os.path.dirname(OUT)))  # weights path is repo-relative
    try:
        np.savez_compressed(os.path.join(OUT, "rollout_mlp.npz"), **rollout(mlp_cfg(10, 5), 40))
    finally:
        os.chdir(cwd)
    qcfg = make_env_cfg("Velocity-Flat", num_envs=6, seed=1)
    qcfg.scene.model = quad_spec()
    qcfg.scene.init_state.joint_pos = (0.3, -0.6, 0.3) * 4
    qcfg.scene.init_state.base_pose = (0.0, 0.3, 0.0)
    np.savez_compressed(os.path.join(OUT, "rollout_quad.npz"), **rollout(qcfg, 30, policy="sine"))
    print("golden vectors written to", OUT, "with stridesim", stridesim.__version__ if hasattr(stridesim, "__version__") else "")


if __name__ == "__main__":
    main()
