"""Host-side task configuration of the 3-D path (no GPU): tracked bodies, contact-sensor tables, feet."""
import numpy as np
import pytest

from paper_2601_22074_b200.sim3d import robots
from paper_2601_22074_b200.sim3d.task import (BEYONDMIMIC_BODIES, LiftTaskCfg, MotionTrackingCfg, VelocityTaskCfg,
                                              padded, pair_sensor_bits, robot_geoms)


def _motion_cfg(m, **kw):
    dq = robots.default_qpos(m, robots.G1_DEFAULT_JOINTS)
    return MotionTrackingCfg(default_qpos=dq, motion_qpos=np.tile(dq, (2, 1)), motion_qvel=np.zeros((2, m.nv)),
                             motion_dt=0.02, **kw)


def test_tracked_bodies_defaults_and_overrides():
    m = robots.g1_like()
    anchor, bodies = _motion_cfg(m).tracked(m)
    assert m.body_names[anchor] == "torso_link" and [m.body_names[b] for b in bodies] == list(BEYONDMIMIC_BODIES)
    anchor, bodies = _motion_cfg(m, anchor_body="pelvis", track_bodies=("left_knee_link", 5)).tracked(m)
    assert anchor == 1 and bodies == (m.body_names.index("left_knee_link"), 5)
    with pytest.raises(ValueError):
        _motion_cfg(m, track_bodies=tuple(range(1, 20))).tracked(m)  # more than S3_MAX_TRACK
    go1 = robots.go1_like()  # no BeyondMimic names: every body of the robot's tree about its root
    anchor, bodies = _motion_cfg(go1).tracked(go1)
    assert anchor == 1 and bodies == tuple(range(1, go1.nbody))


def test_contact_sensor_tables():
    m = robots.g1_like()
    sens = _motion_cfg(m).sensors(m)
    assert sens[0][0] == "self_collision" and set(sens[0][1]) == set(robot_geoms(m))
    bits = pair_sensor_bits(m, sens)
    assert [bool(b & 1) for b in bits] == [g1 != 0 for g1, _ in m.pair_geom]  # robot-robot pairs only
    # a sensor against any geom (None) and a second bit
    any_bits = pair_sensor_bits(m, (("feet_any", (4, 5), None), ("torso_ground", (14,), (0,))))
    for p, (g1, g2) in enumerate(m.pair_geom):
        assert bool(any_bits[p] & 1) == (g1 in (4, 5) or g2 in (4, 5))
        assert bool(any_bits[p] & 2) == ({g1, g2} == {0, 14})
    assert _motion_cfg(m, self_collision=False).sensors(m) == ()


def test_velocity_feet_and_lift_sensors():
    g1, go1 = robots.g1_like(), robots.go1_like()
    cfg = VelocityTaskCfg(default_qpos=g1.qpos0.copy())
    assert [g1.body_names[b] for b in cfg.foot_bodies(g1)] == ["left_ankle_roll_link", "right_ankle_roll_link"]
    assert [s[0] for s in cfg.sensors(g1)] == ["left_ankle_roll_link_ground", "right_ankle_roll_link_ground"]
    assert len(VelocityTaskCfg(default_qpos=go1.qpos0.copy()).foot_bodies(go1)) == 4
    arm = robots.arm_cube_like()
    lift = LiftTaskCfg.for_model(arm, robots.default_qpos(arm, robots.ARM_DEFAULT_JOINTS))
    assert [s[0] for s in lift.sensors(arm)] == ["ee_cube", "ee_ground", "cube_ground"]
    assert padded((1.0, 2.0), 4) == (1.0, 2.0, 0.0, 0.0)
    with pytest.raises(ValueError):
        padded((1.0,) * 11, 10)


def test_beyondmimic_motion_file_round_trip(tmp_path):
    """A clip written in the BeyondMimic / mjlab .npz layout (root body pose and world velocities, joint
    arrays, fps) loads back to the same qpos / qvel (free joint in MuJoCo's convention: angular velocity in
    the body frame), with the file's joints in a permuted, named order."""
    from oracle import sim3d as O
    from paper_2601_22074_b200.sim3d.motion import load_motion_npz, synthetic_walk_clip

    m = robots.g1_like()
    Q, V, dt = synthetic_walk_clip(m, robots.default_qpos(m, robots.G1_DEFAULT_JOINTS), seconds=0.5)
    hinges = [j for j in range(m.njnt) if m.jnt_type[j] != 0]
    perm = np.random.default_rng(0).permutation(len(hinges))
    names = [m.jnt_names[hinges[k]] for k in perm]
    jp = np.stack([Q[:, m.jnt_qposadr[hinges[k]]] for k in perm], 1)
    jv = np.stack([V[:, m.jnt_dofadr[hinges[k]]] for k in perm], 1)
    root_w = np.stack([O.qmat(Q[f, 3:7]) @ V[f, 3:6] for f in range(Q.shape[0])])  # body-frame -> world
    path = tmp_path / "clip.npz"
    np.savez(path, fps=np.array([1.0 / dt]), joint_pos=jp, joint_vel=jv, body_pos_w=Q[:, None, 0:3],
             body_quat_w=Q[:, None, 3:7], body_lin_vel_w=V[:, None, 0:3], body_ang_vel_w=root_w[:, None])
    Q2, V2, dt2 = load_motion_npz(path, m, joint_names=names)
    np.testing.assert_allclose(Q2, Q, atol=1e-12)
    np.testing.assert_allclose(V2, V, atol=1e-12)
    assert abs(dt2 - dt) < 1e-15


def test_adaptive_sampling_weights_follow_failures():
    """BeyondMimic's adaptive sampling: uniform weights before any failure; failures in a bin raise that bin
    and (through the forward kernel) the bins just before it; the host fold (task.fold_bins) and the oracle's
    agree bit for bit; start times land inside the drawn bin."""
    from oracle import sim3d as O
    from paper_2601_22074_b200.sim3d.task import fold_bins

    m = robots.g1_like()
    dq = robots.default_qpos(m, robots.G1_DEFAULT_JOINTS)
    from paper_2601_22074_b200.sim3d.motion import synthetic_walk_clip

    Q, V, dt = synthetic_walk_clip(m, dq, seconds=6.0)
    cfg = MotionTrackingCfg(default_qpos=dq, motion_qpos=Q, motion_qvel=V, motion_dt=dt, adaptive_alpha=0.5)
    nb = cfg.n_bins()
    assert nb == 7
    cum0 = cfg.initial_bin_cum()
    np.testing.assert_allclose(np.diff(np.concatenate([[0.0], cum0])), cum0[0], rtol=1e-12)  # uniform
    ref = O.MotionTaskOracle(m, cfg, 1)
    np.testing.assert_array_equal(ref.bin_cum, cum0)
    now = np.zeros(nb)
    now[4] = 10
    ref.bin_now[:] = now.astype(np.int64)
    ref.fold_bins()
    failed, cum = fold_bins(np.zeros(nb), now, cfg)
    np.testing.assert_array_equal(ref.bin_cum, cum)
    q = np.diff(np.concatenate([[0.0], cum]))
    assert q.argmax() == 4 and q[3] > q[2] > q[1] and q[5] < q[4]  # the failing bin and the lead-up to it
    ref.cmd[:] = 0.0
    for ctr in range(1, 50):
        t0 = ref.start_time(ref.key(0, 1), ctr)
        assert 0.0 <= t0 <= ref.clip_end()
