"""The 3-D oracle (oracle/sim3d.py) pinned by analytic properties (no reference exists).

Each test checks a stage against an independent computation: rotation
composition, finite differences of forward kinematics, kinetic and potential
energy, the Lagrangian, brute-force geometry, and the optimality conditions
of the constraint problem.
"""

import numpy as np
import pytest

from oracle import sim3d as O
from paper_2601_22074_b200.sim3d import robots
from paper_2601_22074_b200.sim3d.model import (ACT_DC, ACT_PD, GEOM_CAPSULE, GEOM_SPHERE, ModelBuilder, Opt)


def _arm(gravity=(0, 0, -9.81)):
    b = ModelBuilder("arm", Opt(gravity=gravity))
    b.plane()
    l1 = b.body("l1", 0, pos=(0, 0, 1.0), quat=(0.9, 0.1, 0.3, 0.2), mass=1.2, inertia=(0.02, 0.03, 0.01),
                ipos=(0.1, 0.02, -0.2), iquat=(0.8, 0.2, 0.1, 0.4))
    b.hinge(l1, (0, 0, 1), pos=(0.05, 0, 0))
    l2 = b.body("l2", l1, pos=(0.0, 0.1, -0.4), mass=0.8, inertia=(0.01, 0.015, 0.004), ipos=(0.0, 0.05, -0.1))
    b.hinge(l2, (1, 1, 0), pos=(0, 0.02, 0.01))
    l3 = b.body("l3", l2, pos=(0.1, 0.0, -0.3), quat=(0.7, 0.0, 0.7, 0.1), mass=0.5, inertia=(0.004, 0.002, 0.003),
                ipos=(0.03, 0.0, -0.05))
    b.hinge(l3, (0.2, 0.3, 0.9))
    b.geom(l3, GEOM_SPHERE, (0.05,))
    return b.compile()


def _random_state(m, rng, scale=0.5):
    q = m.qpos0.copy()
    v = rng.normal(size=m.nv) * scale
    for j in range(m.njnt):
        a = m.jnt_qposadr[j]
        if m.jnt_type[j] == 0:
            q[a:a + 3] += rng.normal(size=3) * 0.1
            quat = rng.normal(size=4)
            q[a + 3:a + 7] = quat / np.linalg.norm(quat)
        else:
            q[a] = rng.uniform(-1, 1)
    return q, v


MODELS = {"g1": robots.g1_like, "go1": robots.go1_like, "arm": _arm, "arm_cube": robots.arm_cube_like}


@pytest.fixture(params=list(MODELS))
def model(request):
    m = MODELS[request.param]()
    O.set_const(m)
    return m


def _homog(q, p):
    T = np.eye(4)
    T[:3, :3] = O.qmat(q)
    T[:3, 3] = p
    return T


def test_fk_matches_homogeneous_composition(model, rng):
    m = model
    q, _ = _random_state(m, rng)
    K = O.kinematics(m, q)
    T = [np.eye(4)]
    for b in range(1, m.nbody):
        Tb = T[m.body_parentid[b]] @ _homog(m.body_quat[b], m.body_pos[b])
        for j in range(m.body_jntadr[b], m.body_jntadr[b] + m.body_jntnum[b]):
            a = m.jnt_qposadr[j]
            if m.jnt_type[j] == 0:
                Tb = _homog(q[a + 3:a + 7] / np.linalg.norm(q[a + 3:a + 7]), q[a:a + 3])
            else:
                ax = m.jnt_axis[j]
                th = q[a] - m.qpos0[a]
                # rotation about the joint axis through jnt_pos (body frame)
                R = O.qmat(O.qaxisangle(ax, th))
                P = np.eye(4)
                P[:3, 3] = m.jnt_pos[j]
                Rh = np.eye(4)
                Rh[:3, :3] = R
                Pi = np.eye(4)
                Pi[:3, 3] = -m.jnt_pos[j]
                Tb = Tb @ P @ Rh @ Pi
        T.append(Tb)
    for b in range(1, m.nbody):
        np.testing.assert_allclose(K["xpos"][b], T[b][:3, 3], atol=1e-12)
        np.testing.assert_allclose(K["xmat"][b], T[b][:3, :3], atol=1e-12)


def _kinetic_from_fd(m, q, v, h=1e-6):
    """sum_b 1/2 m |v_com|^2 + 1/2 w^T I w, body velocities by central differences of FK."""
    Kp = O.kinematics(m, O.integrate_pos(m, q, v, h))
    Km = O.kinematics(m, O.integrate_pos(m, q, v, -h))
    K0 = O.kinematics(m, q)
    T = 0.0
    for b in range(1, m.nbody):
        vc = (Kp["xipos"][b] - Km["xipos"][b]) / (2 * h)
        dR = (Kp["xmat"][b] - Km["xmat"][b]) / (2 * h)
        W = dR @ K0["xmat"][b].T
        w = np.array([W[2, 1], W[0, 2], W[1, 0]])
        Ib = K0["ximat"][b] @ np.diag(m.body_inertia[b]) @ K0["ximat"][b].T
        T += 0.5 * m.body_mass[b] * vc @ vc + 0.5 * w @ Ib @ w
    return T


def test_mass_matrix_is_kinetic_energy(model, rng):
    m = model
    for _ in range(3):
        q, v = _random_state(m, rng)
        F = O.forward(m, q, v, np.zeros(m.nu))
        M = F["M"] - np.diag(m.dof_armature)
        np.testing.assert_allclose(F["M"], F["M"].T, atol=0)
        assert np.all(np.linalg.eigvalsh(F["M"]) > 0)
        T = _kinetic_from_fd(m, q, v)
        assert abs(0.5 * v @ M @ v - T) < 1e-7 * max(1.0, T)


def test_ldl_factor_solves_and_reconstructs(model, rng):
    m = model
    q, v = _random_state(m, rng)
    K = O.kinematics(m, q)
    C = O.com_pos(m, K)
    M, _ = O.crb(m, C)
    L = O.factor_ldl(m, M)
    # reconstruct: M = U^T D U with U unit upper-in-reverse (L below diagonal on ancestor entries)
    U = np.tril(L, -1) + np.eye(m.nv)
    D = np.diag(np.diag(L))
    np.testing.assert_allclose(U.T @ D @ U, M, rtol=1e-12, atol=1e-12)
    for (i, j) in zip(*np.nonzero(np.tril(L, -1))):
        assert j in m.dof_chain[i]  # no fill-in outside the tree pattern
    b = rng.normal(size=m.nv)
    np.testing.assert_allclose(O.solve_ldl(m, L, b), np.linalg.solve(M, b), rtol=1e-9, atol=1e-12)


def test_point_jacobian_is_fd_of_fk(model, rng):
    m = model
    q, v = _random_state(m, rng)
    K = O.kinematics(m, q)
    C = O.com_pos(m, K)
    h = 1e-6
    for b in range(1, m.nbody):
        loc = rng.normal(size=3) * 0.1
        J = O.point_jac(m, C, b, K["xpos"][b] + K["xmat"][b] @ loc)
        Kp = O.kinematics(m, O.integrate_pos(m, q, v, h))
        Km = O.kinematics(m, O.integrate_pos(m, q, v, -h))
        fd = ((Kp["xpos"][b] + Kp["xmat"][b] @ loc) - (Km["xpos"][b] + Km["xmat"][b] @ loc)) / (2 * h)
        np.testing.assert_allclose(J @ v, fd, atol=1e-7)


def test_rne_matches_lagrangian_fixed_base(rng):
    m = _arm()
    O.set_const(m)
    q, v = _random_state(m, rng, 1.0)
    F = O.forward(m, q, v, np.zeros(m.nu))
    h = 1e-6

    def Mof(qq):
        return O.crb(m, O.com_pos(m, O.kinematics(m, qq)))[0]

    def V(qq):
        K = O.kinematics(m, qq)
        return -sum(m.body_mass[b] * np.asarray(m.opt.gravity) @ K["xipos"][b] for b in range(1, m.nbody))

    Mdot = (Mof(q + h * v) - Mof(q - h * v)) / (2 * h)
    dT = np.zeros(m.nv)
    dV = np.zeros(m.nv)
    for i in range(m.nv):
        e = np.zeros(m.nv)
        e[i] = h
        dT[i] = 0.5 * v @ ((Mof(q + e) - Mof(q - e)) / (2 * h)) @ v
        dV[i] = (V(q + e) - V(q - e)) / (2 * h)
    np.testing.assert_allclose(F["bias"], Mdot @ v - dT + dV, rtol=1e-6, atol=1e-6)


@pytest.mark.parametrize("gravity", [(0, 0, 0), (0, 0, -9.81)])
def test_energy_conserved_free_floating(gravity, rng):
    m = robots.go1_like(opt=Opt(gravity=gravity))
    m.actuator_kp[:] = 0
    m.actuator_kv[:] = 0
    O.set_const(m)
    q, v = _random_state(m, rng, 0.3)
    q[2] = 5.0

    def acc(qq, vv):
        F = O.forward(m, qq, vv, np.zeros(m.nu))
        return F["qacc_smooth"]

    def energy(qq, vv):
        F = O.forward(m, qq, vv, np.zeros(m.nu))
        K = F["K"]
        Vp = -sum(m.body_mass[b] * np.asarray(gravity) @ K["xipos"][b] for b in range(1, m.nbody))
        return 0.5 * vv @ F["M"] @ vv + Vp

    E0 = energy(q, v)
    dt = 1e-3
    for _ in range(50):  # RK4 on (q, v) with the manifold update for the free joint
        k1v = acc(q, v)
        k2v = acc(O.integrate_pos(m, q, v, dt / 2), v + dt / 2 * k1v)
        k3v = acc(O.integrate_pos(m, q, v + dt / 2 * k1v, dt / 2), v + dt / 2 * k2v)
        k4v = acc(O.integrate_pos(m, q, v + dt / 2 * k2v, dt), v + dt * k3v)
        vn = v + dt / 6 * (k1v + 2 * k2v + 2 * k3v + k4v)
        vbar = (v + 2 * (v + dt / 2 * k1v) + 2 * (v + dt / 2 * k2v) + (v + dt * k3v)) / 6
        q = O.integrate_pos(m, q, vbar, dt)
        v = vn
    assert abs(energy(q, v) - E0) < 2e-4 * max(1.0, abs(E0))


def test_free_fall_exact():
    b = ModelBuilder("ball")
    b.plane()
    ball = b.body("ball", 0, pos=(0, 0, 10.0), mass=2.0, inertia=(0.01, 0.01, 0.01))
    b.free_joint(ball)
    b.geom(ball, GEOM_SPHERE, (0.1,))
    m = b.compile()
    O.set_const(m)
    q, v = m.qpos0.copy(), np.zeros(6)
    z, vz = 10.0, 0.0
    for _ in range(100):
        q, v, _, F = O.step(m, q, v, np.zeros(0))
        vz = vz + 0.005 * -9.81
        z = z + 0.005 * vz
        assert F["contacts"] == []
    assert abs(q[2] - z) < 1e-12 and abs(v[2] - vz) < 1e-12


def test_ball_comes_to_rest_on_plane_and_forces_in_cone():
    b = ModelBuilder("ball")
    b.plane(friction=0.5)
    ball = b.body("ball", 0, pos=(0, 0, 0.2), mass=2.0, inertia=(0.008, 0.008, 0.008))
    b.free_joint(ball)
    b.geom(ball, GEOM_SPHERE, (0.1,), friction=0.5)
    m = b.compile()
    O.set_const(m)
    q, v = m.qpos0.copy(), np.zeros(6)
    v[0] = 1.0  # sliding, then rolling
    warm = None
    for _ in range(800):
        q, v, warm, F = O.step(m, q, v, np.zeros(0), warm=warm)
    assert len(F["contacts"]) == 1
    # sliding decays into rolling without slip: v_x = w_y r, no vertical motion
    assert abs(q[2] - 0.1) < 2e-3 and abs(v[2]) < 1e-3
    assert abs(v[0] - v[4] * 0.1) < 1e-3 and 0.3 < v[0] < 1.0
    f = F["efc_force"]
    assert np.all(f >= 0)
    # the 4 pyramid edge forces sum to the normal force ~ m g
    assert abs(f.sum() - 2.0 * 9.81) < 0.5


def test_newton_optimality(model, rng):
    m = model
    if m.name == "arm_cube_like":  # cube pressed 3 mm into the table right under the open claw
        q = robots.default_qpos(m, robots.ARM_DEFAULT_JOINTS)
        q[-5] -= 0.003
    else:
        q = robots.default_qpos(m, robots.G1_DEFAULT_JOINTS if m.name == "g1_like" else robots.GO1_DEFAULT_JOINTS) \
            if m.name != "arm" else m.qpos0.copy()
    if m.name not in ("arm", "arm_cube_like"):  # press the lowest geom 5 mm into the ground
        K = O.kinematics(m, q)
        low = min(K["geom_xpos"][g][2] - m.geom_rbound[g] for g in range(1, m.ngeom))
        q[2] -= low + 0.005
    v = rng.normal(size=m.nv) * 0.2
    ctrl = q[m.actuator_qposadr] if m.nu else np.zeros(0)
    F = O.forward(m, q, v, ctrl)
    E = F["efc"]
    if m.name != "arm":
        assert len(F["contacts"]) >= 4
    # KKT: M (a - a0) = J^T f, f = D max(-(J a - aref), 0)
    res = F["M"] @ (F["qacc"] - F["qacc_smooth"]) - F["qfrc_constraint"]
    scale = 1.0 / (m.meaninertia * max(1, m.nv))
    assert scale * np.linalg.norm(res) < 1e-5
    np.testing.assert_allclose(F["efc_force"], E["D"] * np.maximum(-(E["J"] @ F["qacc"] - E["aref"]), 0.0),
                               rtol=1e-12, atol=1e-12)


def test_segment_closest_points_brute_force(rng):
    for _ in range(50):
        p1, q1, p2, q2 = (rng.normal(size=3) for _ in range(4))
        a, b = O.seg_closest(p1, q1, p2, q2)
        t = np.linspace(0, 1, 401)
        A = p1 + (q1 - p1) * t[:, None]
        B = p2 + (q2 - p2) * t[:, None]
        brute = np.min(np.linalg.norm(A[:, None] - B[None], axis=-1))
        assert np.linalg.norm(a - b) <= brute + 1e-12
        assert np.linalg.norm(a - b) > brute - 1e-3


def test_hfield_distance_continuous_and_exact_on_vertices():
    m = robots.g1_like(rough=True)
    H, sp, org = m.hfield_data, m.hfield_spacing, m.hfield_origin
    for (iy, ix) in ((3, 5), (40, 70), (100, 12)):
        x, y = org[0] + ix * sp, org[1] + iy * sp
        d, n = O.hfield_point(m, np.array([x, y, 1.0]), 0.0)
        assert abs((1.0 - H[iy, ix]) * n[2] - d) < 1e-12
    # continuity across the cell diagonal and cell edges
    xs = np.linspace(org[0] + 1.0, org[0] + 1.3, 301)
    hs = []
    for x in xs:
        d, n = O.hfield_point(m, np.array([x, org[1] + 2.013, 1.0]), 0.0)
        hs.append(1.0 - d / n[2])
    assert np.max(np.abs(np.diff(hs))) < 0.01


def test_actuator_laws():
    m = robots.go1_like(actuator_kind=ACT_DC)
    m.actuator_saturation[:] = 20.0
    m.actuator_vmax[:] = 10.0
    q = m.qpos0.copy()
    v = np.zeros(m.nv)
    v[m.actuator_dofadr] = 5.0
    ctrl = q[m.actuator_qposadr] + 1.0
    f, kvd = O.actuation(m, q, v, ctrl)
    tau = m.actuator_kp * 1.0 - m.actuator_kv * 5.0
    hi = np.clip(20.0 * (1 - 5.0 / 10.0), 0, m.actuator_effort)
    np.testing.assert_allclose(f[m.actuator_dofadr], np.minimum(tau, hi))
    assert not kvd.any()
    m2 = robots.go1_like(actuator_kind=ACT_PD)
    f2, kvd2 = O.actuation(m2, q, v, ctrl)
    np.testing.assert_allclose(f2[m2.actuator_dofadr], np.clip(tau, -m2.actuator_effort, m2.actuator_effort))
    assert not kvd2.any()
    m3 = robots.go1_like()  # implicit kv enters only where the force range does not clamp
    f3, kvd3 = O.actuation(m3, q, v, ctrl)
    clamped = np.abs(tau) > m3.actuator_effort
    assert clamped.any() and not clamped.all()
    np.testing.assert_allclose(kvd3[m3.actuator_dofadr], np.where(clamped, 0.0, m3.actuator_kv))


def test_self_collision_pairs_generate_contacts():
    m = robots.g1_like()
    O.set_const(m)
    q = robots.default_qpos(m, robots.G1_DEFAULT_JOINTS)
    # swing the left hip roll inward until the shins cross
    j = m.jnt_names.index("left_hip_roll_joint")
    q[m.jnt_qposadr[j]] = -0.45
    j = m.jnt_names.index("right_hip_roll_joint")
    q[m.jnt_qposadr[j]] = 0.45
    K = O.kinematics(m, q)
    cons, _ = O.collide(m, K)
    self_pairs = [c for c in cons if c["geom1"] != 0]
    assert self_pairs, "crossed legs must touch"
    for c in self_pairs:
        assert m.geom_type[c["geom1"]] == GEOM_CAPSULE and c["dist"] < 0


def test_sphere_box_contact_brute_force(rng):
    """Sphere-box distance equals the brute-force distance from the sphere centre to the box minus r
    (outside), and the normal points from the sphere into the box."""
    R = O.qmat(O.qnormalize(rng.normal(size=4)))
    size = np.array([0.05, 0.03, 0.02])
    bc = rng.normal(size=3)
    for _ in range(40):
        c = bc + rng.normal(size=3) * 0.06
        d, n, pos = O.sphere_box(c, 0.01, bc, R, size)
        g = np.stack(np.meshgrid(*[np.linspace(-s, s, 41) for s in size], indexing="ij"), -1).reshape(-1, 3)
        pts = bc + g @ R.T
        p = R.T @ (c - bc)
        if np.all(np.abs(p) <= size):
            assert d < -0.01 + 1e-12
        else:
            brute = np.min(np.linalg.norm(pts - c, axis=1)) - 0.01
            assert abs(d - brute) < 2e-3
            assert np.dot(n, bc - c) > 0
        assert abs(np.linalg.norm(n) - 1) < 1e-12


def test_two_trees_arm_and_cube():
    """Fixed-base arm + free cube: per-tree com, block-diagonal M across trees, and the cube resting
    on the table with its weight carried by the contacts."""
    m = robots.arm_cube_like()
    O.set_const(m)
    assert m.ntree == 2
    q = robots.default_qpos(m, robots.ARM_DEFAULT_JOINTS)
    v = np.zeros(m.nv)
    F = O.forward(m, q, v, q[m.actuator_qposadr])
    arm = [d for d in range(m.nv) if m.body_treeid[m.dof_bodyid[d]] == 0]
    cube = [d for d in range(m.nv) if m.body_treeid[m.dof_bodyid[d]] == 1]
    assert np.all(F["M"][np.ix_(arm, cube)] == 0)
    np.testing.assert_allclose(F["C"]["com"][1], q[-7:-4], atol=1e-12)  # the cube's com is its centre
    warm = None
    for _ in range(100):
        q, v, warm, F = O.step(m, q, v, q[m.actuator_qposadr] * 0 + F["qfrc_actuator"][m.actuator_dofadr] * 0
                               + robots.default_qpos(m, robots.ARM_DEFAULT_JOINTS)[m.actuator_qposadr], warm=warm)
    cube_contacts = [c for c in F["contacts"] if m.geom_bodyid[c["geom2"]] == m.body_names.index("cube")]
    assert len(cube_contacts) == 4 and abs(q[-5] - 0.025) < 1e-3


def test_capsule_box_contact_brute_force(rng):
    """Capsule-box distance (alternating projections, then sphere-box) vs brute force over the segment
    and the box volume, for capsules outside the box."""
    size = np.array([0.05, 0.04, 0.03])
    for _ in range(30):
        R = O.qmat(O.qnormalize(rng.normal(size=4)))
        bc = rng.normal(size=3) * 0.1
        p0, p1 = bc + rng.normal(size=3) * 0.12, bc + rng.normal(size=3) * 0.12
        d, n, pos = O.capsule_box(p0, p1, 0.01, bc, R, size)
        seg = p0 + (p1 - p0) * np.linspace(0, 1, 201)[:, None]
        loc = (seg - bc) @ R
        if np.any(np.all(np.abs(loc) <= size, axis=1)):
            continue  # segment passes through the box: penetration branch, no brute-force distance
        g = np.stack(np.meshgrid(*[np.linspace(-s, s, 21) for s in size], indexing="ij"), -1).reshape(-1, 3)
        pts = bc + g @ R.T
        brute = np.min(np.linalg.norm(seg[:, None] - pts[None], axis=-1)) - 0.01
        assert abs(d - brute) < 6e-3, (d, brute)
        assert abs(np.linalg.norm(n) - 1) < 1e-12


def test_body_state_velocities_are_fd_of_fk(model, rng):
    """BeyondMimic body states: origin linear velocity and angular velocity == finite differences of FK."""
    m = model
    q, v = _random_state(m, rng)
    K = O.kinematics(m, q)
    C = O.com_pos(m, K)
    h = 1e-6
    Kp = O.kinematics(m, O.integrate_pos(m, q, v, h))
    Km = O.kinematics(m, O.integrate_pos(m, q, v, -h))
    for b in range(1, m.nbody):
        st = O.body_state(m, K, C, v, b)
        np.testing.assert_array_equal(st[0:3], K["xpos"][b])
        np.testing.assert_array_equal(st[3:7], K["xquat"][b])
        np.testing.assert_allclose(st[7:10], (Kp["xpos"][b] - Km["xpos"][b]) / (2 * h), atol=1e-7)
        # angular velocity: dR/dt R^T is its cross-product matrix
        W = (Kp["xmat"][b] - Km["xmat"][b]) / (2 * h) @ K["xmat"][b].T
        np.testing.assert_allclose(st[10:13], [W[2, 1], W[0, 2], W[1, 0]], atol=1e-7)


def test_motion_body_table_and_relative_errors():
    """The clip body table is FK of the clip frames; a robot exactly on the clip has zero body errors, and
    the errors are invariant to the robot's yaw / planar offset about its anchor (BeyondMimic's relative
    frame) but not to a joint deviation."""
    from paper_2601_22074_b200.sim3d.motion import synthetic_walk_clip
    from paper_2601_22074_b200.sim3d.task import MotionTrackingCfg

    m = robots.g1_like()
    O.set_const(m)
    dq = robots.default_qpos(m, robots.G1_DEFAULT_JOINTS)
    Q, V, fdt = synthetic_walk_clip(m, dq, seconds=1.0)
    cfg = MotionTrackingCfg(default_qpos=dq, motion_qpos=Q, motion_qvel=V, motion_dt=fdt, spawn_half_extent=0.0)
    ref = O.MotionTaskOracle(m, cfg, 1, seed=0)
    anchor, bodies = cfg.tracked(m)
    assert m.body_names[anchor] == "torso_link" and len(bodies) == 14
    f = 7
    K = O.kinematics(m, Q[f])
    for k, b in enumerate((anchor,) + bodies):
        np.testing.assert_array_equal(ref.body_table[f, k, 0:3], K["xpos"][b])
    ref.cmd[0] = (f * fdt, 0.0, 0.0)
    ref.qpos[0], ref.qvel[0] = Q[f], V[f]
    np.testing.assert_allclose(ref.body_errors(0), 0.0, atol=1e-20)
    # yaw the whole robot about the world z axis and shift it in the plane: positions / orientations unchanged
    q = Q[f].copy()
    yaw = 0.7
    qz = np.array([np.cos(0.5 * yaw), 0, 0, np.sin(0.5 * yaw)])
    q[0:3] = O.qmat(qz) @ q[0:3] + np.array([0.3, -0.2, 0.0])
    q[3:7] = O.qmul(qz, q[3:7])
    ref.qpos[0], ref.qvel[0] = q, np.zeros(m.nv)
    e = ref.body_errors(0)
    assert e[0] < 1e-20 and e[1] < 1e-20
    q[m.jnt_qposadr[m.jnt_names.index("left_knee_joint")]] += 0.3
    ref.qpos[0] = q
    assert ref.body_errors(0)[0] > 1e-4


def test_contact_sensor_counts_match_pair_bits():
    """Sensor counts from geoms (oracle) == counts through the per-pair bit table the kernel reads."""
    from paper_2601_22074_b200.sim3d.task import MotionTrackingCfg, pair_sensor_bits

    m = robots.g1_like()
    O.set_const(m)
    q = robots.default_qpos(m, robots.G1_DEFAULT_JOINTS)
    q[m.jnt_qposadr[m.jnt_names.index("left_hip_roll_joint")]] = -0.45
    q[m.jnt_qposadr[m.jnt_names.index("right_hip_roll_joint")]] = 0.45
    q[2] -= 0.1  # feet into the ground too
    cfg = MotionTrackingCfg(default_qpos=q, motion_qpos=np.tile(q, (2, 1)), motion_qvel=np.zeros((2, m.nv)),
                            motion_dt=0.02, contact_sensors=(("feet_ground", (4, 5, 6, 7, 10, 11, 12, 13), (0,)),))
    ref = O.MotionTaskOracle(m, cfg, 1)
    cons, _ = O.collide(m, O.kinematics(m, q))
    counts = ref._contact_counts(cons)
    bits = pair_sensor_bits(m, cfg.sensors(m))
    via_bits = [sum(1 for c in cons if (bits[c["pair"]] >> s) & 1) for s in range(2)]
    np.testing.assert_array_equal(counts, via_bits)
    assert counts[0] > 0 and counts[1] > 0


def _rotz(a):
    c, s = np.cos(a), np.sin(a)
    return np.array([[c, -s, 0.0], [s, c, 0.0], [0.0, 0.0, 1.0]])


def _rotx(a):
    c, s = np.cos(a), np.sin(a)
    return np.array([[1.0, 0.0, 0.0], [0.0, c, -s], [0.0, s, c]])


def _roty(a):
    c, s = np.cos(a), np.sin(a)
    return np.array([[c, 0.0, s], [0.0, 1.0, 0.0], [-s, 0.0, c]])


def _inside(x, c, R, h, tol=1e-12):
    return bool(np.all(np.abs(R.T @ (x - c)) <= h + tol))


def test_box_box_face_contacts_analytic():
    """A smaller box pressed 4 mm into a larger one's top face: four contacts at the small box's bottom
    corners (midway into the overlap), depth 4 mm, normal +z; yawed 45 deg and larger than the face, the
    overlap octagon is reduced to four of its corners, all at the same depth."""
    h1, h2, dep = np.array([0.3, 0.2, 0.1]), np.array([0.1, 0.07, 0.05]), 0.004
    c1, R1 = np.zeros(3), np.eye(3)
    c2, R2 = np.array([0.05, -0.02, 0.1 + 0.05 - dep]), _rotz(0.3)
    hits = O.box_box(c1, R1, h1, c2, R2, h2)
    assert len(hits) == 4
    corners = [c2 + R2 @ (np.array([sx, sy, -1.0]) * h2) for sx in (-1, 1) for sy in (-1, 1)]
    for d, n, pos in hits:
        assert abs(d + dep) < 1e-12
        np.testing.assert_allclose(n, [0, 0, 1], atol=1e-12)
        assert min(np.linalg.norm(pos - (cc + np.array([0, 0, dep / 2]))) for cc in corners) < 1e-12
    # wider than box 1 and yawed 45 deg: the overlap is an octagon
    h2 = np.array([0.28, 0.28, 0.05])
    c2, R2 = np.array([0.0, 0.0, 0.1 + 0.05 - dep]), _rotz(np.pi / 4)
    hits = O.box_box(c1, R1, h1, c2, R2, h2)
    assert len(hits) == 4
    for d, n, pos in hits:
        assert abs(d + dep) < 1e-12
        x = pos - np.array([0, 0, dep / 2])  # on box 2's bottom face, inside both footprints
        assert abs(x[2] - (0.1 - dep)) < 1e-12 and np.all(np.abs(x[:2]) <= h1[:2] + 1e-12)
        assert np.all(np.abs((R2.T @ (x - c2))[:2]) <= h2[:2] + 1e-12)


def test_box_box_edge_edge_and_separated():
    """Two edges crossing at right angles (box 1 rolled 45 deg about x, box 2 pitched 45 deg about y and
    pushed down 3 mm): one contact midway between the edges, normal +z, depth 3 mm. Lifted apart: none."""
    h = np.array([0.2, 0.2, 0.2])
    R1, R2 = _rotx(np.pi / 4), _roty(np.pi / 4)
    top = 0.2 * np.sqrt(2.0)
    c1 = np.zeros(3)
    c2 = np.array([0.01, -0.02, 2 * top - 0.003])
    hits = O.box_box(c1, R1, h, c2, R2, h)
    assert len(hits) == 1
    d, n, pos = hits[0]
    assert abs(d + 0.003) < 1e-12
    np.testing.assert_allclose(n, [0, 0, 1], atol=1e-12)
    np.testing.assert_allclose(pos, [0.01, 0.0, top - 0.0015], atol=1e-12)  # box 2 edge x, box 1 edge y
    assert O.box_box(c1, R1, h, c2 + np.array([0, 0, 0.01]), R2, h) == []


def test_box_box_random_poses_contacts_on_and_in_the_boxes(rng):
    """Random overlapping poses: every contact's normal is a unit vector from box 1 towards box 2 with a
    penetration no deeper than the overlap along any of the 15 axes, and the contact's incident point (half
    its depth back along the normal towards the box it belongs to) lies inside the other box."""
    def min_overlap(c1, R1, h1, c2, R2, h2):
        axes = [R1[:, i] for i in range(3)] + [R2[:, j] for j in range(3)]
        axes += [np.cross(R1[:, i], R2[:, j]) for i in range(3) for j in range(3)]
        return min(h1 @ np.abs(R1.T @ u) + h2 @ np.abs(R2.T @ u) - abs(u @ (c2 - c1))
                   for u in (a / np.linalg.norm(a) for a in axes if np.linalg.norm(a) > 1e-6))

    seen = 0
    for _ in range(300):
        h1, h2 = rng.uniform(0.05, 0.3, size=3), rng.uniform(0.05, 0.3, size=3)
        q1, q2 = rng.normal(size=4), rng.normal(size=4)
        R1, R2 = O.qmat(q1 / np.linalg.norm(q1)), O.qmat(q2 / np.linalg.norm(q2))
        c1 = np.zeros(3)
        u = rng.normal(size=3)
        u /= np.linalg.norm(u)
        target, lo_t, hi_t = rng.uniform(0.001, 0.02), 0.0, 2.0  # a shallow overlap (bisection on the offset)
        for _ in range(60):
            mid = 0.5 * (lo_t + hi_t)
            lo_t, hi_t = (mid, hi_t) if min_overlap(c1, R1, h1, mid * u, R2, h2) > target else (lo_t, mid)
        c2 = lo_t * u
        hits = O.box_box(c1, R1, h1, c2, R2, h2)
        assert hits
        for d, n, pos in hits:
            seen += 1
            assert d <= 0.0 and abs(np.linalg.norm(n) - 1.0) < 1e-12
            lo, hi = pos - n * (-d / 2), pos + n * (-d / 2)  # the two surface points along the normal
            # box 2's incident point inside box 1 (box 1 the reference), or box 1's inside box 2
            assert _inside(lo, c1, R1, h1, 1e-9) or _inside(hi, c2, R2, h2, 1e-9)
            axes = [R1[:, i] for i in range(3)] + [R2[:, j] for j in range(3)]
            axes += [np.cross(R1[:, i], R2[:, j]) for i in range(3) for j in range(3)]
            ovs = []
            for u in axes:
                if np.linalg.norm(u) < 1e-6:
                    continue
                u = u / np.linalg.norm(u)
                ovs.append(h1 @ np.abs(R1.T @ u) + h2 @ np.abs(R2.T @ u) - abs(u @ (c2 - c1)))
            assert -d <= min(ovs) / O.BOX_FACE_BIAS + 1e-12
    assert seen > 100


def test_box_stack_settles():
    """Three free boxes stacked 2 mm into each other at different yaws (box-box + box-plane contacts)
    push apart to the soft-contact equilibrium and stay stacked: no drift, no spin, velocities ~0."""
    m = robots.box_stack()
    O.set_const(m)
    q, v, w = m.qpos0.copy(), np.zeros(m.nv), np.zeros(m.nv)
    for _ in range(300):
        q, v, w, F = O.step(m, q, v, np.zeros(0), warm=w)
    dq = q - m.qpos0
    for j in range(m.njnt):
        a = m.jnt_qposadr[j]
        assert np.abs(dq[a:a + 2]).max() < 1e-4           # no sliding
        assert 0.0 < dq[a + 2] < 0.002 * (j + 1) + 1e-4    # rose out of the initial overlap, no more
        assert np.abs(dq[a + 3:a + 7]).max() < 1e-4        # no spin / tilt
    assert np.abs(v).max() < 1e-3
    assert sum(1 for c in F["contacts"] if c["geom1"] != 0) == 8  # 4 per box-box face contact


def test_centroidal_angular_momentum_is_fd_of_fk(model, rng):
    """The velocity task's angular momentum (sum over the robot's bodies of cinert x cvel, angular part about
    the tree's com) equals sum_b I_b w_b + m_b (x_b - c) x v_b with every body's com velocity and angular
    velocity from finite differences of FK."""
    from paper_2601_22074_b200.sim3d.task import VelocityTaskCfg

    m = model
    q, v = _random_state(m, rng)
    cfg = VelocityTaskCfg(default_qpos=m.qpos0.copy(), reward_weights=(0,) * 6 + (1.0, 0.0, 0.0), feet=())
    ref = O.TaskOracle(m, cfg, 1)
    ref.qpos[0], ref.qvel[0] = q, v
    h2, _, _ = ref.velocity_extras(0, np.zeros(0))
    K = O.kinematics(m, q)
    C = O.com_pos(m, K)
    dt = 1e-6
    Kp, Km = O.kinematics(m, O.integrate_pos(m, q, v, dt)), O.kinematics(m, O.integrate_pos(m, q, v, -dt))
    c = C["com"][0]
    h = np.zeros(3)
    for b in range(1, m.nbody):
        if m.body_treeid[b] != 0:
            continue
        R = K["ximat"][b]
        W = (Kp["ximat"][b] - Km["ximat"][b]) / (2 * dt) @ R.T
        wb = np.array([W[2, 1], W[0, 2], W[1, 0]])
        vb = (Kp["xipos"][b] - Km["xipos"][b]) / (2 * dt)
        I = R @ np.diag(m.body_inertia[b]) @ R.T
        h += I @ wb + m.body_mass[b] * np.cross(K["xipos"][b] - c, vb)
    assert abs(h2 - h @ h) < 1e-6 * max(1.0, h @ h)


@pytest.mark.parametrize("name", ["g1", "box_stack"])
def test_cg_solver_reaches_the_newton_optimum(name, rng):
    """The conjugate-gradient solver (Opt.solver="cg", mj_solCG restated) minimises the same constrained
    cost as Newton: with enough iterations both stop at the tolerance with the same accelerations and a
    non-increasing cost along the way; CG never forms the Hessian, so it needs more iterations."""
    from paper_2601_22074_b200.sim3d.model import Opt

    make = {"g1": lambda o: robots.g1_like(opt=o), "box_stack": lambda o: robots.box_stack(opt=o)}[name]
    mn, mc = make(Opt(iterations=200)), make(Opt(iterations=200, solver="cg"))
    O.set_const(mn)
    O.set_const(mc)
    q, v = mn.qpos0.copy(), rng.normal(size=mn.nv) * 0.1
    if name == "g1":
        q = robots.default_qpos(mn, robots.G1_DEFAULT_JOINTS)
        q[2] -= 0.02
    else:
        q[2] -= 0.003
    ctrl = q[mn.actuator_qposadr] if mn.nu else np.zeros(1)
    Fn, Fc = O.forward(mn, q, v, ctrl), O.forward(mc, q, v, ctrl)
    assert Fc["iterations"] > Fn["iterations"] and len(Fn["contacts"]) > 0
    sc = np.abs(Fn["qacc"]).max()
    assert np.abs(Fn["qacc"] - Fc["qacc"]).max() < 1e-3 * sc


def _ball_on_slope(condim, tilt=0.3):
    """A ball resting 1 mm into a plane tilted by `tilt` about x (gravity rotated instead of the plane)."""
    from paper_2601_22074_b200.sim3d.model import Opt

    g = 9.81
    b = ModelBuilder("ball", Opt(gravity=(0.0, g * np.sin(tilt), -g * np.cos(tilt)), iterations=50))
    b.plane(friction=1.0, condim=condim)  # both geoms: a pair takes the larger condim
    ball = b.body("ball", 0, pos=(0, 0, 0.099), mass=1.0, inertia=(0.004, 0.004, 0.004))
    b.free_joint(ball)
    b.geom(ball, GEOM_SPHERE, (0.1,), friction=1.0, condim=condim)
    m = b.compile()
    O.set_const(m)
    return m


def test_condim1_frictionless_contact_equals_one_normal_row():
    """condim 1: the contact's 4 pyramid rows (mu = 0, 4x the normal row's R each) minimise exactly the cost
    of MuJoCo's single frictionless row -- same accelerations as the one-row problem -- and the ball slides
    down the slope without rolling (tangential acceleration g sin(tilt), no spin), while condim 3 rolls."""
    m1, m3 = _ball_on_slope(1), _ball_on_slope(3)
    q, v = m1.qpos0.copy(), np.zeros(m1.nv)
    F1 = O.forward(m1, q, v, np.zeros(1))
    E = F1["efc"]
    assert E["nefc"] == 4 and np.allclose(E["J"], E["J"][0]) and np.allclose(E["D"], E["D"][0])
    E1 = dict(E, J=E["J"][:1], D=4.0 * E["D"][:1], aref=E["aref"][:1], nefc=1)
    a1, _, _, _ = O.newton(m1, F1["M"], E1, F1["qfrc_smooth"], None, None)
    np.testing.assert_allclose(F1["qacc"], a1, rtol=1e-9, atol=1e-12)
    tilt, g = 0.3, 9.81
    assert abs(F1["qacc"][1] - g * np.sin(tilt)) < 1e-6 and np.abs(F1["qacc"][3:6]).max() < 1e-9
    F3 = O.forward(m3, q, v, np.zeros(1))
    assert F3["qacc"][1] < 0.8 * g * np.sin(tilt) and np.abs(F3["qacc"][3:6]).max() > 1.0  # rolls
