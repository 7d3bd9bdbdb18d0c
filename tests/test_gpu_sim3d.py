"""3-D path: the sm_100a warp-per-world step vs the numpy oracle (oracle/sim3d.py).

Parity is unpinned w.r.t. the reference (it has no 3-D engine);
these tests pin the CUDA kernel to the oracle, which is itself pinned by
analytic properties (tests/test_sim3d_oracle_cpu.py). Tolerances:

* float64 kernel, one substep from identical state: every intermediate
  (frames, com, cdof, M, its L^T D L factor, bias, smooth force, contacts,
  constraint forces, qacc, next qpos/qvel) within 1e-9 relative to the
  quantity's scale; contact pair sets and nefc bit-exact;
* float64, 40-substep rollout: qpos within 1e-6;
* float32 kernel (throughput build), one substep: M within 1e-5, qacc within
  2e-3 of the qacc scale, next qvel within 1e-3 * max(1, |qvel|).
"""

import ctypes

import numpy as np
import pytest

from oracle import sim3d as O
from paper_2601_22074_b200.sim3d import robots
from paper_2601_22074_b200.sim3d.model import MAX_CON, Opt

ROBOTS = {
    "g1_flat": (lambda: robots.g1_like(), robots.G1_DEFAULT_JOINTS),
    "g1_rough": (lambda: robots.g1_like(rough=True, seed=3), robots.G1_DEFAULT_JOINTS),
    "go1_flat": (lambda: robots.go1_like(), robots.GO1_DEFAULT_JOINTS),
    "arm_cube": (lambda: robots.arm_cube_like(), robots.ARM_DEFAULT_JOINTS),
    "box_stack": (lambda: robots.box_stack(), {}),
    # the conjugate-gradient solver (Opt.solver = "cg", s3_model.flags bit 7)
    "g1_flat_cg": (lambda: robots.g1_like(opt=Opt(solver="cg")), robots.G1_DEFAULT_JOINTS),
    "box_stack_cg": (lambda: robots.box_stack(opt=Opt(solver="cg")), {}),
    # frictionless (condim 1) contact between the upper two boxes
    "box_stack_condim1": (lambda: robots.box_stack(condims=(3, 1, 1)), {}),
}


def _box_states(m, n, rng):
    """The stack jittered: each box shifted a few mm, sunk up to 3 mm more, tilted up to ~3 deg (no two
    box faces parallel, so the separating-axis choice has no ties), random velocities."""
    Q, V = [], []
    for w in range(n):
        q = m.qpos0.copy()
        for j in range(m.njnt):
            a = m.jnt_qposadr[j]
            q[a:a + 2] += rng.normal(size=2) * 0.003
            q[a + 2] -= rng.uniform(0.0, 0.003)
            ax = rng.normal(size=3)
            q[a + 3:a + 7] = O.qmul(O.qaxisangle(ax / np.linalg.norm(ax), rng.uniform(0.01, 0.05)), q[a + 3:a + 7])
        Q.append(q)
        V.append(rng.normal(size=m.nv) * 0.2)
    return np.array(Q), np.array(V), np.zeros((n, 1))  # Data keeps one ctrl column when nu = 0


def _arm_states(m, table, n, rng):
    """Arm near its default pose; the cube on the table (pressed), between the fingertips, or lifted."""
    q0 = robots.default_qpos(m, table)
    Q, V = [], []
    hinge = m.jnt_qposadr[m.jnt_type == 3]
    K = O.kinematics(m, q0)
    tips = [g for g in range(m.ngeom) if m.geom_type[g] == 2]
    mid = K["geom_xpos"][tips].mean(0)
    for w in range(n):
        q = q0.copy()
        q[hinge] += rng.uniform(-0.05, 0.05, size=hinge.size)
        if w % 3 == 0:
            q[-7:-4] = (0.55 + rng.uniform(-0.05, 0.05), rng.uniform(-0.05, 0.05), 0.025 - 0.003)
        else:  # cube between / against the fingertips
            q[-7:-4] = mid + rng.uniform(-0.01, 0.01, size=3)
        if w % 4 == 3:  # a joint past its limit
            j = np.nonzero(m.jnt_limited)[0][w % m.nlim]
            q[m.jnt_qposadr[j]] = m.jnt_range[j][w % 2] + (0.05 if w % 2 else -0.05)
        Q.append(q)
        V.append(rng.normal(size=m.nv) * 0.2)
    ctrl = np.array([q0[m.actuator_qposadr] + rng.uniform(-0.1, 0.1, size=m.nu) for _ in range(n)])
    return np.array(Q), np.array(V), ctrl


def _states(m, table, n, seed):
    """Standing poses pressed into the ground, jittered joints, random velocities; some worlds tilted
    and sunk deep so that limits, self contacts and many terrain contacts occur."""
    rng = np.random.default_rng(seed)
    if m.name == "arm_cube_like":
        return _arm_states(m, table, n, rng)
    if m.name == "box_stack":
        return _box_states(m, n, rng)
    q0 = robots.default_qpos(m, table)
    K = O.kinematics(m, q0)
    low = min(K["geom_xpos"][g][2] - m.geom_rbound[g] for g in range(1, m.ngeom))
    Q, V = [], []
    for w in range(n):
        q = q0.copy()
        q[2] -= low + 0.004 + 0.01 * rng.uniform()
        q[0:2] += rng.uniform(-0.5, 0.5, size=2)
        hinge = m.jnt_qposadr[m.jnt_type == 3]
        q[hinge] += rng.uniform(-0.3, 0.3, size=hinge.size)
        if w % 3 == 2:  # push some joints past their limits
            j = np.nonzero(m.jnt_limited)[0][w % m.nlim]
            q[m.jnt_qposadr[j]] = m.jnt_range[j][w % 2] + (0.05 if w % 2 else -0.05)
        if w % 4 == 3:  # tilt
            ax = rng.normal(size=3)
            quat = O.qaxisangle(ax / np.linalg.norm(ax), 0.4)
            q[3:7] = O.qmul(quat, q[3:7])
        v = rng.normal(size=m.nv) * 0.3
        Q.append(q)
        V.append(v)
    ctrl = np.array([q0[m.actuator_qposadr] + rng.uniform(-0.2, 0.2, size=m.nu) for _ in range(n)])
    return np.array(Q), np.array(V), ctrl


def _setup(name, dtype, n, seed=0):
    import torch

    from paper_2601_22074_b200.sim3d.device import Data, DeviceModel

    make, table = ROBOTS[name]
    m_gpu = make()
    dm = DeviceModel(m_gpu, dtype)
    dm.set_const()
    m = make()  # oracle copy with its own inverse weights
    O.set_const(m)
    Q, V, C = _states(m, table, n, seed)
    d = Data(dm, n)
    d.qpos.copy_(torch.as_tensor(Q))
    d.qvel.copy_(torch.as_tensor(V))
    d.ctrl.copy_(torch.as_tensor(C))
    return m, dm, d, Q, V, C


def _rel(a, b):
    if np.size(b) == 0:
        return 0.0
    return np.max(np.abs(a - b)) / max(1.0, np.max(np.abs(b)))


@pytest.mark.gpu
@pytest.mark.parametrize("name", list(ROBOTS))
def test_inverse_weights_match_oracle(name):
    from paper_2601_22074_b200.sim3d.device import DeviceModel

    make, _ = ROBOTS[name]
    mg, mo = make(), make()
    DeviceModel(mg, "f64").set_const()
    O.set_const(mo)
    np.testing.assert_allclose(mg.dof_invweight0, mo.dof_invweight0, rtol=1e-10)
    np.testing.assert_allclose(mg.body_invweight0, mo.body_invweight0, rtol=1e-10, atol=1e-14)
    assert abs(mg.meaninertia - mo.meaninertia) < 1e-12 * mo.meaninertia


@pytest.mark.gpu
@pytest.mark.parametrize("name", list(ROBOTS))
def test_single_substep_f64_all_stages(name):
    import torch

    from paper_2601_22074_b200.sim3d.device import unpack_lower

    n = 12
    m, dm, d, Q, V, C = _setup(name, "f64", n)
    out = d.step(1, outputs=True)
    torch.cuda.synchronize()
    out = {k: v.cpu().numpy() for k, v in out.items()}
    qn, vn = d.qpos.cpu().numpy(), d.qvel.cpu().numpy()
    saw_contacts = saw_limits = saw_self = 0
    for w in range(n):
        q1, v1, _, F = O.step(m, Q[w], V[w], C[w], warm=np.zeros(m.nv))
        K, Cc = F["K"], F["C"]
        np.testing.assert_allclose(out["xpos"][w], K["xpos"], atol=1e-12)
        np.testing.assert_allclose(out["xquat"][w], K["xquat"], atol=1e-12)
        np.testing.assert_allclose(out["com"][w][:m.ntree], Cc["com"], atol=1e-12)
        np.testing.assert_allclose(out["cdof"][w], Cc["cdof"], atol=1e-12)
        Mg = unpack_lower(out["qM"][w], m.nv)
        assert _rel(Mg, F["M"]) < 1e-12
        Lg = np.zeros((m.nv, m.nv))
        Lg[np.tril_indices(m.nv)] = out["qLD"][w]
        assert _rel(Lg, np.tril(F["qLD"])) < 1e-10
        assert _rel(out["qfrc_bias"][w], F["bias"]) < 1e-10
        assert _rel(out["qfrc_smooth"][w], F["qfrc_smooth"]) < 1e-10
        assert _rel(out["qacc_smooth"][w], F["qacc_smooth"]) < 1e-9
        # contacts: pair sets bit-exact, geometry to 1e-12
        nc = int(out["ncon"][w])
        cons = F["contacts"]
        assert nc == len(cons) and int(out["ndropped"][w]) == F["dropped"]
        assert [c["pair"] for c in cons] == out["con_pair"][w][:nc].tolist()
        for k, c in enumerate(cons):
            assert abs(out["con_dist"][w][k] - c["dist"]) < 1e-12
            np.testing.assert_allclose(out["con_pos"][w][k], c["pos"], atol=1e-12)
            np.testing.assert_allclose(out["con_frame"][w][k].reshape(3, 3), c["frame"], atol=1e-12)
        E = F["efc"]
        assert int(out["nefc"][w]) == E["nefc"]
        saw_contacts += nc > 0
        saw_limits += E["nlim"] > 0
        saw_self += any(c["geom1"] != 0 for c in cons)
        assert _rel(out["efc_force"][w][:E["nefc"]], F["efc_force"]) < 1e-8
        assert _rel(out["qacc"][w], F["qacc"]) < 1e-8
        assert _rel(out["qfrc_constraint"][w], F["qfrc_constraint"]) < 1e-8
        assert _rel(vn[w], v1) < 1e-9
        assert _rel(qn[w], q1) < 1e-11
    assert saw_contacts >= n // 2 and (saw_limits > 0 or m.nlim == 0)
    if m.name == "box_stack":  # box-box contacts (geom pairs of two boxes) in every world
        assert any(m.pair_condim[c["pair"]] == 1 for c in cons) or m.pair_condim.min() == 3
        assert saw_self == n


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["g1_rough", "go1_flat", "arm_cube", "box_stack"])
def test_rollout_f64(name):
    import torch

    n = 6
    m, dm, d, Q, V, C = _setup(name, "f64", n, seed=5)
    steps = 40
    for _ in range(steps // 4):
        d.step(4)
    torch.cuda.synchronize()
    qn = d.qpos.cpu().numpy()
    for w in range(n):
        q, v, warm = Q[w], V[w], np.zeros(m.nv)
        for _ in range(steps):
            q, v, warm, _ = O.step(m, q, v, C[w], warm=warm)
        assert np.max(np.abs(qn[w] - q)) < 1e-6, (w, np.max(np.abs(qn[w] - q)))


@pytest.mark.gpu
@pytest.mark.parametrize("name", [r for r in ROBOTS if not r.endswith("_cg")])  # CG stops at its iteration
def test_single_substep_f32(name):  # cap short of the optimum: f32 rounding steers it elsewhere (f64 pinned above)
    import torch

    from paper_2601_22074_b200.sim3d.device import unpack_lower

    n = 12
    m, dm, d, Q, V, C = _setup(name, "f32", n)
    out = d.step(1, outputs=True)
    torch.cuda.synchronize()
    out = {k: v.double().cpu().numpy() if v.is_floating_point() else v.cpu().numpy() for k, v in out.items()}
    vn = d.qvel.double().cpu().numpy()
    # the oracle runs on the float32-rounded inputs
    Q32, V32, C32 = (x.astype(np.float32).astype(np.float64) for x in (Q, V, C))
    for w in range(n):
        q1, v1, _, F = O.step(m, Q32[w], V32[w], C32[w], warm=np.zeros(m.nv))
        assert _rel(unpack_lower(out["qM"][w], m.nv), F["M"]) < 1e-5
        assert int(out["ncon"][w]) == len(F["contacts"])
        sc = max(1.0, np.max(np.abs(F["qacc"])))
        assert np.max(np.abs(out["qacc"][w] - F["qacc"])) < 2e-3 * sc
        assert np.max(np.abs(vn[w] - v1)) < 1e-3 * max(1.0, np.max(np.abs(v1)))


@pytest.mark.gpu
def test_contact_capacity_drops_in_pair_order():
    """A humanoid lying flat touches with more than ncon_max points: the kernel keeps the first
    ncon_max in pair order and counts the rest, exactly like the oracle."""
    import torch

    n = 2
    m, dm, d, Q, V, C = _setup("g1_flat", "f64", n)
    q = Q.copy()
    hinge = m.jnt_qposadr[m.jnt_type == 3]
    for w in range(n):
        q[w, hinge] = 0.0
        q[w, 3:7] = O.qaxisangle(np.array([0, 1.0, 0]), np.pi / 2)
        q[w, 2] = -0.01 * w
    d.qpos.copy_(torch.as_tensor(q))
    out = d.step(1, outputs=True)
    torch.cuda.synchronize()
    for w in range(n):
        _, _, _, F = O.step(m, q[w], V[w], C[w], warm=np.zeros(m.nv))
        assert int(out["ncon"][w]) == len(F["contacts"]) == m.ncon_max
        assert int(out["ndropped"][w]) == F["dropped"] > 0


@pytest.mark.gpu
def test_batched_equals_solo():
    """World independence: a world stepped in a batch equals the same world stepped alone (bitwise)."""
    import torch

    from paper_2601_22074_b200.sim3d.device import Data

    m, dm, d, Q, V, C = _setup("g1_rough", "f64", 9, seed=2)
    for _ in range(3):
        d.step(4)
    solo = Data(dm, 1)
    solo.qpos.copy_(torch.as_tensor(Q[4:5]))
    solo.qvel.copy_(torch.as_tensor(V[4:5]))
    solo.ctrl.copy_(torch.as_tensor(C[4:5]))
    for _ in range(3):
        solo.step(4)
    torch.cuda.synchronize()
    assert torch.equal(solo.qpos[0], d.qpos[4]) and torch.equal(solo.qvel[0], d.qvel[4])


def test_sim3d_library_exports_and_plans_on_cpu():
    """The C-ABI loads, exports what the header declares, and plans a layout (no GPU needed)."""
    from paper_2601_22074_b200.sim3d import native as N
    from paper_2601_22074_b200.sim3d.device import DeviceModel

    so = N.lib()
    for name in N.EXPORTED:
        assert hasattr(so, name)
    dm = DeviceModel(robots.g1_like(), "f64", device="cpu")
    lay = dm.layout
    assert lay.warps_per_block >= 1 and lay.bytes_per_block <= 227 * 1024
    assert lay.elems_per_world * 8 * lay.warps_per_block == lay.bytes_per_block
    dm32 = DeviceModel(robots.g1_like(), "f32", device="cpu")
    assert dm32.layout.warps_per_block >= lay.warps_per_block
    bad = N.ModelT()
    ctypes.memmove(ctypes.byref(bad), ctypes.byref(dm.struct), ctypes.sizeof(bad))
    bad.nv = 65
    with pytest.raises(N.NativeError):
        N.call("s3_plan", ctypes.byref(bad), 0, ctypes.byref(N.LayoutT()))


@pytest.mark.gpu
@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_self_contacts_take_the_dense_newton_path(dtype):
    """Crossed shins (a self pair coupling both legs) break the tree pattern of H = M + J^T D J; the
    kernel falls back to the dense Cholesky for that Newton solve -- still equal to the oracle."""
    import torch

    from paper_2601_22074_b200.sim3d.device import Data, DeviceModel

    mg, m = robots.g1_like(), robots.g1_like()
    dm = DeviceModel(mg, dtype)
    dm.set_const()
    O.set_const(m)
    q = robots.default_qpos(m, robots.G1_DEFAULT_JOINTS)
    q[m.jnt_qposadr[m.jnt_names.index("left_hip_roll_joint")]] = -0.45
    q[m.jnt_qposadr[m.jnt_names.index("right_hip_roll_joint")]] = 0.45
    K = O.kinematics(m, q)
    low = min(K["geom_xpos"][g][2] - m.geom_rbound[g] for g in range(1, m.ngeom))
    q[2] -= low + 0.004
    n = 4
    rng = np.random.default_rng(3)
    V = rng.normal(size=(n, m.nv)) * 0.2
    d = Data(dm, n)
    d.qpos.copy_(torch.as_tensor(np.tile(q, (n, 1))))
    d.qvel.copy_(torch.as_tensor(V))
    ctrl = np.tile(q[m.actuator_qposadr], (n, 1))
    d.ctrl.copy_(torch.as_tensor(ctrl))
    out = d.step(1, outputs=True)
    torch.cuda.synchronize()
    tol = 1e-8 if dtype == "f64" else 3e-3
    for w in range(n):
        _, v1, _, F = O.step(m, q, V[w], ctrl[w], warm=np.zeros(m.nv))
        cons = F["contacts"]
        assert any(c["geom1"] != 0 for c in cons)  # a robot-robot (self) contact is present
        assert int(out["ncon"][w]) == len(cons)
        qa = out["qacc"][w].double().cpu().numpy()
        assert np.max(np.abs(qa - F["qacc"])) < tol * max(1.0, np.max(np.abs(F["qacc"])))
