"""Host-side tables of the 3-D kernel (sim3d/device.py), checked on CPU without a GPU: the
factorization update lists, the level schedules and the pair/Jacobian tables drive numpy
re-implementations of the kernel's loops, which must reproduce the oracle's L^T D L and solves."""

import ctypes

import numpy as np
import pytest

from oracle import sim3d as O
from paper_2601_22074_b200.sim3d import robots
from paper_2601_22074_b200.sim3d.device import DeviceModel
from paper_2601_22074_b200.sim3d.model import ModelBuilder, ModelError, GEOM_SPHERE

MODELS = {"g1": robots.g1_like, "go1": robots.go1_like, "arm_cube": robots.arm_cube_like}


def _tables(dm):
    """Read back the packed device buffer (CPU tensor) by table name."""
    buf = dm.buffer.numpy()
    s = dm.struct
    base = dm.buffer.data_ptr()

    def arr(name, dtype, n):
        off = getattr(s, name) - base
        return np.frombuffer(buf[off:off + n * np.dtype(dtype).itemsize].tobytes(), dtype=dtype)
    return arr


def _random_M(m, rng):
    q = m.qpos0.copy()
    q[m.jnt_qposadr[m.jnt_type == 3]] = rng.uniform(-1, 1, size=int((m.jnt_type == 3).sum()))
    return O.crb(m, O.com_pos(m, O.kinematics(m, q)))[0]


@pytest.mark.parametrize("name", list(MODELS))
def test_ldl_update_lists_reproduce_the_oracle_factor(name, rng):
    m = MODELS[name]()
    dm = DeviceModel(m, "f64", device="cpu")
    arr = _tables(dm)
    nv = m.nv
    ldl_ptr = arr("ldl_ptr", np.int32, nv + 1)
    ldl_pair = arr("ldl_pair", np.uint16, int(ldl_ptr[-1]))
    norm = arr("ldl_norm", np.uint16, dm.struct.nldl_norm)
    M = _random_M(m, rng)
    A = M.copy()
    for k in range(nv - 1, -1, -1):  # the kernel's sequential schedule, row normalisation deferred
        for t in range(ldl_ptr[k], ldl_ptr[k + 1]):
            i, j = int(ldl_pair[t]) >> 8, int(ldl_pair[t]) & 255
            A[i, j] -= (A[k, i] / A[k, k]) * A[k, j]
    for t in norm:
        k, i = int(t) >> 8, int(t) & 255
        A[k, i] /= A[k, k]
    L = O.factor_ldl(m, M)
    tree = np.zeros_like(M, dtype=bool)
    for i in range(nv):
        tree[i, m.dof_chain[i]] = True
    np.testing.assert_allclose(A[tree], L[tree], rtol=1e-12, atol=1e-14)


@pytest.mark.parametrize("name", list(MODELS))
def test_level_schedules_reproduce_factor_and_solve(name, rng):
    m = MODELS[name]()
    dm = DeviceModel(m, "f64", device="cpu")
    arr = _tables(dm)
    s = dm.struct
    nh, nd = s.nhlev, s.ndlev
    fl_ptr = arr("fl_ptr", np.int32, nh + 1)
    fl_ent = arr("fl_ent", np.uint16, int(fl_ptr[-1]))
    fl_kptr = arr("fl_kptr", np.int32, int(fl_ptr[-1]) + 1)
    fl_k = arr("fl_k", np.uint8, int(fl_kptr[-1]))
    bl_ptr = arr("bl_ptr", np.int32, nh + 1)
    bl_ent = arr("bl_ent", np.uint8, int(bl_ptr[-1]))
    bl_iptr = arr("bl_iptr", np.int32, int(bl_ptr[-1]) + 1)
    bl_i = arr("bl_i", np.uint8, int(bl_iptr[-1]))
    fw_ptr = arr("fw_ptr", np.int32, nd + 1)
    fw_dof = arr("fw_dof", np.uint8, int(fw_ptr[-1]))
    M = _random_M(m, rng)
    A = M.copy()
    for L_ in range(nh):  # all contributions of a level read the pre-level state
        upd = {}
        for e in range(fl_ptr[L_], fl_ptr[L_ + 1]):
            i, j = int(fl_ent[e]) >> 8, int(fl_ent[e]) & 255
            upd[(i, j)] = sum((A[k, i] / A[k, k]) * A[k, j] for k in fl_k[fl_kptr[e]:fl_kptr[e + 1]])
        for (i, j), v in upd.items():
            A[i, j] -= v
    for k in range(m.nv):
        for i in m.dof_chain[k][:-1]:
            A[k, i] /= A[k, k]
    Lo = O.factor_ldl(m, M)
    for i in range(m.nv):
        np.testing.assert_allclose(A[i, m.dof_chain[i]], Lo[i, m.dof_chain[i]], rtol=1e-11, atol=1e-13)
    b = rng.normal(size=m.nv)
    x = b.copy()
    for L_ in range(nh):
        for e in range(bl_ptr[L_], bl_ptr[L_ + 1]):
            j = int(bl_ent[e])
            x[j] -= sum(Lo[i, j] * x[i] for i in bl_i[bl_iptr[e]:bl_iptr[e + 1]])
    x /= np.diag(Lo)
    for L_ in range(1, nd):
        for i in fw_dof[fw_ptr[L_]:fw_ptr[L_ + 1]]:
            x[i] -= sum(Lo[i, j] * x[j] for j in m.dof_chain[i][:-1])
    np.testing.assert_allclose(x, np.linalg.solve(M, b), rtol=1e-9, atol=1e-12)


@pytest.mark.parametrize("name", list(MODELS))
def test_pair_tables(name):
    m = MODELS[name]()
    dm = DeviceModel(m, "f64", device="cpu")
    arr = _tables(dm)
    npair = m.npair
    tree = arr("pair_tree", np.int32, npair)
    cls = arr("pair_class", np.int32, npair)
    mask = arr("pair_dofmask", np.uint64, npair)
    for p, (g1, g2) in enumerate(m.pair_geom):
        chain = m.pair_chain[p]
        assert int(mask[p]) == sum(1 << d for d in chain)
        c1, c2 = set(m.body_chain[m.geom_bodyid[g1]]), set(m.body_chain[m.geom_bodyid[g2]])
        assert tree[p] == int(c1 <= c2 or c2 <= c1)
        same = [q for q in range(npair) if m.pair_chain[q] == chain]
        assert all(cls[q] == cls[p] for q in same)
    if name == "g1":
        assert not tree.all()  # self pairs couple branches (dense Cholesky fallback exists for them)


def test_model_errors():
    b = ModelBuilder("bad")
    with pytest.raises(ModelError):
        b.body("x", "nope")
    b.plane()
    ball = b.body("ball", 0, pos=(0, 0, 1))
    b.free_joint(ball)
    b.geom(ball, GEOM_SPHERE, (0.1,))
    child = b.body("child", ball)
    with pytest.raises(ModelError):
        b.free_joint(child)  # free joints only on children of the world
    with pytest.raises(ModelError):
        b.actuator("ball_free")  # actuators drive hinges
    b2 = ModelBuilder("noterrain")
    c = b2.body("c", 0)
    b2.geom(c, GEOM_SPHERE, (0.1,))
    with pytest.raises(ModelError):
        b2.compile()  # exactly one terrain geom, first


def test_layout_fits_and_struct_sizes():
    from paper_2601_22074_b200.sim3d import native as N

    for name, make in MODELS.items():
        for dtype, esz in (("f32", 4), ("f64", 8)):
            dm = DeviceModel(make(), dtype, device="cpu")
            lay = dm.layout
            assert lay.bytes_per_block == lay.elems_per_world * esz * lay.warps_per_block <= 227 * 1024
            # O_XPOS .. O_INT: the per-world regions, in order (8-10 hold RNE offsets inside the Jacobian region;
            # the row buffers 27-30 may reuse dead slots: aref / D / J·a after the factorization snapshot in the
            # xipos .. jax region, the force buffer in cdof's slot; 36 is the CG solver's vectors, empty unless
            # flags bit 7)
            offs = [lay.off[k] for k in range(38) if k not in (8, 9, 10, 27, 28, 29, 30)]
            assert offs == sorted(offs) and offs[-1] < lay.elems_per_world
            dm_s = dm.struct
            nrow = min(dm_s.nlimjnt, 32) + 4 * dm_s.ncon_max
            nre = (nrow + 1) & ~1
            raref, rd, rjar, rjp = (lay.off[k] for k in (27, 28, 29, 30))
            assert rd - raref >= nrow and rjar - rd >= nrow
            if raref < lay.off[6]:  # in the snapshot region, after the ntree snapshot entries
                assert raref >= lay.off[2] + dm_s.ntree and rjar + nre <= lay.off[6]
            if rjp == lay.off[7]:  # in cdof's slot
                assert 6 * dm_s.nv >= nrow
            # int region: con_pair, lim_dof, lim_sign (int offsets)
            assert lay.off[38] == dm_s.ncon_max and lay.off[39] == dm_s.ncon_max + min(dm_s.nlimjnt, 32)
            assert lay.off[37] - lay.off[36] == (2 * dm_s.nv if dm_s.flags & 128 else 0)
    assert N.lib().s3_sizeof(3) == ctypes.sizeof(N.TaskT)
