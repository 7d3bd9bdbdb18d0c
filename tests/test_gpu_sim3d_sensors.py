"""3-D ray-cast sensors (height scan rays, depth camera) vs the oracle's raycast specification.

Parity unpinned w.r.t. the reference (its RayScanner is vertical probes on a
1-D heightfield, sensors.py:26-46; there is no depth camera).
float64: hit geoms bit-exact, distances within 1e-9 (heightfield hits are
bisection-limited to spacing * 0.5 / 2^24).
"""

import numpy as np
import pytest

from oracle import sim3d as O
from paper_2601_22074_b200.sim3d import robots


def _setup(n=4, seed=0):
    import torch

    from paper_2601_22074_b200.sim3d.device import Data, DeviceModel

    mg, mo = robots.g1_like(rough=True, seed=2), robots.g1_like(rough=True, seed=2)
    dm = DeviceModel(mg, "f64")
    dm.set_const()
    O.set_const(mo)
    rng = np.random.default_rng(seed)
    q0 = robots.default_qpos(mo, robots.G1_DEFAULT_JOINTS)
    Q = np.tile(q0, (n, 1))
    Q[:, 0:2] += rng.uniform(-3, 3, size=(n, 2))
    hinge = mo.jnt_qposadr[mo.jnt_type == 3]
    Q[:, hinge] += rng.uniform(-0.5, 0.5, size=(n, hinge.size))
    d = Data(dm, n)
    d.enable_geom_frames()
    d.qpos.copy_(torch.as_tensor(Q))
    d.ctrl.copy_(torch.as_tensor(np.tile(q0[mo.actuator_qposadr], (n, 1))))
    d.step(1)
    torch.cuda.synchronize()
    return mo, dm, d


@pytest.mark.gpu
def test_geom_frames_are_final_state_kinematics():
    import torch

    m, dm, d = _setup()
    q = d.qpos.cpu().numpy()
    gp, gm = d.geom_xpos.cpu().numpy(), d.geom_xmat.cpu().numpy()
    for w in range(d.nworld):
        K = O.kinematics(m, q[w])
        np.testing.assert_allclose(gp[w], K["geom_xpos"], atol=1e-12)
        np.testing.assert_allclose(gm[w].reshape(-1, 3, 3), K["geom_xmat"], atol=1e-12)


@pytest.mark.gpu
def test_random_rays_match_oracle():
    import torch

    from paper_2601_22074_b200.sim3d.sensors import RayCaster

    m, dm, d = _setup()
    n, r = d.nworld, 96
    rng = np.random.default_rng(1)
    q = d.qpos.cpu().numpy()
    origin = np.zeros((n, r, 3))
    dirs = rng.normal(size=(n, r, 3))
    for w in range(n):
        origin[w] = q[w, :3] + rng.normal(size=(r, 3)) * [0.6, 0.6, 0.4]
        origin[w, : r // 3, 2] = q[w, 2] + 0.5
        dirs[w, : r // 3] = (0, 0, -1.0)  # height-scan style vertical rays
    dirs /= np.linalg.norm(dirs, axis=-1, keepdims=True)
    rc = RayCaster(dm, max_dist=4.0)
    dist, geom = rc.cast(d, torch.as_tensor(origin, device="cuda"), torch.as_tensor(dirs, device="cuda"))
    torch.cuda.synchronize()
    dist, geom = dist.cpu().numpy(), geom.cpu().numpy()
    gp, gm = d.geom_xpos.cpu().numpy(), d.geom_xmat.cpu().numpy()
    hits = set()
    for w in range(n):
        K = dict(geom_xpos=gp[w], geom_xmat=gm[w].reshape(-1, 3, 3))
        for k in range(r):
            t, g = O.raycast(m, K, origin[w, k], dirs[w, k], 4.0)
            assert g == geom[w, k], (w, k, g, geom[w, k])
            assert abs(t - dist[w, k]) < 1e-9
            hits.add(int(m.geom_type[g]) if g >= 0 else -1)
    assert {1, 2, 3} <= hits  # heightfield, spheres and capsules were all hit


@pytest.mark.gpu
def test_depth_camera_matches_oracle_and_sees_terrain():
    import torch

    from paper_2601_22074_b200.sim3d.sensors import DepthCamera

    m, dm, d = _setup(n=2)
    head = [g for g in range(m.ngeom) if m.geom_type[g] == 2 and abs(m.geom_pos[g][2] - 0.45) < 1e-9][0]
    cam = DepthCamera(dm, head, width=16, height=12, fovy=1.2, max_dist=6.0, offset=(0.08, 0, 0))
    dist, geom = cam.render(d)
    torch.cuda.synchronize()
    dist, geom = dist.cpu().numpy(), geom.cpu().numpy()
    gp, gm = d.geom_xpos.cpu().numpy(), d.geom_xmat.cpu().numpy()
    for w in range(d.nworld):
        K = dict(geom_xpos=gp[w], geom_xmat=gm[w].reshape(-1, 3, 3))
        o, dirs = O.camera_rays(K, head, 16, 12, 1.2, np.array([0.08, 0, 0]))
        for i in range(12):
            for j in range(16):
                t, g = O.raycast(m, K, o, dirs[i, j], 6.0, exclude_body=m.geom_bodyid[head])
                assert g == geom[w, i, j] and abs(t - dist[w, i, j]) < 1e-9
        assert (geom[w] == 0).sum() > 0  # the lower rows see the terrain
