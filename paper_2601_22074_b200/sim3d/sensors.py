"""Ray-cast sensors of the 3-D path: height scanner and depth camera (one thread per ray).

Both read the geom frames the step kernels write at the end of a launch
(``Data.enable_geom_frames()``), i.e. the state the observations see. A ray
returns the nearest hit over every geom of its own world (plane, heightfield,
sphere, capsule, box), -1 on a miss. The reference's counterpart is the
vertical-probe ``RayScanner`` (sensors.py:26-46); mjlab adds a depth camera
(out of the reference's scope), restated here as a range image.
"""

from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import native as N
from .device import Data, DeviceModel


def _stream(dm):
    return torch.cuda.current_stream(dm.device).cuda_stream


class RayCaster:
    """Arbitrary rays per world: origins/dirs (N, R, 3) in world coordinates."""

    def __init__(self, dm: DeviceModel, max_dist: float = 5.0, exclude_body: int = -1):
        self.dm, self.max_dist, self.exclude_body = dm, float(max_dist), int(exclude_body)

    def cast(self, data: Data, origin: torch.Tensor, direction: torch.Tensor):
        if data.geom_xpos is None:
            raise ValueError("enable_geom_frames() on the Data before casting rays")
        n, r = origin.shape[0], origin.shape[1]
        o = origin.to(self.dm.tdtype).contiguous()
        d = direction.to(self.dm.tdtype).contiguous()
        dist = torch.empty(n, r, dtype=self.dm.tdtype, device=self.dm.device)
        geom = torch.empty(n, r, dtype=torch.int32, device=self.dm.device)
        N.call("s3_raycast", ctypes.byref(self.dm.struct), data.geom_xpos.data_ptr(), data.geom_xmat.data_ptr(), n, r,
               o.data_ptr(), d.data_ptr(), self.max_dist, self.exclude_body, dist.data_ptr(), geom.data_ptr(),
               _stream(self.dm), launch=True)
        return dist, geom


class DepthCamera:
    """Pinhole range camera fixed to a geom (forward +x, right -y, up +z of the geom frame)."""

    def __init__(self, dm: DeviceModel, cam_geom: int, width: int = 64, height: int = 48, fovy: float = 1.0,
                 max_dist: float = 5.0, offset=(0.0, 0.0, 0.0), exclude_body: int | None = None):
        self.dm = dm
        self.cam_geom, self.width, self.height = int(cam_geom), int(width), int(height)
        self.fovy, self.max_dist = float(fovy), float(max_dist)
        self.offset = (ctypes.c_double * 3)(*offset)
        self.exclude_body = int(dm.model.geom_bodyid[cam_geom] if exclude_body is None else exclude_body)

    def render(self, data: Data):
        if data.geom_xpos is None:
            raise ValueError("enable_geom_frames() on the Data before rendering")
        n = data.nworld
        dist = torch.empty(n, self.height, self.width, dtype=self.dm.tdtype, device=self.dm.device)
        geom = torch.empty(n, self.height, self.width, dtype=torch.int32, device=self.dm.device)
        N.call("s3_depth", ctypes.byref(self.dm.struct), data.geom_xpos.data_ptr(), data.geom_xmat.data_ptr(), n,
               self.cam_geom, self.offset, self.width, self.height, self.fovy, self.max_dist, self.exclude_body,
               dist.data_ptr(), geom.data_ptr(), _stream(self.dm), launch=True)
        return dist, geom


def scan_grid(size=(1.6, 1.0), resolution=0.1):
    nx = int(round(size[0] / resolution)) + 1
    ny = int(round(size[1] / resolution)) + 1
    xs = (np.arange(nx) - (nx - 1) / 2) * resolution
    ys = (np.arange(ny) - (ny - 1) / 2) * resolution
    return np.array([(x, y) for y in ys for x in xs])
