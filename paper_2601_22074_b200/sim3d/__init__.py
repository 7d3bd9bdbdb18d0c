"""3-D articulated-body path: MjModel/MjData-shaped model and state,
warp-per-env sm_100a kernels (FK, com/cinert, CRB + tree-sparse L^T D L, RNE,
primitive collision, contact Jacobians, Newton solver, implicitfast), sensors and a
fused 3-D velocity task. No reference implementation exists (the reference is planar,
SPEC.md:8), so parity is against this repo's own numpy oracle (oracle/sim3d.py):
parity unpinned with respect to mjlab."""

from .model import Model, ModelBuilder, ModelError, Opt  # noqa: F401
