"""CPU oracle for the B200 ManagerBasedRlEnv.step -- TEST INFRASTRUCTURE ONLY.

A numpy float64 restatement of the reference (`stridesim`, /root/reference)
hot path: counter RNG (rng.py), planar physics (sim/physics.py), actuators
(actuators.py), entity refresh and sensors (entity.py, sensors.py), the
seven managers and the built-in term library (managers/*.py, mdp.py), and
the eight-stage step (env.py). Each function cites the reference lines it
restates.

Pinning: tests/golden/*.npz were produced by importing the UNMODIFIED
reference in the build container (tests/golden/make_golden.py, committed);
tests/test_oracle_golden.py checks this oracle against them bit for bit.

Only tests/, __graft_entry__.smoke() and bench.py (the cpu_baseline leg and
`--impl reference`) may import this package, and only as the checker / the
CPU baseline; the product package never does.
"""

from .env import OracleEnv  # noqa: F401
from .physics import OracleModel, oracle_substep  # noqa: F401
from .rng import OracleStreams  # noqa: F401
