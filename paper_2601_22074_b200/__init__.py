"""B200-native batched ManagerBasedRlEnv.step (drop-in for the stridesim hot path).

The product path is the sm_100a extension ``_stridesim_b200.so`` (built by
``__graft_entry__.build()``); there is no CPU fallback.
"""

__version__ = "0.1.0"
