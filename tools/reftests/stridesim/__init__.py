"""`stridesim` -> the B200 drop-in, so the reference's OWN test-suite runs unmodified against it.

tools/reftests/run.sh copies /root/reference/pkg/tests (build container only) to baseline/_ref_tests
(git-ignored; it travels to the GPU box with the snapshot) and runs it with this directory first on
PYTHONPATH: every `stridesim.<module>` import resolves to `paper_2601_22074_b200.<module>`.

The reference returns numpy arrays, the drop-in CUDA tensors. Only the numpy
*consumption* of results is bridged here -- ``np.asarray``/``np.array_equal``/... on a CUDA tensor copy it
to the host, ``.copy()`` / ``.astype()`` and numpy-style reduction keywords behave as on an ndarray, numpy
operands and values assigned into device state are moved to the device, indexing one element returns a copy
(a numpy scalar is not a view) -- and envs are built with ``copy_outputs=True`` (fresh tensors per step, the
reference's return semantics). Nothing on the package side is altered. Tests that depend on numpy-only semantics beyond that (dtype identity, in-place numpy views,
host-side allocation tracking) are reported as they fail, not skipped.
"""

import importlib
import sys

import numpy as np
import torch

_SUBMODULES = [
    "actuators", "capture", "config", "entity", "env", "mdp", "metrics", "policies", "rng", "sensors",
    "terrain", "tasks", "managers", "managers.action", "managers.base", "managers.command",
    "managers.curriculum", "managers.event", "managers.observation", "managers.reward",
    "managers.termination", "sim", "sim.model", "sim.physics", "sim.spec", "sim.state",
]
_pkg = importlib.import_module("paper_2601_22074_b200")
for _name in _SUBMODULES:
    sys.modules[f"stridesim.{_name}"] = importlib.import_module(f"paper_2601_22074_b200.{_name}")
sys.modules["stridesim.tasks.velocity"] = sys.modules["stridesim.tasks"]  # the task module is one file here
globals().update({k: v for k, v in vars(_pkg).items() if not k.startswith("__")})
__path__ = []  # a package: `import stridesim.x` consults sys.modules first

_orig_array = torch.Tensor.__array__


def _tensor_array(self, dtype=None, copy=None):
    t = self.detach()
    if t.device.type != "cpu":
        t = t.cpu()
    a = t.numpy()
    return a if dtype is None else a.astype(dtype, copy=False)


def _to_dev(x, like):
    """numpy values (arrays, scalars, tuples of numbers) -> a tensor on `like`'s device."""
    if isinstance(x, (np.ndarray, np.generic)) or (isinstance(x, (tuple, list)) and x and
                                                      all(isinstance(v, (int, float, np.generic)) for v in x)):
        return torch.as_tensor(np.asarray(x), device=like.device)
    return x


_orig_setitem = torch.Tensor.__setitem__
_orig_getitem = torch.Tensor.__getitem__


def _tensor_setitem(self, idx, value):
    # numpy values written into device state (tests do `env.state.q[:] = array`)
    value = _to_dev(value, self)
    if isinstance(idx, np.ndarray):
        idx = torch.as_tensor(idx, device=self.device)
    return _orig_setitem(self, idx, value)


def _tensor_getitem(self, idx):
    # an element of a numpy array is a copy (a scalar), a torch 0-d result is a view of the state
    if isinstance(idx, np.ndarray):
        idx = torch.as_tensor(idx, device=self.device)
    out = _orig_getitem(self, idx)
    return out.clone() if out.dim() == 0 and self.is_cuda else out


def _np_reduction(name):
    orig = getattr(torch.Tensor, name)

    def red(self, *args, axis=None, out=None, keepdims=False, **kw):
        # np.all / np.any / np.sum / ... call the method with numpy keywords
        if axis is None and not args and not kw:
            return orig(self)
        if axis is not None:
            kw["dim"] = axis
            kw["keepdim"] = keepdims
        return orig(self, *args, **kw)

    setattr(torch.Tensor, name, red)


for _name in ("all", "any", "sum", "mean", "max", "min", "prod"):
    _np_reduction(_name)


def _binary(name):
    orig = getattr(torch.Tensor, name)

    def op(self, other):
        if isinstance(other, np.ndarray):
            other = _to_dev(other, self)
        elif torch.is_tensor(other) and other.device != self.device and other.dim() > 0:
            # numpy ufuncs wrap their host result back into a CPU tensor (np.abs(cuda_tensor))
            if other.is_cuda:
                self = self.to(other.device)
            else:
                other = other.to(self.device)
        return orig(self, other)

    setattr(torch.Tensor, name, op)


for _name in ("__add__", "__radd__", "__sub__", "__rsub__", "__mul__", "__rmul__", "__truediv__", "__rtruediv__",
              "__matmul__", "__rmatmul__", "__lt__", "__le__", "__gt__", "__ge__", "__eq__", "__ne__", "__and__",
              "__or__", "__xor__"):
    _binary(_name)

torch.Tensor.__array__ = _tensor_array
torch.Tensor.__setitem__ = _tensor_setitem
torch.Tensor.__getitem__ = _tensor_getitem
torch.Tensor.copy = lambda self: self.clone()
torch.Tensor.astype = lambda self, dtype, copy=True: np.asarray(self).astype(dtype)
torch.Tensor.__array_priority__ = -1000.0  # ndarray (op) tensor: numpy converts the tensor (__array__)

# the reference returns fresh arrays from reset/step: run the drop-in in its matching mode
_env = sys.modules["stridesim.env"]
_init = _env.ManagerBasedRlEnv.__init__


def _env_init(self, cfg, task_id="", device=None, copy_outputs=True):
    _init(self, cfg, task_id, device=device, copy_outputs=copy_outputs)


_env.ManagerBasedRlEnv.__init__ = _env_init
