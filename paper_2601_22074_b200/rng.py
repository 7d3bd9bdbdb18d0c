"""Counter-based splitmix64 streams keyed by (seed, world id, purpose).

Semantics follow rng.py of the reference (rng.py:1-131): a draw for stream i
depends only on its key and on how many words stream i has consumed, so a
world is reproducible alone, in any batch, or on any rank.

Two implementations live here:

* ``HostStreams`` -- numpy, used for host-side setup only (terrain
  generation draws per patch, terrain.py:293-328).
* ``StreamPack`` -- the device streams of an env. Counters are (N,) uint64
  tensors on the GPU, one per purpose slot; keys are never stored, the
  kernels recompute ``mix((id + 1) * SALT ^ base)`` from the per-purpose
  ``base`` (64 bits per purpose instead of 8 B per world per purpose).
  Every draw is a launch of ``ss_rng_draw`` or happens inside the fused step.
"""

from __future__ import annotations

import hashlib

import numpy as np

GOLDEN = 0x9E3779B97F4A7C15
MIX_A = 0xBF58476D1CE4E5B9
MIX_B = 0x94D049BB133111EB
KEY_SALT = 0xD6E8FEB86659FD93
UNIT = float(2.0**-53)
M64 = (1 << 64) - 1


def purpose_id(label: str) -> int:
    """First 8 bytes (little endian) of sha256(label) (rng.py:30-33)."""
    return int.from_bytes(hashlib.sha256(label.encode("utf-8")).digest()[:8], "little")


def mix64(x: int) -> int:
    x &= M64
    x = ((x ^ (x >> 30)) * MIX_A) & M64
    x = ((x ^ (x >> 27)) * MIX_B) & M64
    return x ^ (x >> 31)


def purpose_base(seed: int, label: str) -> int:
    """mix(seed * GOLDEN ^ purpose_id) -- the per-purpose half of the key."""
    return mix64(((int(seed) * GOLDEN) & M64) ^ purpose_id(label))


def _mix_np(x: np.ndarray) -> np.ndarray:
    with np.errstate(over="ignore"):
        x = (x ^ (x >> np.uint64(30))) * np.uint64(MIX_A)
        x = (x ^ (x >> np.uint64(27))) * np.uint64(MIX_B)
        return x ^ (x >> np.uint64(31))


class HostStreams:
    """numpy streams for host-side setup (terrain generation)."""

    def __init__(self, seed: int, ids):
        self.seed = int(seed)
        self.ids = np.asarray(ids, dtype=np.uint64)
        self._keys: dict[str, np.ndarray] = {}
        self._ctr: dict[str, np.ndarray] = {}

    def _slot(self, purpose: str):
        if purpose not in self._keys:
            base = np.uint64(purpose_base(self.seed, purpose))
            with np.errstate(over="ignore"):
                self._keys[purpose] = _mix_np(((self.ids + np.uint64(1)) * np.uint64(KEY_SALT)) ^ base)
            self._ctr[purpose] = np.zeros(len(self.ids), dtype=np.uint64)
        return self._keys[purpose], self._ctr[purpose]

    def uniform(self, purpose: str, low, high, sel, dim: int) -> np.ndarray:
        keys, ctr = self._slot(purpose)
        sel = np.arange(len(self.ids)) if sel is None else np.asarray(sel)
        k, c = keys[sel], ctr[sel]
        with np.errstate(over="ignore"):
            words = _mix_np(k[:, None] + (c[:, None] + np.arange(dim, dtype=np.uint64)[None, :]) * np.uint64(GOLDEN))
        ctr[sel] += np.uint64(dim)
        u = (words >> np.uint64(11)).astype(np.float64) * UNIT
        lo = np.asarray(low, dtype=np.float64)
        hi = np.asarray(high, dtype=np.float64)
        if lo.ndim == 1:
            lo = lo[:, None]
        if hi.ndim == 1:
            hi = hi[:, None]
        return lo + u * (hi - lo)


class StreamPack:
    """Device-resident streams of one env: ``uniform`` / ``normal`` /
    ``integers`` return CUDA float64 tensors, exactly the draws of
    StreamPack in the reference (rng.py:86-131)."""

    def __init__(self, seed: int, world_id_offset, n: int | None = None, device=None, on_new_slot=None):
        """``StreamPack(seed, world_id_offset, n, device)``, or the reference's ``StreamPack(seed, ids)``
        (rng.py:53) with ``ids`` a contiguous run of global ids (``offset + arange(n)``, the only form the
        reference creates: env.py:114-115) on the current CUDA device."""
        import torch

        if n is None:
            ids = np.asarray(world_id_offset, dtype=np.int64).reshape(-1)
            if ids.size == 0 or not np.array_equal(ids, ids[0] + np.arange(ids.size)):
                raise ValueError("StreamPack ids must be a contiguous run offset + arange(n)")
            world_id_offset, n = int(ids[0]), int(ids.size)
        if device is None:
            device = torch.device("cuda", torch.cuda.current_device())
        self.seed = int(seed)
        self.world_id_offset = int(world_id_offset)
        self.n = int(n)
        self.device = device
        self.slots: dict[str, int] = {}
        self.bases: list[int] = []
        self.counters: list = []
        self._on_new_slot = on_new_slot
        self._torch = torch

    @property
    def ids(self) -> np.ndarray:
        return (self.world_id_offset + np.arange(self.n)).astype(np.uint64)

    def slot(self, purpose: str) -> int:
        """Slot index of a purpose; first use allocates zeroed counters."""
        s = self.slots.get(purpose)
        if s is None:
            from .native import SS_MAX_SLOTS

            s = len(self.bases)
            if s >= SS_MAX_SLOTS:
                raise RuntimeError(f"more than {SS_MAX_SLOTS} random-stream purposes")
            self.slots[purpose] = s
            self.bases.append(purpose_base(self.seed, purpose))
            self.counters.append(self._torch.zeros(self.n, dtype=self._torch.uint64, device=self.device))
            if self._on_new_slot is not None:
                self._on_new_slot(s)
        return s

    def counter(self, purpose: str):
        return self.counters[self.slot(purpose)]

    def keys(self, purpose: str) -> np.ndarray:
        base = np.uint64(purpose_base(self.seed, purpose))
        with np.errstate(over="ignore"):
            return _mix_np(((self.ids + np.uint64(1)) * np.uint64(KEY_SALT)) ^ base)

    def _draw(self, kind: int, purpose: str, lo, hi, sel, dim: int):
        from . import native

        torch = self._torch
        s = self.slot(purpose)
        sel_t = None
        if sel is not None:
            sel_t = torch.as_tensor(np.asarray(sel) if not torch.is_tensor(sel) else sel, device=self.device)
            sel_t = sel_t.to(torch.int64).reshape(-1).contiguous()
        n_sel = self.n if sel_t is None else int(sel_t.numel())
        out = torch.empty((n_sel, dim), dtype=torch.float64, device=self.device)
        if n_sel == 0 or dim == 0:
            return out
        args = native.RngDrawArgs()
        args.kind = kind
        args.dim = dim
        args.n_sel = n_sel
        args.base = self.bases[s]
        args.world_id_offset = self.world_id_offset
        args.counter = self.counters[s].data_ptr()
        args.sel = sel_t.data_ptr() if sel_t is not None else None
        keep = []
        if kind == 0 and not torch.is_tensor(lo) and not torch.is_tensor(hi) and np.ndim(lo) == 0 and np.ndim(hi) == 0:
            # scalar bounds: no device tensors, no synchronization
            args.lohi_mode = 0
            args.lo = float(lo)
            args.hi = float(hi)
        elif kind == 0:
            lo_t = torch.as_tensor(lo, dtype=torch.float64, device=self.device)
            hi_t = torch.as_tensor(hi, dtype=torch.float64, device=self.device)
            lo_t, hi_t = torch.broadcast_tensors(lo_t, hi_t)
            if lo_t.dim() == 0:
                args.lohi_mode = 1
                lo_t = lo_t.expand(n_sel).contiguous()
                hi_t = hi_t.expand(n_sel).contiguous()
                args.lo_arr, args.hi_arr = lo_t.data_ptr(), hi_t.data_ptr()
                keep = [lo_t, hi_t]
            elif lo_t.dim() == 1:
                args.lohi_mode = 1
                lo_t, hi_t = lo_t.contiguous(), hi_t.contiguous()
                args.lo_arr, args.hi_arr = lo_t.data_ptr(), hi_t.data_ptr()
                keep = [lo_t, hi_t]
            else:
                args.lohi_mode = 2
                lo_t = lo_t.expand(n_sel, dim).contiguous()
                hi_t = hi_t.expand(n_sel, dim).contiguous()
                args.lo_arr, args.hi_arr = lo_t.data_ptr(), hi_t.data_ptr()
                keep = [lo_t, hi_t]
        else:
            args.lo = float(lo)
        args.out = out.data_ptr()
        native.call("ss_rng_draw", native.byref(args), native.current_stream(self.device))
        del keep
        return out

    def uniform(self, purpose: str, low=0.0, high=1.0, sel=None, dim: int = 1):
        """Uniform draws in [low, high), shape (n_selected, dim) (rng.py:86-111)."""
        return self._draw(0, purpose, low, high, sel, dim)

    def normal(self, purpose: str, std: float = 1.0, sel=None, dim: int = 1):
        """Box-Muller draws, shape (n_selected, dim) (rng.py:113-119)."""
        return self._draw(1, purpose, std, None, sel, dim)

    def integers(self, purpose: str, low: int, high: int, sel=None, dim: int = 1):
        """Inclusive integer draws (rng.py:121-131)."""
        u = self.uniform(purpose, 0.0, 1.0, sel, dim)
        return low + self._torch.floor(u * (high - low + 1)).to(self._torch.int64)
