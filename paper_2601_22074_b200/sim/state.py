"""Device-resident batch state, structure-of-arrays.

Every per-world array of the reference BatchState (sim/state.py:20-38) is a
CUDA float64 tensor stored component-major, shape (C, N), so the fused step
reads and writes whole 256 B sectors per warp. Users see the reference's
(N, C) shapes through transposed views (``state.q`` is ``_q.t()``), so code
like ``env.state.q[w, 2] = 1.5`` writes straight into the storage the next
kernel launch reads.
"""

from __future__ import annotations

import numpy as np


def _soa(shape_c, n, device, dtype=None):
    import torch

    return torch.zeros(tuple(shape_c) + (n,), dtype=dtype or torch.float64, device=device)


def _rows(t):
    """(C..., N) storage -> (N, C...) view."""
    nd = t.dim()
    if nd == 1:
        return t
    return t.permute(nd - 1, *range(nd - 1))


class ContactCache:
    """Per-foot contact quantities applied during the last substep (sim/state.py:10-17)."""

    def __init__(self, n_worlds: int, n_feet: int, device):
        import torch

        self._normal = _soa((n_feet,), n_worlds, device)
        self._tangent = _soa((n_feet,), n_worlds, device)
        self._foot_pos = _soa((n_feet, 2), n_worlds, device)
        self._foot_vel = _soa((n_feet, 2), n_worlds, device)
        self._in_contact = _soa((n_feet,), n_worlds, device, torch.bool)

    normal_force = property(lambda self: _rows(self._normal))
    tangent_force = property(lambda self: _rows(self._tangent))
    foot_pos = property(lambda self: _rows(self._foot_pos))
    foot_vel = property(lambda self: _rows(self._foot_vel))
    in_contact = property(lambda self: _rows(self._in_contact))

    def native_into(self, st) -> None:
        st.c_normal = self._normal.data_ptr()
        st.c_tangent = self._tangent.data_ptr()
        st.c_foot_pos = self._foot_pos.data_ptr()
        st.c_foot_vel = self._foot_vel.data_ptr()
        st.c_in_contact = self._in_contact.data_ptr()


class BatchState:
    """q, qd, ctrl and bookkeeping for N worlds on one GPU.

    q columns: [base x, base z, base pitch, joint angles...]; ``ext_force`` is
    an (N, 2) world-frame push consumed by exactly one substep; ``sim_step``
    is a host integer shared by all worlds (it never needs a device read).
    """

    def __init__(self, model):
        n, nq, k = model.n_worlds, model.nq, model.num_joints
        dev = model.device
        self.n_worlds = n
        self.nq = nq
        self.device = dev
        self._q = _soa((nq,), n, dev)
        self._qd = _soa((nq,), n, dev)
        self._ctrl = _soa((k,), n, dev)
        self._ext = _soa((2,), n, dev)
        self.time = _soa((), n, dev)
        self.sim_step = 0
        self.contact = ContactCache(n, len(model.feet), dev)

    def _assign(self, name: str, value) -> None:
        import torch

        getattr(self, name)[...] = torch.as_tensor(np.asarray(value) if not torch.is_tensor(value) else value,
                                                   dtype=torch.float64, device=self.device)

    q = property(lambda self: self._q.t(), lambda self, v: self._assign("q", v))
    qd = property(lambda self: self._qd.t(), lambda self, v: self._assign("qd", v))
    ctrl = property(lambda self: self._ctrl.t(), lambda self, v: self._assign("ctrl", v))
    ext_force = property(lambda self: self._ext.t(), lambda self, v: self._assign("ext_force", v))

    def native_into(self, st) -> None:
        st.q = self._q.data_ptr()
        st.qd = self._qd.data_ptr()
        st.ctrl = self._ctrl.data_ptr()
        st.ext_force = self._ext.data_ptr()
        st.time = self.time.data_ptr()
        self.contact.native_into(st)


class StateFrame:
    """Deep host copy of the replayable part of a BatchState (sim/state.py:41-50)."""

    __slots__ = ("q", "qd", "ctrl", "sim_step")

    def __init__(self, q, qd, ctrl, sim_step: int):
        self.q = q
        self.qd = qd
        self.ctrl = ctrl
        self.sim_step = sim_step


def snapshot(state: BatchState) -> StateFrame:
    return StateFrame(
        state.q.cpu().numpy().copy(), state.qd.cpu().numpy().copy(), state.ctrl.cpu().numpy().copy(), state.sim_step
    )


def restore(state: BatchState, frame: StateFrame) -> None:
    fq, fc = np.asarray(frame.q), np.asarray(frame.ctrl)
    if tuple(fq.shape) != tuple(state.q.shape) or tuple(fc.shape) != tuple(state.ctrl.shape):
        raise ValueError(
            f"frame shape {tuple(fq.shape)}/{tuple(fc.shape)} does not match "
            f"state {tuple(state.q.shape)}/{tuple(state.ctrl.shape)}"
        )
    state.q = frame.q
    state.qd = frame.qd
    state.ctrl = frame.ctrl
    state.sim_step = int(frame.sim_step)


def detect_nonfinite(state: BatchState):
    """Per-world flag: any NaN/Inf in q, qd or ctrl (sim/state.py:69-74)."""
    import torch

    bad = ~torch.isfinite(state._q).all(dim=0)
    bad |= ~torch.isfinite(state._qd).all(dim=0)
    if state._ctrl.shape[0]:
        bad |= ~torch.isfinite(state._ctrl).all(dim=0)
    return bad
