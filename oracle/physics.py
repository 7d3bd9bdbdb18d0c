"""numpy restatement of the planar batched dynamics (sim/physics.py:22-249).

State arrays are row-major (N, C) float64 exactly like the reference; the
expression order below is the reference's, so results are bit-identical to
it on the same machine (pinned by tests/golden).
"""

from __future__ import annotations

import numpy as np


class OracleModel:
    """Chain constants + field table of one ModelSpec (sim/model.py:41-144)."""

    def __init__(self, spec, n_worlds: int):
        k = len(spec.joints)
        self.spec = spec
        self.n = n_worlds
        self.k = k
        self.nq = 3 + k
        self.parents = [int(j.parent) for j in spec.joints]
        self.offsets = np.array([j.attach_offset for j in spec.joints], dtype=np.float64).reshape(k, 2)
        self.lengths = np.array([j.link_length for j in spec.joints], dtype=np.float64)
        self.limits = np.array([j.pos_limits for j in spec.joints], dtype=np.float64).reshape(k, 2)
        self.soft = np.array([j.soft_limit_fraction for j in spec.joints], dtype=np.float64)
        self.feet = [int(f) for f in spec.feet]
        self.chains = []
        for j in range(k):
            c, node = [], j
            while node != -1:
                c.append(node)
                node = self.parents[node]
            self.chains.append(c[::-1])
        self.dt = spec.physics_dt
        self.g = spec.gravity
        # field table: name -> [value, expanded, base]
        self.fields: dict[str, list] = {}
        for name, base in (
            ("base_mass", spec.base_mass),
            ("base_inertia", spec.base_inertia),
            ("link_mass", [j.link_mass for j in spec.joints]),
            ("rotor_inertia", [j.rotor_inertia for j in spec.joints]),
            ("damping", [j.damping for j in spec.joints]),
            ("friction", spec.friction),
        ):
            self.add_field(name, base)

    def add_field(self, name: str, base) -> None:
        b = np.array(base, dtype=np.float64)
        self.fields[name] = [b.copy(), False, b]

    def value(self, name: str):
        return self.fields[name][0]

    def expand(self, name: str) -> None:
        f = self.fields[name]
        if not f[1]:
            f[0] = np.broadcast_to(f[0], (self.n,) + f[2].shape).copy()
            f[1] = True


def heights_fn(samples, spacing):
    """Heightfield.heights restated (terrain.py:159-169); None -> flat ground."""
    if samples is None or not np.any(samples):
        return lambda x: np.zeros_like(x)
    samples = np.asarray(samples, dtype=np.float64)
    last = len(samples) - 1

    def h(x):
        x = np.asarray(x, dtype=np.float64)
        pos = np.where(np.isfinite(x), x, 0.0) / spacing
        pos = np.clip(pos, 0.0, float(last))
        idx = np.minimum(pos.astype(np.int64), last - 1)
        frac = pos - idx
        return samples[idx] * (1.0 - frac) + samples[idx + 1] * frac

    return h


def raw_heights(samples, spacing, x):
    """Heightfield.heights without the flat shortcut (spawn, ray scan)."""
    samples = np.asarray(samples, dtype=np.float64)
    last = len(samples) - 1
    x = np.asarray(x, dtype=np.float64)
    pos = np.clip(np.where(np.isfinite(x), x, 0.0) / spacing, 0.0, float(last))
    idx = np.minimum(pos.astype(np.int64), last - 1)
    frac = pos - idx
    return samples[idx] * (1.0 - frac) + samples[idx + 1] * frac


def fk(m: OracleModel, q):
    """Link angles, pivots, tips and link-angle sines (sim/physics.py:22-57)."""
    n, k = q.shape[0], m.k
    th = np.empty((n, k))
    for j in range(k):
        p = m.parents[j]
        th[:, j] = (q[:, 2] if p == -1 else th[:, p]) + q[:, 3 + j]
    st, ct = np.sin(th), np.cos(th)
    sp, cp = np.sin(q[:, 2]), np.cos(q[:, 2])
    piv = np.empty((n, k, 2))
    tip = np.empty((n, k, 2))
    for j in range(k):
        p = m.parents[j]
        ox, oz = m.offsets[j]
        if p == -1:
            s, c, px, pz = sp, cp, q[:, 0], q[:, 1]
        else:
            s, c, px, pz = st[:, p], ct[:, p], piv[:, p, 0], piv[:, p, 1]
        piv[:, j, 0] = px + (c * ox - s * oz)
        piv[:, j, 1] = pz + (s * ox + c * oz)
        tip[:, j, 0] = piv[:, j, 0] + m.lengths[j] * st[:, j]
        tip[:, j, 1] = piv[:, j, 1] - m.lengths[j] * ct[:, j]
    return th, piv, tip, st


def oracle_substep(m: OracleModel, heights, S: dict) -> None:
    """One physics_dt for all worlds, in place on the state dict S
    (keys q, qd, ctrl, ext, time, fn, ft, fpos, fvel, fin, sim_step)."""
    spec = m.spec
    q, qd = S["q"], S["qd"]
    with np.errstate(invalid="ignore", over="ignore"):
        _, piv, tip, st = fk(m, q)
        n, nf = q.shape[0], len(m.feet)
        f_n = np.zeros((n, nf))
        f_t = np.zeros((n, nf))
        vel = np.zeros((n, nf, 2))
        touch = np.zeros((n, nf), dtype=bool)
        fric = m.value("friction")
        # compute_contact (sim/physics.py:75-111)
        for i, foot in enumerate(m.feet):
            px, pz = tip[:, foot, 0], tip[:, foot, 1]
            vx = qd[:, 0] - qd[:, 2] * (pz - q[:, 1])
            vz = qd[:, 1] + qd[:, 2] * (px - q[:, 0])
            for j in m.chains[foot]:
                vx -= qd[:, 3 + j] * (pz - piv[:, j, 1])
                vz += qd[:, 3 + j] * (px - piv[:, j, 0])
            phi = heights(px) - pz
            on = phi > 0.0
            nrm = np.where(on, np.maximum(0.0, spec.contact_stiffness * phi - spec.contact_damping * vz), 0.0)
            bnd = fric * nrm
            tan = np.where(on, np.clip(-spec.tangential_gain * vx, -bnd, bnd), 0.0)
            f_n[:, i], f_t[:, i] = nrm, tan
            vel[:, i, 0], vel[:, i, 1] = vx, vz
            touch[:, i] = on
        # stage_forces (sim/physics.py:191-214)
        lm = m.value("link_mass")
        tau = np.zeros_like(q)
        tau[:, 3:] += S["ctrl"]
        tau[:, 3:] -= m.value("damping") * qd[:, 3:]
        m_tot = m.value("base_mass") + lm.sum(axis=-1)
        tau[:, 1] -= m_tot * m.g
        tau[:, 3:] -= lm * m.g * (0.5 * m.lengths) * st
        tau[:, 0] += S["ext"][:, 0]
        tau[:, 1] += S["ext"][:, 1]
        for i, foot in enumerate(m.feet):
            fx, fz = f_t[:, i], f_n[:, i]
            px, pz = tip[:, foot, 0], tip[:, foot, 1]
            tau[:, 0] += fx
            tau[:, 1] += fz
            tau[:, 2] += (px - q[:, 0]) * fz - (pz - q[:, 1]) * fx
            for j in m.chains[foot]:
                tau[:, 3 + j] += (px - piv[:, j, 0]) * fz - (pz - piv[:, j, 1]) * fx
        S["ext"][...] = 0.0
        # stage_integrate (sim/physics.py:216-224)
        inv = 1.0 / m_tot
        tau[:, 0] *= inv
        tau[:, 1] *= inv
        tau[:, 2] *= 1.0 / m.value("base_inertia")
        tau[:, 3:] *= 1.0 / m.value("rotor_inertia")
        qd += tau * m.dt
        q += qd * m.dt
        # stage_finalize (sim/physics.py:226-235)
        S["fn"][...] = f_n
        S["ft"][...] = f_t
        S["fvel"][...] = vel
        for i, foot in enumerate(m.feet):
            S["fpos"][:, i, :] = tip[:, foot, :]
        S["fin"][...] = touch
        S["time"] += m.dt
        S["sim_step"] += 1


def new_state(m: OracleModel) -> dict:
    n, nf = m.n, len(m.feet)
    return {
        "q": np.zeros((n, m.nq)),
        "qd": np.zeros((n, m.nq)),
        "ctrl": np.zeros((n, m.k)),
        "ext": np.zeros((n, 2)),
        "time": np.zeros(n),
        "sim_step": 0,
        "fn": np.zeros((n, nf)),
        "ft": np.zeros((n, nf)),
        "fpos": np.zeros((n, nf, 2)),
        "fvel": np.zeros((n, nf, 2)),
        "fin": np.zeros((n, nf), dtype=bool),
    }
