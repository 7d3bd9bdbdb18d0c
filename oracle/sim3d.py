"""numpy float64 oracle of the 3-D articulated path -- TEST INFRASTRUCTURE ONLY.

PARITY UNPINNED with respect to the reference: the reference is planar
(SPEC.md:8 drops MuJoCo Warp and 3-D dynamics; sim/physics.py:1-11) and no
MuJoCo / MJWarp / mjlab is installed here, so there is no 3-D golden vector to
pin against. This module is this repo's own restatement of the published
MuJoCo pipeline stages, one function per stage, written as the specification
the CUDA kernel (paper_2601_22074_b200/csrc/s3_kernel.cuh) follows operation
for operation. It is pinned instead by analytic properties
(tests/test_sim3d_oracle_cpu.py): FK vs independent rotation composition,
1/2 qd^T M qd == kinetic energy summed over bodies, L^T D L == M, the point
Jacobian == finite differences of FK, RNE == Lagrangian finite differences
(fixed base), free fall exact, energy conservation, Newton KKT optimality
and the friction-cone bound of the contact forces.

Stages (MuJoCo names in brackets):
  kinematics [mj_kinematics] -> com [mj_comPos] (subtree com, cinert, cdof)
  -> crb [mj_crb] (M) -> factor [mj_factorM] (tree-sparse L^T D L)
  -> com_vel [mj_comVel] -> rne [mj_rne, no acc] -> passive + actuation
  -> qacc_smooth -> collision (broadphase + primitive narrowphase)
  -> constraints (limits + pyramidal contacts, soft impedance)
  -> Newton solver with exact line search [mj_solNewton]
  -> implicitfast [mj_implicitSkip] -> integrate [mj_integratePos].
"""

from __future__ import annotations

import numpy as np

from paper_2601_22074_b200.sim3d.model import (ACT_DC, ACT_IMPLICIT, GEOM_BOX, GEOM_CAPSULE, GEOM_HFIELD,
                                               GEOM_PLANE, GEOM_SPHERE, JNT_FREE, MAX_CON, MAX_LIM)

MINVAL = 1e-15


# ----------------------------------------------------------------------------- small math


def qmul(a, b):
    aw, ax, ay, az = a
    bw, bx, by, bz = b
    return np.array([aw * bw - ax * bx - ay * by - az * bz,
                     aw * bx + ax * bw + ay * bz - az * by,
                     aw * by - ax * bz + ay * bw + az * bx,
                     aw * bz + ax * by - ay * bx + az * bw])


def qmat(q):
    w, x, y, z = q
    return np.array([[1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y)],
                     [2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x)],
                     [2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)]])


def qnormalize(q):
    return q / np.sqrt(q @ q)


def qaxisangle(axis, angle):
    s, c = np.sin(0.5 * angle), np.cos(0.5 * angle)
    return np.array([c, axis[0] * s, axis[1] * s, axis[2] * s])


def cross_motion(v, u):
    """[w x u_ang ; w x u_lin + v_lin x u_ang] (mju_crossMotion)."""
    w, vl = v[:3], v[3:]
    return np.concatenate([np.cross(w, u[:3]), np.cross(w, u[3:]) + np.cross(vl, u[:3])])


def cross_force(v, f):
    """[w x f_ang + v_lin x f_lin ; w x f_lin] (mju_crossForce)."""
    w, vl = v[:3], v[3:]
    return np.concatenate([np.cross(w, f[:3]) + np.cross(vl, f[3:]), np.cross(w, f[3:])])


def inert_mul(ci, v):
    """10-vector spatial inertia (Ixx Iyy Izz Ixy Ixz Iyz mdx mdy mdz m) times a motion vector."""
    I = np.array([[ci[0], ci[3], ci[4]], [ci[3], ci[1], ci[5]], [ci[4], ci[5], ci[2]]])
    md, m = ci[6:9], ci[9]
    w, vl = v[:3], v[3:]
    return np.concatenate([I @ w + np.cross(md, vl), m * vl - np.cross(md, w)])


# ----------------------------------------------------------------------------- stages


def kinematics(m, qpos):
    """Body frames in topological order (mj_kinematics)."""
    nb = m.nbody
    xpos = np.zeros((nb, 3))
    xquat = np.zeros((nb, 4))
    xquat[0] = (1, 0, 0, 0)
    xmat = np.zeros((nb, 3, 3))
    xmat[0] = np.eye(3)
    xanchor = np.zeros((m.njnt, 3))
    xaxis = np.zeros((m.njnt, 3))
    for b in range(1, nb):
        p = m.body_parentid[b]
        pos = xpos[p] + xmat[p] @ m.body_pos[b]
        quat = qmul(xquat[p], m.body_quat[b])
        for j in range(m.body_jntadr[b], m.body_jntadr[b] + m.body_jntnum[b]):
            a = m.jnt_qposadr[j]
            if m.jnt_type[j] == JNT_FREE:
                pos = qpos[a:a + 3].copy()
                quat = qnormalize(qpos[a + 3:a + 7])
                xanchor[j] = pos
                xaxis[j] = (0, 0, 1)
            else:
                R = qmat(quat)
                xanchor[j] = R @ m.jnt_pos[j] + pos
                xaxis[j] = R @ m.jnt_axis[j]
                quat = qmul(quat, qaxisangle(m.jnt_axis[j], qpos[a] - m.qpos0[a]))
                pos = xanchor[j] - qmat(quat) @ m.jnt_pos[j]
        quat = qnormalize(quat)
        xquat[b] = quat
        xmat[b] = qmat(quat)
        xpos[b] = pos
    xipos = xpos + np.einsum("bij,bj->bi", xmat, m.body_ipos)
    ximat = np.array([xmat[b] @ qmat(m.body_iquat[b]) for b in range(nb)])
    gxpos = xpos[m.geom_bodyid] + np.einsum("gij,gj->gi", xmat[m.geom_bodyid], m.geom_pos)
    gxmat = np.array([xmat[m.geom_bodyid[g]] @ qmat(m.geom_quat[g]) for g in range(m.ngeom)])
    return dict(xpos=xpos, xquat=xquat, xmat=xmat, xipos=xipos, ximat=ximat, xanchor=xanchor, xaxis=xaxis,
                geom_xpos=gxpos, geom_xmat=gxmat)


def body_mass_scaled(m, mscale):
    """Per-world base-mass randomisation: body 1 (the robot base) scaled in mass and inertia."""
    mass = m.body_mass.copy()
    inertia = m.body_inertia.copy()
    if mscale != 1.0:
        mass[1] = mass[1] * mscale
        inertia[1] = inertia[1] * mscale
    return mass, inertia


def com_pos(m, K, mscale=1.0):
    """Subtree com of every kinematic tree, cinert about its tree's com, cdof (mj_comPos).
    ``mscale``: the world's base-mass scale (domain randomisation)."""
    mass, inertia = body_mass_scaled(m, mscale)
    coms = np.zeros((m.ntree, 3))
    for t in range(m.ntree):
        sel = [b for b in range(1, m.nbody) if m.body_treeid[b] == t]
        tmass = m.tree_mass[t] + (mass[1] - m.body_mass[1] if m.body_treeid[1] == t else 0.0)
        coms[t] = (mass[sel][:, None] * K["xipos"][sel]).sum(0) / tmass
    cinert = np.zeros((m.nbody, 10))
    for b in range(1, m.nbody):
        com = coms[m.body_treeid[b]]
        R = K["ximat"][b]
        I = R @ np.diag(inertia[b]) @ R.T
        d = K["xipos"][b] - com
        mb = mass[b]
        I = I + mb * ((d @ d) * np.eye(3) - np.outer(d, d))
        cinert[b] = (I[0, 0], I[1, 1], I[2, 2], I[0, 1], I[0, 2], I[1, 2], mb * d[0], mb * d[1], mb * d[2], mb)
    cdof = np.zeros((m.nv, 6))
    for j in range(m.njnt):
        b, da = m.jnt_bodyid[j], m.jnt_dofadr[j]
        com = coms[m.body_treeid[b]]
        if m.jnt_type[j] == JNT_FREE:
            for i in range(3):
                cdof[da + i, 3 + i] = 1.0
            off = com - K["xanchor"][j]
            for i in range(3):
                ax = K["xmat"][b][:, i]
                cdof[da + 3 + i] = np.concatenate([ax, np.cross(ax, off)])
        else:
            ax = K["xaxis"][j]
            cdof[da] = np.concatenate([ax, np.cross(ax, com - K["xanchor"][j])])
    return dict(com=coms, cinert=cinert, cdof=cdof)


def crb(m, C):
    """Composite inertia + dense symmetric M over ancestor pairs (mj_crb); armature on the diagonal."""
    c = C["cinert"].copy()
    for b in range(m.nbody - 1, 0, -1):
        p = m.body_parentid[b]
        if p > 0:
            c[p] += c[b]
    M = np.zeros((m.nv, m.nv))
    for i in range(m.nv):
        f = inert_mul(c[m.dof_bodyid[i]], C["cdof"][i])
        j = i
        while j >= 0:
            M[i, j] = M[j, i] = C["cdof"][j] @ f
            j = m.dof_parentid[j]
        M[i, i] += m.dof_armature[i]
    return M, c


def factor_ldl(m, M):
    """Tree-sparse L^T D L (mj_factorM): returns qLD with D on the diagonal and L below it
    (only ancestor entries are touched; no fill-in for a kinematic tree)."""
    L = M.copy()
    par = m.dof_parentid
    for k in range(m.nv - 1, -1, -1):
        i = par[k]
        while i >= 0:
            t = L[k, i] / L[k, k]
            j = i
            while j >= 0:
                L[i, j] -= t * L[k, j]
                j = par[j]
            L[k, i] = t
            i = par[i]
    return L


def solve_ldl(m, L, b):
    x = b.copy()
    par = m.dof_parentid
    for i in range(m.nv - 1, -1, -1):
        j = par[i]
        while j >= 0:
            x[j] -= L[i, j] * x[i]
            j = par[j]
    x = x / np.diag(L)
    for i in range(m.nv):
        j = par[i]
        while j >= 0:
            x[i] -= L[i, j] * x[j]
            j = par[j]
    return x


def com_vel(m, C, qvel):
    """cvel per body and cdof_dot per dof (mj_comVel)."""
    cvel = np.zeros((m.nbody, 6))
    cdofd = np.zeros((m.nv, 6))
    for b in range(1, m.nbody):
        v = cvel[m.body_parentid[b]].copy()
        for j in range(m.body_jntadr[b], m.body_jntadr[b] + m.body_jntnum[b]):
            da = m.jnt_dofadr[j]
            if m.jnt_type[j] == JNT_FREE:
                for i in range(3):
                    v = v + C["cdof"][da + i] * qvel[da + i]
                for i in range(3, 6):
                    cdofd[da + i] = cross_motion(v, C["cdof"][da + i])
                for i in range(3, 6):
                    v = v + C["cdof"][da + i] * qvel[da + i]
            else:
                cdofd[da] = cross_motion(v, C["cdof"][da])
                v = v + C["cdof"][da] * qvel[da]
        cvel[b] = v
    return cvel, cdofd


def rne(m, C, cvel, cdofd, qvel):
    """Bias forces C(q,qd) qd + g(q) (mj_rne with qacc = 0); gravity as a base acceleration."""
    g = np.asarray(m.opt.gravity, dtype=np.float64)
    cacc = np.zeros((m.nbody, 6))
    cacc[0, 3:] = -g
    cfrc = np.zeros((m.nbody, 6))
    for b in range(1, m.nbody):
        a = cacc[m.body_parentid[b]].copy()
        da, nd = m.body_dofadr[b], m.body_dofnum[b]
        for d in range(da, da + nd) if nd else ():
            a = a + cdofd[d] * qvel[d]
        cacc[b] = a
        ci = C["cinert"][b]
        cfrc[b] = inert_mul(ci, a) + cross_force(cvel[b], inert_mul(ci, cvel[b]))
    for b in range(m.nbody - 1, 0, -1):
        p = m.body_parentid[b]
        if p > 0:
            cfrc[p] += cfrc[b]
    bias = np.array([C["cdof"][i] @ cfrc[m.dof_bodyid[i]] for i in range(m.nv)])
    return bias


def actuation(m, qpos, qvel, ctrl):
    """Joint-space actuator forces and the implicit velocity derivative per dof.
    ctrl is the position target per actuator. PD / DC follow actuators.py:104-117 of the
    reference (explicit kd); IMPLICIT is a position actuator kp (ctrl - q) - kv qd whose kv
    enters implicitfast (skipped when the force range clamps it)."""
    f = np.zeros(m.nv)
    kvd = np.zeros(m.nv)
    for u in range(m.nu):
        d, a = m.actuator_dofadr[u], m.actuator_qposadr[u]
        kp, kv, eff = m.actuator_kp[u], m.actuator_kv[u], m.actuator_effort[u]
        q, qd = qpos[a], qvel[d]
        tau = kp * (ctrl[u] - q) + kv * (0.0 - qd)
        if m.actuator_kind[u] == ACT_DC:
            sat, vmax = m.actuator_saturation[u], m.actuator_vmax[u]
            hi = min(max(sat * (1.0 - qd / vmax), 0.0), eff)
            lo = min(max(sat * (-1.0 - qd / vmax), -eff), 0.0)
            tau = min(max(tau, lo), hi)
        else:
            clamped = tau > eff or tau < -eff
            tau = min(max(tau, -eff), eff)
            if m.actuator_kind[u] == ACT_IMPLICIT and not clamped:
                kvd[d] += kv
        f[d] += tau
    return f, kvd


# ----------------------------------------------------------------------------- collision


def make_frame(n):
    e = np.array([0.0, 1.0, 0.0]) if abs(n[1]) < 0.5 else np.array([1.0, 0.0, 0.0])
    t1 = np.cross(n, e)
    t1 = t1 / np.sqrt(t1 @ t1)
    t2 = np.cross(n, t1)
    return np.array([n, t1, t2])


def hfield_point(m, q, r):
    """Signed distance of a sphere (centre q, radius r) to the heightfield triangle under q.
    Grid rows run along y, columns along x; each cell is split along the (0,0)-(1,1) diagonal."""
    H = m.hfield_data
    nr, nc = H.shape
    sp = m.hfield_spacing
    fx = (q[0] - m.hfield_origin[0]) / sp
    fy = (q[1] - m.hfield_origin[1]) / sp
    if not (fx >= 0.0 and fy >= 0.0 and fx < nc - 1 and fy < nr - 1):
        return None
    ix, iy = int(np.floor(fx)), int(np.floor(fy))
    u, v = fx - ix, fy - iy
    x0 = m.hfield_origin[0] + ix * sp
    y0 = m.hfield_origin[1] + iy * sp
    h00, h10, h01, h11 = H[iy, ix], H[iy, ix + 1], H[iy + 1, ix], H[iy + 1, ix + 1]
    if u >= v:  # triangle (0,0) (1,0) (1,1)
        n = np.array([-(h10 - h00) * sp, -(h11 - h10) * sp, sp * sp])
        v0 = np.array([x0, y0, h00])
    else:       # triangle (0,0) (1,1) (0,1)
        n = np.array([-(h11 - h01) * sp, -(h01 - h00) * sp, sp * sp])
        v0 = np.array([x0, y0, h00])
    n = n / np.sqrt(n @ n)
    d = n @ (q - v0) - r
    return d, n


def seg_closest(p1, q1, p2, q2):
    d1, d2, r = q1 - p1, q2 - p2, p1 - p2
    a, e, f = d1 @ d1, d2 @ d2, d2 @ r
    c, b = d1 @ r, d1 @ d2
    if e <= 1e-12:  # second segment degenerate (a sphere centre)
        s = min(max(-c / a, 0.0), 1.0) if a > 1e-12 else 0.0
        return p1 + d1 * s, p2
    if a <= 1e-12:
        t = min(max(f / e, 0.0), 1.0)
        return p1, p2 + d2 * t
    den = a * e - b * b
    s = min(max((b * f - c * e) / den, 0.0), 1.0) if den > 1e-12 else 0.0
    t = (b * s + f) / e
    if t < 0.0:
        t = 0.0
        s = min(max(-c / a, 0.0), 1.0)
    elif t > 1.0:
        t = 1.0
        s = min(max((b - c) / a, 0.0), 1.0)
    return p1 + d1 * s, p2 + d2 * t


def _sphere_sphere(c1, r1, c2, r2):
    dv = c2 - c1
    L = np.sqrt(dv @ dv)
    n = dv / L if L > 1e-12 else np.array([0.0, 0.0, 1.0])
    d = L - r1 - r2
    return d, n, c1 + n * (r1 + 0.5 * d)


def sphere_box(c, r, bc, R, size):
    """Sphere (centre c, radius r) vs box (centre bc, rotation R, half sizes): (dist, normal sphere->box,
    contact point). Centre outside: closest point on the box; inside: the face of least penetration."""
    p = R.T @ (c - bc)
    q = np.minimum(np.maximum(p, -size), size)
    dq = p - q
    L = np.sqrt(dq @ dq)
    if L > 1e-12:
        n_loc = -dq / L          # from the sphere centre towards the box
        d = L - r
        pos = bc + R @ q - (R @ n_loc) * (0.5 * d)  # midpoint of the two surface points
        return d, R @ n_loc, pos
    # inside: push out through the nearest face
    gap = size - np.abs(p)
    k = int(np.argmin(gap))
    n_loc = np.zeros(3)
    n_loc[k] = -1.0 if p[k] >= 0.0 else 1.0  # towards the box interior from that face
    d = -gap[k] - r
    face = p.copy()
    face[k] = size[k] if p[k] >= 0.0 else -size[k]
    pos = bc + R @ face - (R @ n_loc) * (0.5 * d)
    return d, R @ n_loc, pos


CAPSULE_BOX_ITERS = 8


def capsule_box(p0, p1, r, bc, R, size):
    """Capsule (segment p0-p1, radius r) vs box: the segment point closest to the box by alternating
    projections (box clamp <-> segment projection, CAPSULE_BOX_ITERS rounds from the midpoint), then the
    sphere-box contact at that point."""
    a = R.T @ (p0 - bc)
    b = R.T @ (p1 - bc)
    d = b - a
    dd = d @ d
    t = 0.5
    for _ in range(CAPSULE_BOX_ITERS):
        p = a + d * t
        q = np.minimum(np.maximum(p, -size), size)
        t = min(max(((q - a) @ d) / dd, 0.0), 1.0) if dd > 1e-12 else 0.0
    c = bc + R @ (a + d * t)
    return sphere_box(c, r, bc, R, size)


BOX_FACE_BIAS = 0.95  # an edge axis wins only below this fraction of the best face overlap (face contacts first)
BOX_TIE = 1e-12  # a candidate axis / face / point replaces the current one only when better by this margin, so
# symmetric configurations (equal overlaps, rectangle corners) pick the same one in every rounding


def box_box(c1, R1, h1, c2, R2, h2):
    """Box-box narrowphase: the separating-axis test over the 3 + 3 face normals and the 9 edge-edge cross
    products (parallel pairs skipped), then for a face axis the incident face of the other box clipped
    (Sutherland-Hodgman) against the reference face's four side planes -- the clipped points below the
    reference face are the contacts, at most 4 (the deepest, then repeatedly the point farthest from those
    chosen) -- and for an edge axis one contact at the closest points of the two support edges. Normal from
    box 1 to box 2; each contact (dist = -depth, normal, midpoint)."""
    dv = c2 - c1
    A = [R1[:, i] for i in range(3)]
    B = [R2[:, j] for j in range(3)]

    def overlap(u):
        r1 = h1[0] * abs(u @ A[0]) + h1[1] * abs(u @ A[1]) + h1[2] * abs(u @ A[2])
        r2 = h2[0] * abs(u @ B[0]) + h2[1] * abs(u @ B[1]) + h2[2] * abs(u @ B[2])
        sd = u @ dv
        return r1 + r2 - abs(sd), sd

    face = None
    for k in range(6):
        u = A[k] if k < 3 else B[k - 3]
        ov, sd = overlap(u)
        if ov < 0.0:
            return []
        if face is None or ov < face[0] - BOX_TIE:
            face = (ov, k, u, sd)
    edge = None
    for i in range(3):
        for j in range(3):
            u = np.cross(A[i], B[j])
            L = np.sqrt(u @ u)
            if L < 1e-6:
                continue
            u = u / L
            ov, sd = overlap(u)
            if ov < 0.0:
                return []
            if edge is None or ov < edge[0] - BOX_TIE:
                edge = (ov, 6 + 3 * i + j, u, sd)
    best = edge if (edge is not None and edge[0] < BOX_FACE_BIAS * face[0]) else face
    ov, k, u, sd = best
    n = u if sd >= 0.0 else -u
    if k >= 6:
        i, j = (k - 6) // 3, (k - 6) % 3
        e1 = c1.copy()
        for q in range(3):
            if q != i:
                e1 = e1 + (1.0 if A[q] @ n >= 0.0 else -1.0) * h1[q] * A[q]
        e2 = c2.copy()
        for q in range(3):
            if q != j:
                e2 = e2 + (1.0 if B[q] @ n <= 0.0 else -1.0) * h2[q] * B[q]
        P, Q = seg_closest(e1 - A[i] * h1[i], e1 + A[i] * h1[i], e2 - B[j] * h2[j], e2 + B[j] * h2[j])
        return [(-ov, n, 0.5 * (P + Q))]
    if k < 3:
        cr, Ar, hr, ia, ci, Ai, hi, nref = c1, A, h1, k, c2, B, h2, n
    else:
        cr, Ar, hr, ia, ci, Ai, hi, nref = c2, B, h2, k - 3, c1, A, h1, -n
    cf = cr + nref * hr[ia]
    proj = [abs(Ai[q] @ nref) for q in range(3)]
    jf = 0
    for q in (1, 2):
        if proj[q] > proj[jf] + BOX_TIE:
            jf = q
    ninc = -Ai[jf] if Ai[jf] @ nref >= 0.0 else Ai[jf]
    fi = ci + ninc * hi[jf]
    ua, va = [q for q in range(3) if q != jf]
    poly = [fi + su * hi[ua] * Ai[ua] + sv * hi[va] * Ai[va] for su, sv in ((-1.0, -1.0), (1.0, -1.0), (1.0, 1.0),
                                                                             (-1.0, 1.0))]
    for t in [q for q in range(3) if q != ia]:
        for sg in (1.0, -1.0):
            out = []
            for idx in range(len(poly)):
                P, Q = poly[idx], poly[(idx + 1) % len(poly)]
                dP = hr[t] - sg * ((P - cr) @ Ar[t])
                dQ = hr[t] - sg * ((Q - cr) @ Ar[t])
                if dP >= 0.0:
                    out.append(P)
                if (dP >= 0.0) != (dQ >= 0.0):
                    out.append(P + (Q - P) * (dP / (dP - dQ)))
            poly = out
            if not poly:
                return []
    pts = [(nref @ (cf - x), x) for x in poly]
    pts = [(dep, x) for dep, x in pts if dep > 0.0]
    chosen = []
    if pts:
        b = 0
        for q in range(1, len(pts)):
            if pts[q][0] > pts[b][0] + BOX_TIE:
                b = q
        chosen.append(b)
        while len(chosen) < min(4, len(pts)):
            bq, bd = -1, -1.0
            for q in range(len(pts)):
                if q in chosen:
                    continue
                dm = min(float((pts[q][1] - pts[c][1]) @ (pts[q][1] - pts[c][1])) for c in chosen)
                if dm > bd + BOX_TIE:
                    bq, bd = q, dm
            chosen.append(bq)
    return [(-pts[q][0], n, pts[q][1] + nref * (0.5 * pts[q][0])) for q in chosen]


def _segment(m, K, g):
    a = K["geom_xmat"][g][:, 2] * m.geom_size[g][1]
    c = K["geom_xpos"][g]
    return c - a, c + a


def _point_set(m, K, g):
    """Points + radii standing in for geom g against the terrain."""
    t, s = m.geom_type[g], m.geom_size[g]
    c = K["geom_xpos"][g]
    if t == GEOM_SPHERE:
        return [(c, s[0])]
    if t == GEOM_CAPSULE:
        p, q = _segment(m, K, g)
        return [(p, s[0]), (q, s[0])]
    R = K["geom_xmat"][g]
    out = []
    for i in range(8):
        loc = np.array([s[0] if i & 1 else -s[0], s[1] if i & 2 else -s[1], s[2] if i & 4 else -s[2]])
        out.append((c + R @ loc, 0.0))
    return out


def collide(m, K, fscale=1.0):
    """Broadphase (bounding spheres) + narrowphase over the compiled candidate pairs, in pair order;
    at most m.ncon_max contacts (later ones dropped and counted). ``fscale``: the world's friction
    scale (domain randomisation), multiplying every pair's friction."""
    cons, dropped = [], 0
    hmax = float(m.hfield_data.max())
    for p, (g1, g2) in enumerate(m.pair_geom):
        t1, t2 = m.geom_type[g1], m.geom_type[g2]
        c1, c2 = K["geom_xpos"][g1], K["geom_xpos"][g2]
        mu = 0.0 if m.pair_condim[p] == 1 else max(m.geom_friction[g1], m.geom_friction[g2]) * fscale
        found = []
        if t1 == GEOM_PLANE:
            n = K["geom_xmat"][g1][:, 2]
            if n @ (c2 - c1) - m.geom_rbound[g2] >= 0.0:
                continue
            for q, r in _point_set(m, K, g2):
                d = n @ (q - c1) - r
                if d < 0.0:
                    found.append((d, n, q - n * (r + 0.5 * d)))
        elif t1 == GEOM_HFIELD:
            if c2[2] - m.geom_rbound[g2] >= hmax:
                continue
            for q, r in _point_set(m, K, g2):
                h = hfield_point(m, q, r)
                if h is not None and h[0] < 0.0:
                    d, n = h
                    found.append((d, n, q - n * (r + 0.5 * d)))
        elif t1 == GEOM_BOX:  # box-box (both boxes; pairs put a box first only against a box)
            dv = c2 - c1
            rb = m.geom_rbound[g1] + m.geom_rbound[g2]
            if dv @ dv >= rb * rb:
                continue
            found += box_box(c1, K["geom_xmat"][g1], m.geom_size[g1], c2, K["geom_xmat"][g2], m.geom_size[g2])
        elif t2 == GEOM_BOX:  # sphere or capsule (g1) vs box (g2)
            dv = c2 - c1
            rb = m.geom_rbound[g1] + m.geom_rbound[g2]
            if dv @ dv >= rb * rb:
                continue
            if t1 == GEOM_CAPSULE:
                p0, p1 = _segment(m, K, g1)
                h = capsule_box(p0, p1, m.geom_size[g1][0], c2, K["geom_xmat"][g2], m.geom_size[g2])
            else:
                h = sphere_box(c1, m.geom_size[g1][0], c2, K["geom_xmat"][g2], m.geom_size[g2])
            if h is not None and h[0] < 0.0:
                found.append(h)
        else:
            dv = c2 - c1
            rb = m.geom_rbound[g1] + m.geom_rbound[g2]
            if dv @ dv >= rb * rb:
                continue
            r1, r2 = m.geom_size[g1][0], m.geom_size[g2][0]
            if t1 == GEOM_SPHERE and t2 == GEOM_SPHERE:
                a, b = c1, c2
            elif t1 == GEOM_SPHERE:
                p2, q2 = _segment(m, K, g2)
                b, a = seg_closest(p2, q2, c1, c1)
            elif t2 == GEOM_SPHERE:
                p1, q1 = _segment(m, K, g1)
                a, b = seg_closest(p1, q1, c2, c2)
            else:
                p1, q1 = _segment(m, K, g1)
                p2, q2 = _segment(m, K, g2)
                a, b = seg_closest(p1, q1, p2, q2)
            d, n, pos = _sphere_sphere(a, r1, b, r2)
            if d < 0.0:
                found.append((d, n, pos))
        if t2 == GEOM_BOX:
            found = found[:4]
        for d, n, pos in found:
            if len(cons) >= m.ncon_max:
                dropped += 1
                continue
            cons.append(dict(dist=d, pos=pos, frame=make_frame(n), mu=mu, pair=p, geom1=g1, geom2=g2))
    return cons, dropped


# ----------------------------------------------------------------------------- constraints


def point_jac(m, C, b, p):
    """3 x nv translational Jacobian of world point p attached to body b (mj_jac)."""
    J = np.zeros((3, m.nv))
    com = C["com"][m.body_treeid[b]]
    for d in m.body_chain[b]:
        J[:, d] = C["cdof"][d][3:] + np.cross(C["cdof"][d][:3], p - com)
    return J


def impedance(r, solimp):
    dmin, dmax, width, mid, power = solimp
    x = abs(r) / width
    if x >= 1.0:
        d = dmax
    else:
        y = x ** power / mid ** (power - 1) if x <= mid else 1.0 - (1.0 - x) ** power / (1.0 - mid) ** (power - 1)
        d = dmin + y * (dmax - dmin)
    return min(max(d, 1e-4), 0.9999)


def constraints(m, C, cons, qpos, qvel):
    """Rows: active joint limits (dof order), then 4 pyramid edges per contact
    [n + mu t1, n - mu t1, n + mu t2, n - mu t2]. Each row: dense J (nv), pos, aref, D."""
    rows = []
    for j in range(m.njnt):
        if not m.jnt_limited[j]:
            continue
        a, d = m.jnt_qposadr[j], m.jnt_dofadr[j]
        lo, hi = m.jnt_range[j]
        for dist, sgn in ((qpos[a] - lo, 1.0), (hi - qpos[a], -1.0)):
            if dist < 0.0 and len(rows) < MAX_LIM:
                J = np.zeros(m.nv)
                J[d] = sgn
                rows.append(dict(J=J, pos=dist, A=m.dof_invweight0[d]))
    nlim = len(rows)
    for c in cons:
        b1, b2 = m.geom_bodyid[c["geom1"]], m.geom_bodyid[c["geom2"]]
        Jp = point_jac(m, C, b2, c["pos"]) - point_jac(m, C, b1, c["pos"])
        Jc = c["frame"] @ Jp
        mu = c["mu"]
        # condim 1 (frictionless): mu = 0 turns the 4 pyramid rows into the normal row; with 4x the normal
        # row's R each, their sum is MuJoCo's single frictionless row (identical cost, Hessian, total force)
        A = (4.0 if m.pair_condim[c["pair"]] == 1 else 1.0 + mu * mu) * (m.body_invweight0[b1] + m.body_invweight0[b2])
        for k in (1, 2):
            for s in (1.0, -1.0):
                rows.append(dict(J=Jc[0] + (s * mu) * Jc[k], pos=c["dist"], A=A))
    tc = max(m.opt.solref[0], 2.0 * m.opt.timestep)
    dr = m.opt.solref[1]
    dmax = m.opt.solimp[1]
    kk = 1.0 / (dmax * dmax * tc * tc * dr * dr)
    bb = 2.0 / (dmax * tc)
    nefc = len(rows)
    J = np.array([r["J"] for r in rows]).reshape(nefc, m.nv)
    pos = np.array([r["pos"] for r in rows])
    imp = np.array([impedance(p, m.opt.solimp) for p in pos])
    A = np.array([r["A"] for r in rows])
    R = np.maximum((1.0 - imp) / imp * A, MINVAL)
    vel = J @ qvel
    aref = -bb * vel - kk * imp * pos
    return dict(J=J, pos=pos, aref=aref, D=1.0 / R, R=R, imp=imp, nlim=nlim, nefc=nefc)


def cholesky(H):
    """Right-looking dense Cholesky H = L L^T (lower)."""
    n = H.shape[0]
    L = H.copy()
    for k in range(n):
        L[k, k] = np.sqrt(L[k, k])
        L[k + 1:, k] = L[k + 1:, k] / L[k, k]
        L[k + 1:, k + 1:] -= np.outer(L[k + 1:, k], L[k + 1:, k])
    return np.tril(L)


def chol_solve(L, b):
    n = L.shape[0]
    y = b.copy()
    for i in range(n):
        y[i] = (y[i] - L[i, :i] @ y[:i]) / L[i, i]
    x = y.copy()
    for i in range(n - 1, -1, -1):
        x[i] = (x[i] - L[i + 1:, i] @ x[i + 1:]) / L[i, i]
    return x


def _cost(E, qfrc_smooth, a, Ma, jar):
    """1/2 a^T M a - a^T f + sum_i 1/2 D_i min(J_i a - aref_i, 0)^2: the Gauss term
    1/2 (a-a0)^T M (a-a0) up to the constant 1/2 a0^T f (a0 = M^-1 f), so differences are exact
    and qacc_smooth is not needed by the solver."""
    act = jar < 0.0
    gauss = 0.5 * (a @ (Ma - 2.0 * qfrc_smooth))
    return gauss + 0.5 * np.sum(E["D"][act] * jar[act] ** 2)


def newton(m, M, E, qfrc_smooth, a0, warm):
    """Primal Newton on 1/2 (a-a0)^T M (a-a0) + sum_i 1/2 D_i min(J_i a - aref_i, 0)^2, started
    from the warm start (zeros when there is none), with an exact (bracketed 1-D Newton) line search
    (mj_solNewton restated). ``a0`` is unused by the iteration (see _cost)."""
    J, D, aref = E["J"], E["D"], E["aref"]
    scale = 1.0 / (m.meaninertia * max(1, m.nv))
    a = np.zeros(m.nv) if warm is None else warm.copy()
    Ma = M @ a
    jar = J @ a - aref
    cost = _cost(E, qfrc_smooth, a, Ma, jar)
    its = 0
    for it in range(m.opt.iterations):
        act = jar < 0.0
        grad = Ma - qfrc_smooth + J.T @ (D * act * jar)
        if scale * np.sqrt(grad @ grad) < m.opt.tolerance:
            break
        its += 1
        H = M + (J.T * (D * act)) @ J
        L = cholesky(H)
        p = -chol_solve(L, grad)
        Mp = M @ p
        Jp = J @ p
        alpha = line_search(m, p, Ma - qfrc_smooth, Mp, jar, Jp, D)
        if alpha == 0.0:
            break
        a = a + alpha * p
        Ma = Ma + alpha * Mp
        jar = jar + alpha * Jp
        new = _cost(E, qfrc_smooth, a, Ma, jar)
        imp = scale * (cost - new)
        cost = new
        if imp < m.opt.tolerance:
            break
    act = jar < 0.0
    force = -D * act * jar
    return a, force, J.T @ force, its


def cg(m, M, L, E, qfrc_smooth, warm):
    """Primal conjugate gradient on the same cost as ``newton`` (mj_solCG restated): the gradient
    preconditioned by M^-1 (``L``, the L^T D L factor of M), Polak-Ribiere directions (beta clamped at 0),
    the same exact line search and stopping rules; no Hessian is formed or factored."""
    J, D, aref = E["J"], E["D"], E["aref"]
    scale = 1.0 / (m.meaninertia * max(1, m.nv))
    a = np.zeros(m.nv) if warm is None else warm.copy()
    Ma = M @ a
    jar = J @ a - aref
    cost = _cost(E, qfrc_smooth, a, Ma, jar)
    grad = Ma - qfrc_smooth + J.T @ (D * (jar < 0.0) * jar)
    Mgrad = solve_ldl(m, L, grad)
    search = -Mgrad
    its = 0
    for it in range(m.opt.iterations):
        if scale * np.sqrt(grad @ grad) < m.opt.tolerance:
            break
        its += 1
        Mp = M @ search
        Jp = J @ search
        alpha = line_search(m, search, Ma - qfrc_smooth, Mp, jar, Jp, D)
        if alpha == 0.0:
            break
        a = a + alpha * search
        Ma = Ma + alpha * Mp
        jar = jar + alpha * Jp
        new = _cost(E, qfrc_smooth, a, Ma, jar)
        imp = scale * (cost - new)
        cost = new
        gold, Mgold = grad, Mgrad
        grad = Ma - qfrc_smooth + J.T @ (D * (jar < 0.0) * jar)
        Mgrad = solve_ldl(m, L, grad)
        if imp < m.opt.tolerance:
            break
        beta = max(0.0, float(grad @ (Mgrad - Mgold)) / max(MINVAL, float(gold @ Mgold)))
        search = -Mgrad + beta * search
    act = jar < 0.0
    force = -D * act * jar
    return a, force, J.T @ force, its


def line_search(m, p, res, Mp, jar, Jp, D):
    """Exact minimiser of the convex piecewise-quadratic cost along p: bracketed Newton on phi'."""
    g0 = p @ res
    h0 = p @ Mp

    def deriv(al):
        x = jar + al * Jp
        act = x < 0.0
        return g0 + al * h0 + np.sum(D[act] * x[act] * Jp[act]), h0 + np.sum(D[act] * Jp[act] ** 2)

    d0, _ = deriv(0.0)
    if not d0 < 0.0:
        return 0.0
    lo, hi, al = 0.0, np.inf, 1.0
    for _ in range(m.opt.ls_iterations):
        d1, d2 = deriv(al)
        if abs(d1) < m.opt.ls_tolerance * abs(d0):
            break
        if d1 < 0.0:
            lo = al
        else:
            hi = al
        an = al - d1 / d2
        if not (lo < an < hi):
            an = 0.5 * (lo + hi)
        al = an
    return al


# ----------------------------------------------------------------------------- step


def integrate_pos(m, qpos, qvel, dt):
    q = qpos.copy()
    for j in range(m.njnt):
        a, d = m.jnt_qposadr[j], m.jnt_dofadr[j]
        if m.jnt_type[j] == JNT_FREE:
            q[a:a + 3] = q[a:a + 3] + dt * qvel[d:d + 3]
            w = qvel[d + 3:d + 6]
            nw = np.sqrt(w @ w)
            quat = q[a + 3:a + 7]
            if nw > MINVAL:
                quat = qmul(quat, qaxisangle(w / nw, nw * dt))
            q[a + 3:a + 7] = qnormalize(quat)
        else:
            q[a] = q[a] + dt * qvel[d]
    return q


def forward(m, qpos, qvel, ctrl, qfrc_applied=None, warm=None, fscale=1.0, mscale=1.0):
    """Everything of one substep up to (and including) the constraint solve."""
    K = kinematics(m, qpos)
    C = com_pos(m, K, mscale)
    M, crbs = crb(m, C)
    L = factor_ldl(m, M)
    cvel, cdofd = com_vel(m, C, qvel)
    bias = rne(m, C, cvel, cdofd, qvel)
    fact, kvd = actuation(m, qpos, qvel, ctrl)
    smooth = fact - m.dof_damping * qvel - bias
    if qfrc_applied is not None:
        smooth = smooth + qfrc_applied
    a0 = solve_ldl(m, L, smooth)
    cons, dropped = collide(m, K, fscale)
    E = constraints(m, C, cons, qpos, qvel)
    if getattr(m.opt, "solver", "newton") == "cg":
        qacc, force, qfrc_con, its = cg(m, M, L, E, smooth, warm)
    else:
        qacc, force, qfrc_con, its = newton(m, M, E, smooth, a0, warm)
    return dict(K=K, C=C, M=M, qLD=L, crb=crbs, cvel=cvel, cdofd=cdofd, bias=bias, qfrc_actuator=fact, kvd=kvd,
                qfrc_smooth=smooth, qacc_smooth=a0, contacts=cons, dropped=dropped, efc=E, qacc=qacc,
                efc_force=force, qfrc_constraint=qfrc_con, iterations=its)


def step(m, qpos, qvel, ctrl, qfrc_applied=None, warm=None, fscale=1.0, mscale=1.0):
    """One substep: forward, implicitfast velocity update, position integration.
    Returns (qpos, qvel, qacc_warmstart, forward-dict)."""
    dt = m.opt.timestep
    F = forward(m, qpos, qvel, ctrl, qfrc_applied, warm, fscale, mscale)
    Mt = F["M"].copy()
    Mt[np.diag_indices(m.nv)] += dt * (m.dof_damping + F["kvd"])
    Lt = factor_ldl(m, Mt)
    acc = solve_ldl(m, Lt, F["qfrc_smooth"] + F["qfrc_constraint"])
    qvel_new = qvel + dt * acc
    qpos_new = integrate_pos(m, qpos, qvel_new, dt)
    return qpos_new, qvel_new, F["qacc"], F


def set_const(m, qpos0=None):
    """Inverse weights at qpos0 from this oracle's own M (model.set_const)."""
    q = m.qpos0 if qpos0 is None else qpos0
    K = kinematics(m, q)
    C = com_pos(m, K)
    M, _ = crb(m, C)
    jac = [np.zeros((3, m.nv))] + [point_jac(m, C, b, K["xipos"][b]) for b in range(1, m.nbody)]
    m.set_const(M, jac)
    return M


# ----------------------------------------------------------------------------- velocity task (3-D)
# The fused task stage of paper_2601_22074_b200/sim3d/task.py restated: the reference's manager
# pipeline (env.py:219-259: action -> decimation x substep -> termination -> reward -> masked reset ->
# command -> observation) on the 3-D model, with mjlab's velocity-tracking terms.

U64 = np.uint64
GOLDEN = U64(0x9E3779B97F4A7C15)
SALT = U64(0xD1B54A32D192ED03)


def mix64(z):
    with np.errstate(over="ignore"):
        z = U64(z)
        z = (z ^ (z >> U64(30))) * U64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> U64(27))) * U64(0x94D049BB133111EB)
        return z ^ (z >> U64(31))


def stream_key(seed, world, purpose):
    with np.errstate(over="ignore"):
        return mix64(mix64(U64(seed) * GOLDEN) ^ (U64(world + 1) * SALT) ^ mix64(U64(purpose)))


def uniform(key, ctr):
    """U[0,1) from word mix(key + ctr * GOLDEN) (the rng.py:97-105 construction)."""
    with np.errstate(over="ignore"):
        w = mix64(U64(key) + U64(ctr) * GOLDEN)
    return float(w >> U64(11)) * (1.0 / 9007199254740992.0)


def terrain_height(m, x, y):
    if not m.terrain_is_hfield:
        return 0.0
    h = hfield_point(m, np.array([x, y, 0.0]), 0.0)
    if h is None:
        return 0.0
    d, n = h
    return -d / n[2]


def base_frame(m, qpos, qvel):
    R = qmat(qnormalize(qpos[3:7]))
    return R.T @ qvel[0:3], qvel[3:6].copy(), R.T @ np.array([0.0, 0.0, -1.0]), R


class TaskOracle:
    """Per-world numpy restatement of the fused 3-D velocity task (one control step = decimation substeps)."""

    def __init__(self, m, cfg, nworld, seed=0, world_offset=0):
        self.m, self.cfg, self.n, self.seed, self.off = m, cfg, nworld, seed, world_offset
        self.default = cfg.default_qpos.copy()
        act = m.actuator_qposadr
        self.qpos = np.tile(self.default, (nworld, 1))
        self.qvel = np.zeros((nworld, m.nv))
        self.warm = np.zeros((nworld, m.nv))
        self.action = np.zeros((nworld, m.nu))
        self.prev_action = np.zeros((nworld, m.nu))
        self.cmd = np.zeros((nworld, 3))
        self.cmd_timer = np.zeros(nworld, dtype=np.int64)
        self.episode_step = np.zeros(nworld, dtype=np.int64)
        self.ep_return = np.zeros(nworld)
        self.global_step = 0
        self.act_default = self.default[act]
        self.fscale = np.ones(nworld)          # startup event: per-world friction scale
        self.mscale = np.ones(nworld)          # startup event: per-world base-mass scale
        self.ev_timer = np.zeros(nworld)       # interval event: time to the next push
        self.level = np.zeros(nworld, dtype=np.int64)   # terrain curriculum row
        self.spawn = np.zeros((nworld, 2))
        self.cmd_dist = np.zeros(nworld)
        self.sensors = tuple(cfg.sensors(m)) if hasattr(cfg, "sensors") else ()
        self.sensor = np.zeros((nworld, len(self.sensors)))

    def _contact_counts(self, contacts):
        """Contacts of each sensor among one substep's (kept) contacts: one geom in the sensor's first set,
        the other in its second (None: any)."""
        out = np.zeros(len(self.sensors))
        for c in contacts:
            g1, g2 = c["geom1"], c["geom2"]
            for k, (_, a, b) in enumerate(self.sensors):
                if (g1 in a and (b is None or g2 in b)) or (g2 in a and (b is None or g1 in b)):
                    out[k] += 1.0
        return out

    def _substeps(self, w, ctrl, fscale=1.0, mscale=1.0):
        """decimation substeps of world w; sensor[w] = the most contacts of each sensor in one substep."""
        q, v, warm = self.qpos[w], self.qvel[w], self.warm[w]
        found = np.zeros(len(self.sensors))
        for _ in range(self.cfg.decimation):
            q, v, warm, F = step(self.m, q, v, ctrl, warm=warm, fscale=fscale, mscale=mscale)
            found = np.maximum(found, self._contact_counts(F["contacts"]))
        self.qpos[w], self.qvel[w], self.warm[w] = q, v, warm
        self.sensor[w] = found
        return q, v, found

    def _curriculum_on(self):
        return getattr(self.cfg, "curriculum", None) is not None

    def _events_on(self):
        return getattr(self.cfg, "push_interval", None) is not None

    def key(self, w, purpose):
        return stream_key(self.seed, self.off + w, purpose)

    def reset_world(self, w, ctr):
        m, cfg = self.m, self.cfg
        kr = self.key(w, 1)
        q = self.default.copy()
        hinge = m.jnt_qposadr[m.jnt_type == 3]
        for i, a in enumerate(hinge):
            q[a] += cfg.reset_joint_jitter * (2.0 * uniform(kr, ctr * 256 + i) - 1.0)
        q[0] = cfg.spawn_half_extent * (2.0 * uniform(kr, ctr * 256 + 200) - 1.0)
        q[1] = cfg.spawn_half_extent * (2.0 * uniform(kr, ctr * 256 + 201) - 1.0)
        if self._curriculum_on():  # centre of the world's (level, column) patch
            rows, cols, patch = cfg.curriculum
            q[0] += ((self.off + w) % cols + 0.5) * patch
            q[1] += (self.level[w] + 0.5) * patch
            self.spawn[w] = q[0:2]
            self.cmd_dist[w] = 0.0
        yaw = np.pi * (2.0 * uniform(kr, ctr * 256 + 202) - 1.0)
        q[2] = self.default[2] + terrain_height(m, q[0], q[1])
        q[3:7] = (np.cos(0.5 * yaw), 0.0, 0.0, np.sin(0.5 * yaw))
        self.qpos[w] = q
        self.qvel[w] = 0.0
        self.warm[w] = 0.0
        self.action[w] = 0.0
        self.prev_action[w] = 0.0
        self.episode_step[w] = 0
        self.ep_return[w] = 0.0
        self.resample(w, ctr)
        if self._events_on():
            self.draw_push_timer(w, ctr, 1)

    def resample(self, w, ctr):
        kc = self.key(w, 2)
        for i, (lo, hi) in enumerate(self.cfg.command_ranges):
            self.cmd[w, i] = lo + (hi - lo) * uniform(kc, ctr * 4 + i)
        self.cmd_timer[w] = self.cfg.command_resample_steps

    def reset(self):
        if self._curriculum_on():  # initial levels (purpose 6, counter 0)
            for w in range(self.n):
                u = uniform(self.key(w, 6), 0)
                self.level[w] = min(int(u * (self.cfg.curriculum_max_init_level + 1)), self.cfg.curriculum[0] - 1)
        if self._events_on():  # startup randomisation (purpose 5, counter 0, slot 0)
            lo, hi = self.cfg.friction_range
            mlo, mhi = self.cfg.base_mass_range
            for w in range(self.n):
                self.fscale[w] = lo + (hi - lo) * uniform(self.key(w, 5), 0)
                self.mscale[w] = mlo + (mhi - mlo) * uniform(self.key(w, 5), 5)
        for w in range(self.n):
            self.reset_world(w, 0)
        return self.observe(0)

    def interval_push(self, w, ctr):
        """EventManager.apply_interval: U(-v, v) on the base's planar velocity when the timer runs out."""
        if not self._events_on():
            return
        cfg = self.cfg
        self.ev_timer[w] -= self.m.opt.timestep * cfg.decimation
        if self.ev_timer[w] <= 0.0:
            k5, pv = self.key(w, 5), cfg.push_velocity
            self.qvel[w, 0] += pv * (2.0 * uniform(k5, ctr * 8 + 2) - 1.0)
            self.qvel[w, 1] += pv * (2.0 * uniform(k5, ctr * 8 + 3) - 1.0)
            self.draw_push_timer(w, ctr, 4)

    def draw_push_timer(self, w, ctr, slot):
        lo, hi = self.cfg.push_interval
        self.ev_timer[w] = lo + (hi - lo) * uniform(self.key(w, 5), ctr * 8 + slot)

    def observe(self, ctr):
        m, cfg = self.m, self.cfg
        act = m.actuator_qposadr
        dofs = m.actuator_dofadr
        out = np.zeros((self.n, cfg.obs_dim(m)))
        for w in range(self.n):
            v, om, g, R = base_frame(m, self.qpos[w], self.qvel[w])
            parts = [v, om, g, self.cmd[w], self.qpos[w][act] - self.act_default, self.qvel[w][dofs], self.action[w]]
            o = np.concatenate(parts)
            if cfg.height_scan:
                o = np.concatenate([o, self.height_scan(w)])
            ko = self.key(w, 3)
            scales = cfg.noise_vector(m)
            for i in range(o.size):
                if scales[i] > 0.0:
                    o[i] += scales[i] * (2.0 * uniform(ko, ctr * 1024 + i) - 1.0)
            out[w] = o
        return out

    def velocity_extras(self, w, found):
        """(|centroidal angular momentum of the robot|^2, joint-limit violation, foot slip) at the final state
        (the velocity kind's mjlab penalties; each computed only when its weight is nonzero)."""
        m, cfg = self.m, self.cfg
        wts = tuple(cfg.reward_weights) + (0.0,) * 9
        q, v = self.qpos[w], self.qvel[w]
        lim = 0.0
        if wts[7] != 0.0:
            for j in range(m.njnt):
                if m.jnt_limited[j]:
                    lo, hi = m.jnt_range[j]
                    x = q[m.jnt_qposadr[j]]
                    lim += max(lo - x, 0.0) + max(x - hi, 0.0)
        feet = cfg.foot_bodies(m)
        h, slip = np.zeros(3), 0.0
        if wts[6] != 0.0 or (wts[8] != 0.0 and feet):
            K = kinematics(m, q)
            C = com_pos(m, K, self.mscale[w])
            if wts[6] != 0.0:
                for b in range(1, m.nbody):
                    if m.body_treeid[b] != 0:
                        continue
                    vb = np.zeros(6)
                    for dd in m.body_chain[b]:
                        vb = vb + C["cdof"][dd] * v[dd]
                    h = h + inert_mul(C["cinert"][b], vb)[:3]
            if wts[8] != 0.0:
                for k, b in enumerate(feet):
                    if found[k] > 0:
                        st = body_state(m, K, C, v, b)
                        slip += st[7] * st[7] + st[8] * st[8]
        return float(h @ h), lim, slip

    def height_scan(self, w):
        m, cfg = self.m, self.cfg
        q = self.qpos[w]
        quat = qnormalize(q[3:7])
        yaw = np.arctan2(2.0 * (quat[0] * quat[3] + quat[1] * quat[2]), 1.0 - 2.0 * (quat[2] ** 2 + quat[3] ** 2))
        c, s = np.cos(yaw), np.sin(yaw)
        out = []
        for (ox, oy) in cfg.scan_points():
            x = q[0] + c * ox - s * oy
            y = q[1] + s * ox + c * oy
            h = q[2] - terrain_height(m, x, y) - cfg.scan_offset
            out.append(min(max(h, -1.0), 1.0))
        return np.array(out)

    def step(self, actions):
        """One control step of every world; returns (obs, reward, terminated, truncated)."""
        m, cfg = self.m, self.cfg
        self.global_step += 1
        ctr = self.global_step
        dtc = m.opt.timestep * cfg.decimation
        rew = np.zeros(self.n)
        term = np.zeros(self.n, dtype=bool)
        trunc = np.zeros(self.n, dtype=bool)
        act = m.actuator_qposadr
        for w in range(self.n):
            a = np.clip(actions[w], -cfg.action_clip, cfg.action_clip)
            self.prev_action[w] = self.action[w]
            self.action[w] = a
            ctrl = self.act_default + cfg.action_scale * a
            q, v, found = self._substeps(w, ctrl, self.fscale[w], self.mscale[w])
            vb, om, g, _ = base_frame(m, q, v)
            e_xy = (self.cmd[w, 0] - vb[0]) ** 2 + (self.cmd[w, 1] - vb[1]) ** 2
            terms = (np.exp(-e_xy / cfg.track_sigma), np.exp(-((self.cmd[w, 2] - om[2]) ** 2) / cfg.track_sigma),
                     vb[2] * vb[2], om[0] * om[0] + om[1] * om[1],
                     float(np.sum((self.action[w] - self.prev_action[w]) ** 2)), g[0] * g[0] + g[1] * g[1],
                     *self.velocity_extras(w, found))
            r = 0.0
            for wt, t in zip(cfg.reward_weights, terms):
                r += wt * t * dtc
            rew[w] = r
            self.ep_return[w] += r
            h = q[2] - terrain_height(m, q[0], q[1])
            nonfinite = not (np.all(np.isfinite(q)) and np.all(np.isfinite(v)))
            term[w] = bool(h < cfg.min_height or g[2] > cfg.max_tilt_cos or nonfinite)
            self.episode_step[w] += 1
            trunc[w] = bool(self.episode_step[w] >= cfg.episode_steps)
            if self._curriculum_on():
                self.cmd_dist[w] += np.sqrt(self.cmd[w, 0] ** 2 + self.cmd[w, 1] ** 2) * dtc
        for w in range(self.n):
            if (term[w] or trunc[w]) and self._curriculum_on():  # on the finished episode, before the reset
                walked = np.sqrt(np.sum((self.qpos[w, 0:2] - self.spawn[w]) ** 2))
                if walked > cfg.curriculum_promote * self.cmd_dist[w]:
                    self.level[w] = min(self.level[w] + 1, cfg.curriculum[0] - 1)
                elif walked < cfg.curriculum_demote * self.cmd_dist[w]:
                    self.level[w] = max(self.level[w] - 1, 0)
            if term[w] or trunc[w]:
                self.reset_world(w, ctr)
            else:
                self.cmd_timer[w] -= 1
                if self.cmd_timer[w] <= 0:
                    self.resample(w, ctr)
            self.interval_push(w, ctr)  # every world, after resets / commands
        return self.observe(ctr), rew, term, trunc


# ----------------------------------------------------------------------------- ray casting (sensors)
# Specification of s3_raycast / s3_depth: nearest hit along o + t d (|d| = 1, 0 < t <= max_dist)
# over every geom of the world except those on `exclude_body`; -1 / geom -1 when nothing is hit.

HF_MARCH = 0.5     # march step in units of the heightfield spacing
HF_BISECT = 24     # bisection steps after a sign change


def ray_plane(n, p0, o, d):
    den = n @ d
    if not den < 0.0:
        return np.inf
    t = (n @ (p0 - o)) / den
    return t if t > 0.0 else np.inf


def ray_sphere(c, r, o, d):
    oc = o - c
    b = oc @ d
    cc = oc @ oc - r * r
    disc = b * b - cc
    if disc < 0.0:
        return np.inf
    sq = np.sqrt(disc)
    t = -b - sq
    if t > 0.0:
        return t
    t = -b + sq
    return t if t > 0.0 else np.inf


def ray_capsule(c, ax, hl, r, o, d):
    best = min(ray_sphere(c - ax * hl, r, o, d), ray_sphere(c + ax * hl, r, o, d))
    # cylinder part
    oc = o - c
    dd = d - ax * (d @ ax)
    oo = oc - ax * (oc @ ax)
    a = dd @ dd
    if a > 1e-12:
        b = oo @ dd
        cc = oo @ oo - r * r
        disc = b * b - a * cc
        if disc >= 0.0:
            sq = np.sqrt(disc)
            for t in ((-b - sq) / a, (-b + sq) / a):
                if t > 0.0:
                    z = (oc + d * t) @ ax
                    if -hl <= z <= hl and t < best:
                        best = t
                    break
    return best


def ray_box(c, R, size, o, d):
    ol = R.T @ (o - c)
    dl = R.T @ d
    tmin, tmax = -np.inf, np.inf
    for k in range(3):
        if abs(dl[k]) < 1e-12:
            if ol[k] < -size[k] or ol[k] > size[k]:
                return np.inf
            continue
        t1 = (-size[k] - ol[k]) / dl[k]
        t2 = (size[k] - ol[k]) / dl[k]
        if t1 > t2:
            t1, t2 = t2, t1
        tmin = max(tmin, t1)
        tmax = min(tmax, t2)
    if tmax < tmin or tmax <= 0.0:
        return np.inf
    return tmin if tmin > 0.0 else tmax


def _hf_f(m, p):
    h = hfield_point(m, p, 0.0)
    if h is None:
        return 1.0  # outside the grid: no terrain
    return h[0]


def ray_hfield(m, o, d, tmax):
    step = HF_MARCH * m.hfield_spacing
    t0 = 0.0
    f0 = _hf_f(m, o)
    if f0 < 0.0:
        return np.inf  # starts below the terrain
    nstep = int(np.ceil(tmax / step))
    for i in range(1, nstep + 1):
        t1 = min(i * step, tmax)
        f1 = _hf_f(m, o + d * t1)
        if f1 < 0.0:
            a, b = t0, t1
            for _ in range(HF_BISECT):
                mid = 0.5 * (a + b)
                if _hf_f(m, o + d * mid) < 0.0:
                    b = mid
                else:
                    a = mid
            return b
        t0 = t1
    return np.inf


def raycast(m, K, o, d, max_dist, exclude_body=-1):
    best, gid = np.inf, -1
    for g in range(m.ngeom):
        if m.geom_bodyid[g] == exclude_body:
            continue
        t = m.geom_type[g]
        c, R, s = K["geom_xpos"][g], K["geom_xmat"][g], m.geom_size[g]
        if t == GEOM_PLANE:
            tt = ray_plane(R[:, 2], c, o, d)
        elif t == GEOM_HFIELD:
            tt = ray_hfield(m, o, d, max_dist)
        elif t == GEOM_SPHERE:
            tt = ray_sphere(c, s[0], o, d)
        elif t == GEOM_CAPSULE:
            tt = ray_capsule(c, R[:, 2], s[1], s[0], o, d)
        else:
            tt = ray_box(c, R, s, o, d)
        if tt < best:
            best, gid = tt, g
    if not best <= max_dist:
        return -1.0, -1
    return best, gid


def camera_rays(K, cam_geom, width, height, fovy, offset=np.zeros(3)):
    """Pinhole rays of a camera fixed to geom `cam_geom`: forward +x, right -y, up +z of the geom frame."""
    R, c = K["geom_xmat"][cam_geom], K["geom_xpos"][cam_geom]
    ty = np.tan(0.5 * fovy)
    tx = ty * width / height
    o = c + R @ offset
    dirs = np.zeros((height, width, 3))
    for i in range(height):
        for j in range(width):
            a = (2.0 * (j + 0.5) / width - 1.0) * tx
            b = (1.0 - 2.0 * (i + 0.5) / height) * ty
            dl = np.array([1.0, -a, b])
            dl = dl / np.sqrt(dl @ dl)
            dirs[i, j] = R @ dl
    return o, dirs


# ----------------------------------------------------------------------------- motion imitation task (3-D)
# The fused task of paper_2601_22074_b200/sim3d/task.py with kind = motion (BeyondMimic-style): a
# reference-motion command (per-world motion time + spawn anchor), reference state initialisation,
# exp-kernel tracking rewards, deviation terminations, end-of-clip truncation.


def qconj(q):
    return np.array([q[0], -q[1], -q[2], -q[3]])


def quat_rotvec(q):
    """Rotation vector of a unit quaternion (shortest arc)."""
    if q[0] < 0.0:
        q = -q
    s = np.sqrt(q[1] * q[1] + q[2] * q[2] + q[3] * q[3])
    if s < 1e-12:
        return 2.0 * q[1:4]
    ang = 2.0 * np.arctan2(s, q[0])
    return q[1:4] * (ang / s)


def motion_ref(cfg, t):
    """Reference qpos / qvel at motion time t (linear; quaternion nlerp with sign alignment)."""
    Q, V, fdt = cfg.motion_qpos, cfg.motion_qvel, cfg.motion_dt
    F = Q.shape[0]
    f = t / fdt
    i0 = int(np.floor(f))
    i0 = min(max(i0, 0), F - 2)
    a = f - i0
    q = (1.0 - a) * Q[i0] + a * Q[i0 + 1]
    q0, q1 = Q[i0, 3:7], Q[i0 + 1, 3:7]
    if q0 @ q1 < 0.0:
        q1 = -q1
    qq = (1.0 - a) * q0 + a * q1
    q[3:7] = qq / np.sqrt(qq @ qq)
    v = (1.0 - a) * V[i0] + a * V[i0 + 1]
    return q, v


def body_state(m, K, C, qvel, b):
    """World state of body b: position, orientation, linear velocity of its origin, angular velocity
    (the sum of the motion vectors of the dofs on its chain, about the tree's com)."""
    v = np.zeros(6)
    for d in m.body_chain[b]:
        v = v + C["cdof"][d] * qvel[d]
    r = K["xpos"][b] - C["com"][m.body_treeid[b]]
    return np.concatenate([K["xpos"][b], K["xquat"][b], v[3:6] + np.cross(v[0:3], r), v[0:3]])


def motion_body_table(m, cfg):
    """(F, 1 + ntrack, 13) clip body states, anchor first (s3_motion_bodies)."""
    anchor, bodies = cfg.tracked(m)
    Q, V = cfg.motion_qpos, cfg.motion_qvel
    out = np.zeros((Q.shape[0], 1 + len(bodies), 13))
    for f in range(Q.shape[0]):
        K = kinematics(m, Q[f])
        C = com_pos(m, K)
        for k, b in enumerate((anchor,) + tuple(bodies)):
            out[f, k] = body_state(m, K, C, V[f], b)
    return out


def motion_body_ref(cfg, table, t):
    """Clip body states at motion time t (linear; quaternion nlerp with sign alignment)."""
    F = table.shape[0]
    f = t / cfg.motion_dt
    i0 = min(max(int(np.floor(f)), 0), F - 2)
    a = f - i0
    b0, b1 = table[i0], table[i0 + 1]
    o = (1.0 - a) * b0 + a * b1
    for k in range(table.shape[1]):
        if b0[k, 3:7] @ b1[k, 3:7] < 0.0:
            o[k, 3:7] = (1.0 - a) * b0[k, 3:7] - a * b1[k, 3:7]
        o[k, 3:7] /= np.sqrt(o[k, 3:7] @ o[k, 3:7])
    return o


def quat_err2(a, b):
    """Squared angle of the rotation conj(a) b."""
    e = qmul(qconj(a), b)
    ang = 2.0 * np.arctan2(np.sqrt(e[1:4] @ e[1:4]), abs(e[0]))
    return ang * ang


class MotionTaskOracle(TaskOracle):
    """Per-world numpy restatement of the motion-imitation kind of the fused 3-D task.
    cmd[w] = (motion time, anchor x, anchor y)."""

    def __init__(self, m, cfg, nworld, seed=0, world_offset=0):
        super().__init__(m, cfg, nworld, seed, world_offset)
        self.anchor, self.bodies = cfg.tracked(m)
        self.body_table = motion_body_table(m, cfg)
        # adaptive start-time sampling (BeyondMimic): failure average, cumulative weights, this step's counts
        self.nbins = cfg.n_bins()
        self.bin_failed = np.zeros(self.nbins)
        self.bin_cum = np.zeros(self.nbins)
        self.bin_now = np.zeros(self.nbins, dtype=np.int64)
        if self.nbins:
            self.fold_bins()  # zero counts: the uniform initial weights

    def fold_bins(self):
        """failed <- alpha now + (1 - alpha) failed; cumulative sums of q_b = sum_i w_i (failed_min(b+i, nb-1)
        + uniform / nb), w_i = lambda^i normalised (BeyondMimic's adaptive sampling, bins in order)."""
        cfg, nb = self.cfg, self.nbins
        a = cfg.adaptive_alpha
        for b in range(nb):
            self.bin_failed[b] = a * float(self.bin_now[b]) + (1.0 - a) * self.bin_failed[b]
        self.bin_now[:] = 0
        lam = cfg.adaptive_lambda ** np.arange(cfg.adaptive_kernel_size, dtype=np.float64)
        w = lam / lam.sum()
        u = cfg.adaptive_uniform_ratio / nb
        acc = 0.0
        for b in range(nb):
            q = 0.0
            for i in range(len(w)):
                q += w[i] * (self.bin_failed[min(b + i, nb - 1)] + u)
            acc += q
            self.bin_cum[b] = acc

    def start_time(self, kr, ctr):
        """Start time of a reset: a bin by the cumulative weights of the last fold and a uniform time inside
        it (adaptive), or uniform over the first motion_start_frac of the clip."""
        if not self.nbins:
            return self.cfg.motion_start_frac * self.clip_end() * uniform(kr, ctr * 256 + 203)
        target = uniform(kr, ctr * 256 + 203) * self.bin_cum[-1]
        b = 0
        while b < self.nbins - 1 and not target < self.bin_cum[b]:
            b += 1
        return (b + uniform(kr, ctr * 256 + 204)) / self.nbins * self.clip_end()

    def body_errors(self, w):
        """BeyondMimic's body errors (means over the tracked bodies): position and orientation with the
        clip's bodies re-expressed about the robot's anchor (its xy, the clip anchor's height over the terrain
        under the spawn anchor, the yaw between the anchors), world linear and angular velocity."""
        m = self.m
        K = kinematics(m, self.qpos[w])
        C = com_pos(m, K)
        rb = [body_state(m, K, C, self.qvel[w], b) for b in (self.anchor,) + tuple(self.bodies)]
        rf = motion_body_ref(self.cfg, self.body_table, self.cmd[w, 0])
        pa, qa, pr, qr = rb[0][0:3], rb[0][3:7], rf[0, 0:3], rf[0, 3:7]
        dq = qmul(qa, qconj(qr))
        yaw = np.arctan2(2.0 * (dq[0] * dq[3] + dq[1] * dq[2]), 1.0 - 2.0 * (dq[2] * dq[2] + dq[3] * dq[3]))
        dy = np.array([np.cos(0.5 * yaw), 0.0, 0.0, np.sin(0.5 * yaw)])
        tz = pr[2] + terrain_height(m, pr[0] + self.cmd[w, 1], pr[1] + self.cmd[w, 2])
        R = qmat(dy)
        e = np.zeros(4)
        for k in range(1, len(rb)):
            p = np.array([pa[0], pa[1], tz]) + R @ (rf[k, 0:3] - pr)
            e[0] += float((p - rb[k][0:3]) @ (p - rb[k][0:3]))
            e[1] += quat_err2(qmul(dy, rf[k, 3:7]), rb[k][3:7])
            e[2] += float((rf[k, 7:10] - rb[k][7:10]) @ (rf[k, 7:10] - rb[k][7:10]))
            e[3] += float((rf[k, 10:13] - rb[k][10:13]) @ (rf[k, 10:13] - rb[k][10:13]))
        return e / len(self.bodies)

    def clip_end(self):
        return (self.cfg.motion_qpos.shape[0] - 1) * self.cfg.motion_dt

    def reset_world(self, w, ctr):
        m, cfg = self.m, self.cfg
        kr = self.key(w, 1)
        t0 = self.start_time(kr, ctr)
        ax = cfg.spawn_half_extent * (2.0 * uniform(kr, ctr * 256 + 200) - 1.0)
        ay = cfg.spawn_half_extent * (2.0 * uniform(kr, ctr * 256 + 201) - 1.0)
        q, v = motion_ref(cfg, t0)
        q = q.copy()
        q[0] += ax
        q[1] += ay
        q[2] += terrain_height(m, q[0], q[1])
        self.qpos[w] = q
        self.qvel[w] = v
        self.warm[w] = 0.0
        self.action[w] = 0.0
        self.prev_action[w] = 0.0
        self.episode_step[w] = 0
        self.ep_return[w] = 0.0
        self.cmd[w] = (t0, ax, ay)
        self.cmd_timer[w] = 0
        if self._events_on():
            self.draw_push_timer(w, ctr, 1)

    def resample(self, w, ctr):
        pass

    def _errors(self, w):
        m, cfg = self.m, self.cfg
        q, v = self.qpos[w], self.qvel[w]
        qr, vr = motion_ref(cfg, self.cmd[w, 0])
        pr = qr[0:3] + np.array([self.cmd[w, 1], self.cmd[w, 2], terrain_height(m, qr[0] + self.cmd[w, 1],
                                                                               qr[1] + self.cmd[w, 2])])
        quat = qnormalize(q[3:7])
        R = qmat(quat)
        pos_err_b = R.T @ (pr - q[0:3])
        rot_err = quat_rotvec(qmul(qconj(quat), qnormalize(qr[3:7])))
        return qr, vr, pos_err_b, rot_err

    def observe(self, ctr):
        m, cfg = self.m, self.cfg
        act, dofs = m.actuator_qposadr, m.actuator_dofadr
        out = np.zeros((self.n, cfg.obs_dim(m)))
        for w in range(self.n):
            vb, om, g, _ = base_frame(m, self.qpos[w], self.qvel[w])
            qr, vr, pe, re = self._errors(w)
            o = np.concatenate([qr[act] - self.act_default, vr[dofs], vb, om, g, pe, re,
                                self.qpos[w][act] - self.act_default, self.qvel[w][dofs], self.action[w]])
            ko = self.key(w, 3)
            scales = cfg.noise_vector(m)
            for i in range(o.size):
                if scales[i] > 0.0:
                    o[i] += scales[i] * (2.0 * uniform(ko, ctr * 1024 + i) - 1.0)
            out[w] = o
        return out

    def step(self, actions):
        m, cfg = self.m, self.cfg
        self.global_step += 1
        ctr = self.global_step
        dtc = m.opt.timestep * cfg.decimation
        rew = np.zeros(self.n)
        term = np.zeros(self.n, dtype=bool)
        trunc = np.zeros(self.n, dtype=bool)
        act, dofs = m.actuator_qposadr, m.actuator_dofadr
        for w in range(self.n):
            a = np.clip(actions[w], -cfg.action_clip, cfg.action_clip)
            self.prev_action[w] = self.action[w]
            self.action[w] = a
            ctrl = self.act_default + cfg.action_scale * a
            q, v, found = self._substeps(w, ctrl, self.fscale[w], self.mscale[w])
            self.cmd[w, 0] += dtc
            qr, vr, pe, re = self._errors(w)
            s = cfg.motion_sigmas
            ej = float(np.sum((q[act] - qr[act]) ** 2))
            ev = float(np.sum((v[dofs] - vr[dofs]) ** 2))
            terms = [np.exp(-ej / s[0]), np.exp(-ev / s[1]), np.exp(-float(pe @ pe) / s[2]),
                     np.exp(-float(re @ re) / s[3]), float(np.sum((self.action[w] - self.prev_action[w]) ** 2)),
                     0.0, 0.0, 0.0, 0.0, float(found[0]) if (cfg.self_collision and len(found)) else 0.0]
            be = self.body_errors(w)
            for k in range(4):
                terms[5 + k] = np.exp(-be[k] / s[4 + k])
            r = 0.0
            for wt, t in zip(cfg.reward_weights, terms):
                r += wt * t * dtc
            rew[w] = r
            self.ep_return[w] += r
            nonfinite = not (np.all(np.isfinite(q)) and np.all(np.isfinite(v)))
            term[w] = bool(abs(pe[2]) > cfg.max_height_error or float(np.sqrt(re @ re)) > cfg.max_ori_error
                           or nonfinite)
            if term[w] and self.nbins:  # a failure in the bin of its motion time
                b = int(np.floor(self.cmd[w, 0] / self.clip_end() * self.nbins))
                self.bin_now[min(max(b, 0), self.nbins - 1)] += 1
            self.episode_step[w] += 1
            trunc[w] = bool(self.episode_step[w] >= cfg.episode_steps or self.cmd[w, 0] >= self.clip_end() - 1e-9)
        for w in range(self.n):
            if term[w] or trunc[w]:
                self.reset_world(w, ctr)  # with the weights of the previous fold
            self.interval_push(w, ctr)
        if self.nbins:  # the launch's fold, after every world (the kernel's last-world ticket)
            self.fold_bins()
        return self.observe(ctr), rew, term, trunc


# ----------------------------------------------------------------------------- cube lift task (3-D)
# kind = lift (BASELINE configs[3], mjlab's manipulation example): reach the cube with the claw, lift it
# above lift_height, carry it to a goal; cmd[w] = goal position.


class LiftTaskOracle(TaskOracle):
    def _ee(self, q):
        K = kinematics(self.m, q)
        return K["geom_xpos"][list(self.cfg.tip_geoms)].mean(0)

    def reset_world(self, w, ctr):
        m, cfg = self.m, self.cfg
        kr = self.key(w, 1)
        q = self.default.copy()
        ca = cfg.cube_qposadr
        hinge = [a for a in m.jnt_qposadr[m.jnt_type == 3]]
        for i, a in enumerate(hinge):
            q[a] += cfg.reset_joint_jitter * (2.0 * uniform(kr, ctr * 256 + i) - 1.0)
        q[ca] = cfg.cube_x[0] + (cfg.cube_x[1] - cfg.cube_x[0]) * uniform(kr, ctr * 256 + 200)
        q[ca + 1] = cfg.cube_y[0] + (cfg.cube_y[1] - cfg.cube_y[0]) * uniform(kr, ctr * 256 + 201)
        q[ca + 2] = cfg.cube_half
        yaw = np.pi * (2.0 * uniform(kr, ctr * 256 + 202) - 1.0)
        q[ca + 3:ca + 7] = (np.cos(0.5 * yaw), 0.0, 0.0, np.sin(0.5 * yaw))
        self.qpos[w] = q
        self.qvel[w] = 0.0
        self.warm[w] = 0.0
        self.action[w] = 0.0
        self.prev_action[w] = 0.0
        self.episode_step[w] = 0
        self.ep_return[w] = 0.0
        kc = self.key(w, 2)
        for i, (lo, hi) in enumerate(cfg.goal_ranges):
            self.cmd[w, i] = lo + (hi - lo) * uniform(kc, ctr * 4 + i)
        self.cmd_timer[w] = 0

    def resample(self, w, ctr):
        pass

    def observe(self, ctr):
        m, cfg = self.m, self.cfg
        act, dofs = m.actuator_qposadr, m.actuator_dofadr
        ca = cfg.cube_qposadr
        out = np.zeros((self.n, cfg.obs_dim(m)))
        for w in range(self.n):
            q = self.qpos[w]
            o = np.concatenate([q[act] - self.act_default, self.qvel[w][dofs], q[ca:ca + 3], q[ca + 3:ca + 7],
                                self._ee(q), self.cmd[w], self.action[w]])
            ko = self.key(w, 3)
            scales = cfg.noise_vector(m)
            for i in range(o.size):
                if scales[i] > 0.0:
                    o[i] += scales[i] * (2.0 * uniform(ko, ctr * 1024 + i) - 1.0)
            out[w] = o
        return out

    def step(self, actions):
        m, cfg = self.m, self.cfg
        self.global_step += 1
        ctr = self.global_step
        dtc = m.opt.timestep * cfg.decimation
        rew = np.zeros(self.n)
        term = np.zeros(self.n, dtype=bool)
        trunc = np.zeros(self.n, dtype=bool)
        ca, dofs = cfg.cube_qposadr, m.actuator_dofadr
        for w in range(self.n):
            a = np.clip(actions[w], -cfg.action_clip, cfg.action_clip)
            self.prev_action[w] = self.action[w]
            self.action[w] = a
            ctrl = self.act_default + cfg.action_scale * a
            q, v, found = self._substeps(w, ctrl)
            ee = self._ee(q)
            cube = q[ca:ca + 3]
            d_ee = np.sqrt(np.sum((ee - cube) ** 2))
            lifted = 1.0 if cube[2] > cfg.lift_height else 0.0
            d_goal = np.sqrt(np.sum((cube - self.cmd[w]) ** 2))
            terms = (1.0 - np.tanh(d_ee / cfg.reach_std), lifted, lifted * (1.0 - np.tanh(d_goal / cfg.goal_std)),
                     float(np.sum((self.action[w] - self.prev_action[w]) ** 2)), float(np.sum(v[dofs] ** 2)),
                     float(found[1]) if len(found) > 1 else 0.0)
            r = 0.0
            for wt, t in zip(cfg.reward_weights, terms):
                r += wt * t * dtc
            rew[w] = r
            self.ep_return[w] += r
            nonfinite = not (np.all(np.isfinite(q)) and np.all(np.isfinite(v)))
            term[w] = bool(cube[2] < cfg.min_cube_z or nonfinite)
            self.episode_step[w] += 1
            trunc[w] = bool(self.episode_step[w] >= cfg.episode_steps)
        for w in range(self.n):
            if term[w] or trunc[w]:
                self.reset_world(w, ctr)
        return self.observe(ctr), rew, term, trunc
