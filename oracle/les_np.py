"""CPU oracle (test infrastructure only): numpy restatement of the reference's
eddy-viscosity closures, /root/reference/pkg/src/stagflow/les.py.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline use this
module, as the checker.  Pinned against golden vectors produced by the
reference itself (tests/golden/les*.npz, tests/test_oracle_golden.py).

Layout follows oracle/stagflow_np.py: extended C-order arrays, OGrid tables.
"""

import numpy as np

from .stagflow_np import _sh


def _cell_table(g, table, axis):
    """Per-axis table on the interior (pressure) range, broadcastable."""
    return g.col(table[axis], axis, slice(1, g.shape[axis] + 1))


def gradient_tensor(g, u):
    """les.py:58-88: velocity gradient at the pressure points as (..., 3, 3);
    diagonal from the two faces, off-diagonal from the mean of the four
    surrounding corner differences.  u must have filled ghosts."""
    d = g.dim
    p = g.pdof()
    A = np.zeros(g.shape + (3, 3), dtype=g.dtype)
    for i in range(d):
        A[..., i, i] = (u[i][p] - u[i][_sh(p, i, -1)]) / _cell_table(g, g.dx, i)
    for i in range(d):
        for j in range(d):
            if i == j:
                continue
            # corner differences on the (i, j) lattice: face index ci = 0..n_i
            # along i, corner cj = 0..n_j along j
            box = list(p)
            box[i] = slice(0, g.shape[i] + 1)
            box[j] = slice(0, g.shape[j] + 1)
            box = tuple(box)
            dj = g.col(g.du[j], j, slice(0, g.shape[j] + 1))
            corner = (u[i][_sh(box, j, 1)] - u[i][box]) / dj
            total = None
            for oi in (0, 1):
                for oj in (0, 1):
                    pick = [slice(None)] * d
                    pick[i] = slice(oi, g.shape[i] + oi)
                    pick[j] = slice(oj, g.shape[j] + oj)
                    part = corner[tuple(pick)]
                    total = part if total is None else total + part
            A[..., i, j] = 0.25 * total
    return A


def _tr_prod(x, y):
    return np.einsum("...ij,...ji->...", x, y)


def invariants(A):
    """les.py:91-119: the invariants the models consume."""
    S = 0.5 * (A + np.swapaxes(A, -1, -2))
    W = 0.5 * (A - np.swapaxes(A, -1, -2))
    inv = {}
    inv["q_a"] = -0.5 * _tr_prod(A, A)
    inv["q_s"] = -0.5 * _tr_prod(S, S)
    inv["q_w"] = -0.5 * _tr_prod(W, W)
    r_s = np.einsum("...ij,...jk,...ki->...", S, S, S) / 3.0
    planar = np.all(A[..., 2, :] == 0.0, axis=-1) & np.all(A[..., :, 2] == 0.0, axis=-1)
    if np.any(planar):
        tr2 = S[..., 0, 0] + S[..., 1, 1]
        det2 = S[..., 0, 0] * S[..., 1, 1] - S[..., 0, 1] * S[..., 1, 0]
        r_s = np.where(planar, tr2 * (tr2 * tr2 - 3.0 * det2) / 3.0, r_s)
    inv["r_s"] = r_s
    r_a = np.einsum("...ij,...jk,...ki->...", A, A, A) / 3.0
    axial = np.stack((W[..., 2, 1], W[..., 0, 2], W[..., 1, 0]), axis=-1)
    s_ax = np.einsum("...ij,...j->...i", S, axial)
    v2 = 4.0 * np.einsum("...i,...i->...", s_ax, s_ax)
    inv["v2"] = v2
    inv["p_aa"] = np.einsum("...ij,...ij->...", A, A)
    inv["q_aa"] = v2 + inv["q_a"] * inv["q_a"]
    inv["r_aa"] = r_a * r_a
    return S, inv


def _sym_eigs(m):
    """les.py:122-148: closed-form eigenvalues of symmetric 3x3, descending."""
    m00, m11, m22 = m[..., 0, 0], m[..., 1, 1], m[..., 2, 2]
    m01, m02, m12 = m[..., 0, 1], m[..., 0, 2], m[..., 1, 2]
    off = m01 ** 2 + m02 ** 2 + m12 ** 2
    q = (m00 + m11 + m22) / 3.0
    p2 = (m00 - q) ** 2 + (m11 - q) ** 2 + (m22 - q) ** 2 + 2.0 * off
    pp = np.sqrt(np.maximum(p2 / 6.0, 0.0))
    ok = pp > 0
    ps = np.where(ok, pp, 1.0)
    b00, b11, b22 = (m00 - q) / ps, (m11 - q) / ps, (m22 - q) / ps
    b01, b02, b12 = m01 / ps, m02 / ps, m12 / ps
    det = b00 * (b11 * b22 - b12 * b12) - b01 * (b01 * b22 - b12 * b02) + b02 * (b01 * b12 - b11 * b02)
    phi = np.arccos(np.clip(det / 2.0, -1.0, 1.0)) / 3.0
    e1 = q + 2.0 * pp * np.cos(phi)
    e3 = q + 2.0 * pp * np.cos(phi + 2.0 * np.pi / 3.0)
    e2 = 3.0 * q - e1 - e3
    return np.where(ok, e1, q), np.where(ok, e2, q)


def _det(a):
    return (a[..., 0, 0] * (a[..., 1, 1] * a[..., 2, 2] - a[..., 1, 2] * a[..., 2, 1])
            - a[..., 0, 1] * (a[..., 1, 0] * a[..., 2, 2] - a[..., 1, 2] * a[..., 2, 0])
            + a[..., 0, 2] * (a[..., 1, 0] * a[..., 2, 1] - a[..., 1, 1] * a[..., 2, 0]))


def singular_values(A, extended=True):
    """les.py:160-179: the two leading values from A^T A (extended precision
    in the reference), the smallest from |det| / (s1 s2)."""
    a = A.astype(np.longdouble) if extended else A
    ata = np.einsum("...ki,...kj->...ij", a, a)
    e1, e2 = _sym_eigs(ata)
    s1 = np.sqrt(np.maximum(e1, 0.0)).astype(np.float64)
    s2 = np.sqrt(np.maximum(e2, 0.0)).astype(np.float64)
    det = np.abs(_det(a)).astype(np.float64)
    prod = s1 * s2
    s3 = np.minimum(np.where(prod > 0.0, det / np.where(prod > 0.0, prod, 1.0), 0.0), s2)
    return s1, s2, s3


def singular_values_invariant(A):
    """Check for the product's sigma model (csrc/les.cu): the second
    singular value from the characteristic invariants (no cancellation),
    e2 + e3 = (I2 - I3/e1)/e1, e2 e3 = I3/e1, I2 = sum |c_i x c_j|^2, in
    longdouble.  For nearly two-component gradients this is more accurate
    than the closed form of les.py:122-148 (whose e2 = 3q - e1 - e3 cancels)."""
    a = A.astype(np.longdouble)
    ata = np.einsum("...ki,...kj->...ij", a, a)
    e1, _ = _sym_eigs(ata)
    det = np.abs(_det(a))
    cols = np.swapaxes(a, -1, -2)
    i2 = np.zeros(a.shape[:-2], dtype=np.longdouble)
    for i in range(3):
        for j in range(i + 1, 3):
            cr = np.cross(cols[..., i, :], cols[..., j, :])
            i2 = i2 + np.einsum("...k,...k->...", cr, cr)
    ok = e1 > 0
    e1s = np.where(ok, e1, 1.0)
    p23 = det * det / e1s
    s23 = np.maximum((i2 - p23) / e1s, 0.0)
    e2 = np.where(ok, 0.5 * (s23 + np.sqrt(np.maximum(s23 * s23 - 4.0 * p23, 0.0))), 0.0)
    s1 = np.sqrt(np.maximum(e1, 0.0)).astype(np.float64)
    s2 = np.sqrt(np.maximum(e2, 0.0)).astype(np.float64)
    det = det.astype(np.float64)
    prod = s1 * s2
    s3 = np.minimum(np.where(prod > 0.0, det / np.where(prod > 0.0, prod, 1.0), 0.0), s2)
    return s1, s2, s3


def nu_t_sigma_accurate(g, u, c=None):
    """The sigma model with singular_values_invariant (see there)."""
    c = float(MODEL_CONSTANTS["sigma"] if c is None else c)
    A = gradient_tensor(g, u)
    s1, s2, s3 = singular_values_invariant(A)
    ok = s1 > 0
    val = s3 * (s1 - s2) * (s2 - s3) / np.where(ok, s1 ** 2, 1.0)
    return (c * filter_width(g)) ** 2 * np.where(ok, np.maximum(val, 0.0), 0.0)


def filter_width(g):
    """les.py:297-305 ('geometric'): (prod of the cell widths)^(1/d)."""
    prod = np.ones((1,) * g.dim, dtype=g.dtype)
    for a in range(g.dim):
        prod = prod * _cell_table(g, g.dx, a)
    return np.ascontiguousarray(np.broadcast_to(prod, g.shape)) ** (1.0 / g.dim)


MODEL_CONSTANTS = {
    "smagorinsky": 0.17,
    "vreman": float(np.sqrt(2.5 * 0.17 ** 2)),
    "qr": float(np.sqrt(1.5) / np.pi),
    "wale": float(np.sqrt(2.5 * 0.17)),
    "sigma": 1.35,
    "s3pqr": 0.762,
}


def _pow_or_flag(x, e, bad):
    """les.py:252-261: x^e on x > 0, else 0; a negative exponent on x <= 0
    flags the point degenerate."""
    if e == 0.0:
        return np.ones_like(x), bad
    pos = x > 0
    with np.errstate(divide="ignore", invalid="ignore"):
        v = np.where(pos, x, 1.0) ** e
    if e < 0:
        bad = bad | ~pos
    return np.where(pos, v, 0.0), bad


def nu_t(g, u, kind, c=None, p=-2.5):
    """les.py:360-383: eddy viscosity of one model at the pressure points."""
    c = float(MODEL_CONSTANTS[kind] if c is None else c)
    A = gradient_tensor(g, u)
    S, inv = invariants(A)
    delta = filter_width(g)
    cd2 = (c * delta) ** 2
    if kind == "smagorinsky":
        return cd2 * np.sqrt(np.maximum(-4.0 * inv["q_s"], 0.0))
    if kind == "vreman":
        dm = np.zeros(A.shape[:-2] + (3,), dtype=A.dtype)
        for m in range(g.dim):
            dm[..., m] = np.broadcast_to(_cell_table(g, g.dx, m), g.shape)
        rows = A * dm[..., None, :]
        b = np.zeros(A.shape[:-2], dtype=A.dtype)
        for i in range(3):
            for j in range(i + 1, 3):
                cr = np.cross(rows[..., i, :], rows[..., j, :])
                b = b + np.einsum("...k,...k->...", cr, cr)
        den = inv["p_aa"] / 2.0
        ok = den > 0
        return c ** 2 * np.where(ok, np.sqrt(b / np.where(ok, den, 1.0)), 0.0)
    if kind == "qr":
        ok = inv["q_s"] < 0
        return cd2 * np.where(ok, np.abs(inv["r_s"]) / np.where(ok, -inv["q_s"], 1.0), 0.0)
    if kind == "wale":
        A2 = np.einsum("...ij,...jk->...ik", A, A)
        sd = 0.5 * (A2 + np.swapaxes(A2, -1, -2))
        tr = np.einsum("...ii->...", sd)
        for i in range(3):
            sd[..., i, i] -= tr / 3.0
        sdsd = np.einsum("...ij,...ij->...", sd, sd)
        ss = np.einsum("...ij,...ij->...", S, S)
        den = ss ** 2.5 + sdsd ** 1.25
        ok = den > 0
        return cd2 * np.where(ok, sdsd ** 1.5 / np.where(ok, den, 1.0), 0.0)
    if kind == "sigma":
        s1, s2, s3 = singular_values(A)
        ok = s1 > 0
        val = s3 * (s1 - s2) * (s2 - s3) / np.where(ok, s1 ** 2, 1.0)
        return cd2 * np.where(ok, np.maximum(val, 0.0), 0.0)
    if kind == "s3pqr":
        bad = np.zeros(inv["p_aa"].shape, dtype=bool)
        f1, bad = _pow_or_flag(inv["p_aa"], p, bad)
        f2, bad = _pow_or_flag(inv["q_aa"], -(p + 1.0), bad)
        f3, bad = _pow_or_flag(inv["r_aa"], (p + 2.5) / 3.0, bad)
        return cd2 * np.where(bad, 0.0, f1 * f2 * f3)
    raise ValueError(kind)


def fill_like_pressure(g, f):
    """les.py:420-434: wrap on periodic axes, copy (zero gradient) otherwise."""
    d = g.dim
    for a, n in enumerate(g.shape):
        lo = [slice(None)] * d
        hi = [slice(None)] * d
        s0 = [slice(None)] * d
        s1 = [slice(None)] * d
        lo[a], hi[a] = 0, n + 1
        s0[a], s1[a] = (n, 1) if g.periodic[a] else (1, n)
        f[tuple(lo)] = f[tuple(s0)]
        f[tuple(hi)] = f[tuple(s1)]
    return f


def eddy_stress_divergence(g, u, nut, out=None):
    """les.py:343-417: div(2 nu_t S) on the velocity DOFs, nu_t native at the
    centres (diagonal) and averaged over the four pressure points around a
    corner (off-diagonal); accumulates into ``out`` when given."""
    d = g.dim
    nut = fill_like_pressure(g, nut.copy())
    if out is None:
        out = g.zeros_vel()
    for a in range(d):
        sl = g.udof(a)
        for b in range(d):
            if b == a:
                cs = list(sl)
                cs[a] = slice(sl[a].start, sl[a].stop + 1)
                cs = tuple(cs)
                flux = (u[a][cs] - u[a][_sh(cs, a, -1)]) / g.col(g.dx[a], a, cs[a])
                flux = flux * nut[cs]
                flux = flux * 2.0
                hi = [slice(None)] * d
                hi[a] = slice(1, None)
                lo = [slice(None)] * d
                lo[a] = slice(0, -1)
                out[a][sl] += (flux[tuple(hi)] - flux[tuple(lo)]) / g.col(g.du[a], a, sl[a])
            else:
                cs = list(sl)
                cs[b] = slice(sl[b].start - 1, sl[b].stop)
                cs = tuple(cs)
                s2 = (u[a][_sh(cs, b, 1)] - u[a][cs]) / g.col(g.du[b], b, cs[b])
                s2 = s2 + (u[b][_sh(cs, a, 1)] - u[b][cs]) / g.col(g.du[a], a, cs[a])
                nc = (nut[cs] + nut[_sh(cs, a, 1)]) + (nut[_sh(cs, b, 1)] + nut[_sh(_sh(cs, a, 1), b, 1)])
                nc = nc * 0.25
                flux = s2 * nc
                hi = [slice(None)] * d
                hi[b] = slice(1, None)
                lo = [slice(None)] * d
                lo[b] = slice(0, -1)
                out[a][sl] += (flux[tuple(hi)] - flux[tuple(lo)]) / g.col(g.dx[b], b, sl[b])
    return out


# ---------------------------------------------------------------------------
# Adjoint of the Smagorinsky closure term (no reference counterpart: the
# reference's tape leaves closures out, adjoint.py:374).  Checker for
# csrc/les.cu k_cpb1-3; pinned by the FD identity in
# tests/test_oracle_les_adjoint.py (the reference's checks.py:72-126 protocol).
# ---------------------------------------------------------------------------
def smagorinsky_pullback(g, u, vbar, c=None, scratch_out=None):
    """(dE/du)^T vbar for E(u) = eddy_stress_divergence(u, nu_t(u, smagorinsky))
    on a periodic 3D grid, through the resolved gradients and through nu_t;
    interior result on velocity-shaped extended arrays (ghosts zero)."""
    from .stagflow_np import fill_velocity, periodic_bcs

    c = float(MODEL_CONSTANTS["smagorinsky"] if c is None else c)
    assert g.dim == 3 and all(g.periodic)
    bcs = periodic_bcs(3)
    u = [x.copy() for x in u]
    fill_velocity(g, bcs, u)
    eb = [x.copy() for x in vbar]
    fill_velocity(g, bcs, eb)
    nut = np.zeros(g.ext_shape, dtype=g.dtype)
    nut[g.pdof()] = nu_t(g, u, "smagorinsky", c=c)
    fill_like_pressure(g, nut)
    shape = g.shape
    sl = tuple(slice(1, n + 1) for n in shape)
    idx = [np.arange(1, n + 1) for n in shape]

    def sh(*offs):  # interior slice shifted by (axis, offset) pairs
        s = list(sl)
        for a, o in zip(offs[::2], offs[1::2]):
            s[a] = slice(1 + o, shape[a] + 1 + o)
        return tuple(s)

    def tab(table, a, i):
        r = [1, 1, 1]
        r[a] = -1
        return (1.0 / table[a][i]).reshape(r)

    pairs = [(0, 1), (0, 2), (1, 2)]
    scr = np.zeros((16,) + g.ext_shape, dtype=g.dtype)
    nud = 0.0
    for a in range(3):
        # centre fluxes 2 nu_t A_aa: cotangent Fbar, then gbar = 2 nu Fbar
        fb = eb[a][sh(a, -1)] * tab(g.du, a, idx[a] - 1) - eb[a][sl] * tab(g.du, a, idx[a])
        ga = (u[a][sl] - u[a][sh(a, -1)]) * tab(g.dx, a, idx[a])
        scr[a][sl] = 2.0 * nut[sl] * fb
        nud = nud + 2.0 * ga * fb
    scr[6][sl] = nud
    for p, (a, b) in enumerate(pairs):
        # corner fluxes 2 nu_t S_ab (shared by E_a along b and E_b along a)
        fcb = (eb[a][sl] * tab(g.dx, b, idx[b]) - eb[a][sh(b, 1)] * tab(g.dx, b, idx[b] + 1)) + (
            eb[b][sl] * tab(g.dx, a, idx[a]) - eb[b][sh(a, 1)] * tab(g.dx, a, idx[a] + 1))
        sab = (u[a][sh(b, 1)] - u[a][sl]) * tab(g.du, b, idx[b]) + (u[b][sh(a, 1)] - u[b][sl]) * tab(g.du, a, idx[a])
        nc = 0.25 * ((nut[sl] + nut[sh(a, 1)]) + (nut[sh(b, 1)] + nut[sh(a, 1, b, 1)]))
        scr[3 + p][sl] = fcb * nc
        scr[7 + p][sl] = fcb * sab
    for f in range(10):
        fill_like_pressure(g, scr[f])
    nub = scr[6][sl].copy()
    for p, (a, b) in enumerate(pairs):
        w = scr[7 + p]
        nub += 0.25 * ((w[sl] + w[sh(a, -1)]) + (w[sh(b, -1)] + w[sh(a, -1, b, -1)]))
    A = gradient_tensor(g, u)
    S = 0.5 * (A + np.swapaxes(A, -1, -2))
    mag = np.sqrt(np.maximum(2.0 * np.einsum("...ij,...ij->...", S, S), 0.0))
    cd2 = (c * filter_width(g)) ** 2
    f = np.where(mag > 0, nub * cd2 * 2.0 / np.where(mag > 0, mag, 1.0), 0.0)
    for k, (i, j) in enumerate([(0, 0), (1, 1), (2, 2), (0, 1), (0, 2), (1, 2)]):
        scr[10 + k][sl] = f * S[..., i, j]
    for k in range(10, 16):
        fill_like_pressure(g, scr[k])
    out = g.zeros_vel()
    for i in range(3):
        v = (scr[i][sl] + scr[10 + i][sl]) * tab(g.dx, i, idx[i]) - (
            scr[i][sh(i, 1)] + scr[10 + i][sh(i, 1)]) * tab(g.dx, i, idx[i] + 1)
        for o in range(3):
            if o == i:
                continue
            pr = min(i, o) + max(i, o) - 1
            sb = scr[3 + pr]
            v = v + sb[sh(o, -1)] * tab(g.du, o, idx[o] - 1) - sb[sl] * tab(g.du, o, idx[o])
            ab = scr[13 + pr]
            lo = (ab[sl] + ab[sh(i, 1)]) + (ab[sh(o, -1)] + ab[sh(i, 1, o, -1)])
            hi = (ab[sl] + ab[sh(i, 1)]) + (ab[sh(o, 1)] + ab[sh(i, 1, o, 1)])
            v = v + 0.25 * (lo * tab(g.du, o, idx[o] - 1) - hi * tab(g.du, o, idx[o]))
        out[i][sl] = v
    if scratch_out is not None:
        scratch_out.append(scr)
    return out
