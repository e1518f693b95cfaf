"""numpy restatement of the reference time-step path (TEST INFRASTRUCTURE ONLY).

Every routine cites the reference function it restates
(``/root/reference/pkg/src/stagflow/<file>:<line>``).  Arrays are the
reference's extended C-order arrays (one ghost layer per side, axis 0
slowest).  The floating-point operation order of the reference is kept
(slice-wise numpy ufuncs in the same sequence) so that, for the operators,
fills and steps, the oracle agrees with the reference bit-for-bit; the
golden-vector tests check exactly that.

Fields are plain Python lists of ndarrays (one per velocity component); a
scalar field is a single ndarray.  Boundary conditions are per-axis pairs of
``"P"`` (periodic), ``("D", value)`` (constant Dirichlet, scalar or d-vector)
or ``"S"`` (symmetric).
"""

import math

import numpy as np

try:  # same FFT backend as the reference (transforms.py:9-12)
    from scipy.fft import irfftn as _irfftn, rfftn as _rfftn
except ImportError:  # pragma: no cover
    from numpy.fft import irfftn as _irfftn, rfftn as _rfftn


# --------------------------------------------------------------------------
# grid tables  (grid.py:68-104 profiles, grid.py:127-175 tables)
# --------------------------------------------------------------------------

def uniform_bounds(a, b, n):
    """grid.py:68-71"""
    return np.linspace(a, b, n + 1)


def tanh_bounds(a, b, n, gamma):
    """grid.py:83-91"""
    xi = np.arange(n + 1) / n
    x = a + (b - a) / 2.0 * (1.0 + np.tanh(gamma * (2.0 * xi - 1.0)) / np.tanh(gamma))
    x[0], x[-1] = a, b
    return x


def cosine_bounds(a, b, n):
    """grid.py:74-80"""
    i = np.arange(n + 1)
    x = a + (1.0 - np.cos(np.pi * i / n)) / 2.0 * (b - a)
    x[0], x[-1] = a, b
    return x


def _ext_tables(bnd, periodic):
    """Extended widths/staggered widths/faces/centers of one axis
    (grid.py:143-166), all in float64."""
    bnd = np.asarray(bnd, dtype=float)
    w = np.diff(bnd)
    n = w.size
    dx = np.empty(n + 2)
    dx[1:n + 1] = w
    if periodic:
        dx[0], dx[n + 1], far = w[-1], w[0], w[1 % n]
    else:
        dx[0], dx[n + 1], far = w[0], w[-1], w[-1]
    du = np.empty(n + 2)
    du[:n + 1] = 0.5 * (dx[:n + 1] + dx[1:])
    du[n + 1] = 0.5 * (dx[n + 1] + far)
    xb = np.empty(n + 2)
    xb[:n + 1] = bnd
    xb[n + 1] = bnd[-1] + dx[n + 1]
    xc = np.empty(n + 2)
    xc[1:n + 1] = 0.5 * (bnd[:-1] + bnd[1:])
    xc[0] = bnd[0] - 0.5 * dx[0]
    xc[n + 1] = bnd[-1] + 0.5 * dx[n + 1]
    return dx, du, xb, xc


class OGrid:
    """Immutable staggered grid description (grid.py:115-216) with the
    derived stencil tables of operators.py:38-84."""

    def __init__(self, bounds, periodic, dtype=np.float64):
        self.bounds = [np.asarray(b, dtype=float) for b in bounds]
        self.periodic = tuple(bool(p) for p in periodic)
        self.dtype = np.dtype(dtype)
        self.dim = len(self.bounds)
        self.shape = tuple(b.size - 1 for b in self.bounds)
        self.ext_shape = tuple(n + 2 for n in self.shape)
        self.widths = [np.diff(b) for b in self.bounds]
        tabs = [_ext_tables(b, p) for b, p in zip(self.bounds, self.periodic)]
        cast = lambda v: v.astype(self.dtype)  # noqa: E731  (grid.py:168-171)
        self.dx = [cast(t[0]) for t in tabs]
        self.du = [cast(t[1]) for t in tabs]
        self.xb = [cast(t[2]) for t in tabs]
        self.xc = [cast(t[3]) for t in tabs]
        # interpolation weights (operators.py:47-57)
        self.w_lo = [dx / (2.0 * du) for dx, du in zip(self.dx, self.du)]
        self.w_hi = [1.0 - lo for lo in self.w_lo]
        # diffusion bands (operators.py:69-84)
        self.own_hi, self.own_lo, self.tan_hi, self.tan_lo = [], [], [], []
        for n, dx, du in zip(self.shape, self.dx, self.du):
            oh = np.zeros(n + 2, self.dtype)
            ol = np.zeros(n + 2, self.dtype)
            th = np.zeros(n + 2, self.dtype)
            tl = np.zeros(n + 2, self.dtype)
            oh[:n + 1] = 1.0 / (du[:n + 1] * dx[1:])
            ol[:n + 1] = 1.0 / (du[:n + 1] * dx[:n + 1])
            th[:n + 1] = 1.0 / (dx[:n + 1] * du[:n + 1])
            tl[1:] = 1.0 / (dx[1:] * du[:-1])
            self.own_hi.append(oh)
            self.own_lo.append(ol)
            self.tan_hi.append(th)
            self.tan_lo.append(tl)

    @property
    def uniform(self):
        """grid.py:177-183"""
        return all(np.allclose(w, w[0], rtol=1e-12, atol=0.0) for w in self.widths)

    def col(self, table, axis, sl):
        """A 1D table slice shaped to broadcast along ``axis``."""
        v = table[sl]
        shp = [1] * self.dim
        shp[axis] = v.shape[0]
        return v.reshape(shp)

    def pdof(self):
        """grid.py:193-195"""
        return tuple(slice(1, n + 1) for n in self.shape)

    def udof(self, comp):
        """grid.py:197-209"""
        return tuple(
            slice(1, n) if (a == comp and not self.periodic[a]) else slice(1, n + 1)
            for a, n in enumerate(self.shape)
        )

    def face_coords(self, comp):
        """grid.py:211-216"""
        return [self.xb[a] if a == comp else self.xc[a] for a in range(self.dim)]

    # allocation helpers
    def zeros(self):
        return np.zeros(self.ext_shape, self.dtype)

    def zeros_vel(self):
        return [self.zeros() for _ in range(self.dim)]


def _sh(sl, axis, off):
    """Shift one axis of a slice tuple (operators.py:25-30)."""
    out = list(sl)
    out[axis] = slice(out[axis].start + off, out[axis].stop + off)
    return tuple(out)


def _plane(ndim, axis, idx):
    sl = [slice(None)] * ndim
    sl[axis] = idx
    return tuple(sl)


def periodic_bcs(dim):
    return [("P", "P")] * dim


def channel_bcs(dim=3, wall_axis=1, value=0.0):
    """bcs.py:74-83"""
    return [(("D", value), ("D", value)) if a == wall_axis else ("P", "P") for a in range(dim)]


def _kind(c):
    return c if isinstance(c, str) else c[0]


def _dval(c, comp):
    """bcs.py:34-39 (constant values only)"""
    v = c[1]
    return v if np.isscalar(v) else v[comp]


# --------------------------------------------------------------------------
# ghost fills  (fields.py:81-140)
# --------------------------------------------------------------------------

def fill_scalar(g, bcs, f):
    """fields.py:81-93"""
    d = g.dim
    for a, n in enumerate(g.shape):
        if _kind(bcs[a][0]) == "P":
            f[_plane(d, a, 0)] = f[_plane(d, a, n)]
            f[_plane(d, a, n + 1)] = f[_plane(d, a, 1)]
        else:
            f[_plane(d, a, 0)] = f[_plane(d, a, 1)]
            f[_plane(d, a, n + 1)] = f[_plane(d, a, n)]
    return f


def fill_velocity(g, bcs, u):
    """fields.py:96-140 (constant Dirichlet values)."""
    d = g.dim
    for a, n in enumerate(g.shape):
        lo, hi = bcs[a]
        for c in range(d):
            x = u[c]
            P = lambda i: _plane(d, a, i)  # noqa: E731
            if _kind(lo) == "P":
                x[P(0)] = x[P(n)]
                x[P(n + 1)] = x[P(1)]
                continue
            normal = c == a
            if _kind(lo) == "D":
                val = _dval(lo, c)
                x[P(0)] = val if normal else 2.0 * val - x[P(1)]
            elif _kind(lo) == "S":
                x[P(0)] = 0.0 if normal else x[P(1)]
            if _kind(hi) == "D":
                val = _dval(hi, c)
                if normal:
                    x[P(n)] = val
                    x[P(n + 1)] = 2.0 * val - x[P(n - 1)]
                else:
                    x[P(n + 1)] = 2.0 * val - x[P(n)]
            elif _kind(hi) == "S":
                if normal:
                    x[P(n)] = 0.0
                    x[P(n + 1)] = -x[P(n - 1)]
                else:
                    x[P(n + 1)] = x[P(n)]
    return u


# --------------------------------------------------------------------------
# forward stencils  (operators.py:108-301)
# --------------------------------------------------------------------------

def divergence(g, u):
    """operators.py:108-122"""
    out = g.zeros()
    p = g.pdof()
    for a in range(g.dim):
        t = np.subtract(u[a][p], u[a][_sh(p, a, -1)])
        t /= g.col(g.dx[a], a, p[a])
        out[p] += t
    return out


def pressure_gradient(g, pf):
    """operators.py:125-137"""
    out = g.zeros_vel()
    for a in range(g.dim):
        sl = g.udof(a)
        t = np.subtract(pf[_sh(sl, a, 1)], pf[sl])
        t /= g.col(g.du[a], a, sl[a])
        out[a][sl] = t
    return out


def diffusion(g, u, nu, out=None):
    """operators.py:140-170 (accumulates into ``out`` when given)."""
    if nu < 0:
        raise ValueError(f"viscosity must be nonnegative, got {nu}")
    if out is None:
        out = g.zeros_vel()
    for a in range(g.dim):
        sl = g.udof(a)
        ua = u[a]
        for b in range(g.dim):
            if a == b:
                khi, klo = g.col(g.own_hi[a], a, sl[a]), g.col(g.own_lo[a], a, sl[a])
            else:
                khi, klo = g.col(g.tan_hi[b], b, sl[b]), g.col(g.tan_lo[b], b, sl[b])
            up = np.subtract(ua[_sh(sl, b, 1)], ua[sl])
            up *= khi
            dn = np.subtract(ua[sl], ua[_sh(sl, b, -1)])
            dn *= klo
            up -= dn
            up *= nu
            out[a][sl] += up
    return out


def convection(g, u, out=None):
    """operators.py:173-215 (accumulates into ``out`` when given)."""
    if out is None:
        out = g.zeros_vel()
    for a in range(g.dim):
        sl = g.udof(a)
        ua = u[a]
        for b in range(g.dim):
            fp = np.add(ua[sl], ua[_sh(sl, b, 1)])
            fp *= 0.5
            fm = np.add(ua[_sh(sl, b, -1)], ua[sl])
            fm *= 0.5
            if a == b:
                np.multiply(fp, fp, out=fp)
                np.multiply(fm, fm, out=fm)
                width = g.col(g.du[a], a, sl[a])
            else:
                ub = u[b]
                wl = g.col(g.w_lo[a], a, sl[a])
                wh = g.col(g.w_hi[a], a, sl[a])
                lo_sl = _sh(sl, b, -1)
                cp = np.multiply(ub[sl], wl)
                cp += np.multiply(ub[_sh(sl, a, 1)], wh)
                fp *= cp
                cm = np.multiply(ub[lo_sl], wl)
                cm += np.multiply(ub[_sh(lo_sl, a, 1)], wh)
                fm *= cm
                width = g.col(g.dx[b], b, sl[b])
            fp -= fm
            fp /= width
            out[a][sl] -= fp
    return out


def momentum_rhs(g, u, nu, force=None, closure=None):
    """operators.py:218-238; ``force`` is a d-vector of constants
    (operators.py:241-259 casts them to the grid dtype) or of DOF-shaped
    arrays (a sampled callable, operators.py:249-258, operators.py:232-233); ``closure`` is a
    callable (g, u, out) that accumulates the eddy-stress term
    (operators.py:236-237, oracle/les_np.py)."""
    out = convection(g, u)
    if nu != 0.0:
        diffusion(g, u, nu, out=out)
    if force is not None:
        for a in range(g.dim):
            if np.ndim(force[a]) == 0:
                fa = g.dtype.type(force[a])
                if fa != 0.0:
                    out[a][g.udof(a)] += fa
            else:  # sampled per-DOF array (sample_force of a callable, operators.py:249-258)
                out[a][g.udof(a)] += force[a]
    if closure is not None:
        closure(g, u, out)
    return out


def velocity_weights(g):
    """operators.py:262-272"""
    res = []
    for a in range(g.dim):
        sl = g.udof(a)
        w = np.ones((1,) * g.dim, dtype=g.dtype)
        for ax in range(g.dim):
            w = w * g.col(g.du[ax] if ax == a else g.dx[ax], ax, sl[ax])
        res.append(np.ascontiguousarray(np.broadcast_to(w, tuple(s.stop - s.start for s in sl))))
    return res


def pressure_weights(g):
    """operators.py:275-281"""
    p = g.pdof()
    w = np.ones((1,) * g.dim, dtype=g.dtype)
    for ax in range(g.dim):
        w = w * g.col(g.dx[ax], ax, p[ax])
    return np.ascontiguousarray(np.broadcast_to(w, g.shape))


def kinetic_energy(g, u):
    """operators.py:284-291"""
    tot = 0.0
    for a, w in enumerate(velocity_weights(g)):
        x = u[a][g.udof(a)]
        tot += float(np.sum(w * x * x))
    return 0.5 * tot


def weighted_inner(g, u, v):
    """operators.py:294-301"""
    tot = 0.0
    for a, w in enumerate(velocity_weights(g)):
        sl = g.udof(a)
        tot += float(np.sum(w * u[a][sl] * v[a][sl]))
    return tot


# --------------------------------------------------------------------------
# pressure solves and projection  (poisson.py:167-200, 321-348)
# --------------------------------------------------------------------------

class SpectralSolve:
    """poisson.py:167-200: FFT diagonalisation on periodic uniform grids."""

    def __init__(self, g):
        if not all(g.periodic):
            raise ValueError("spectral pressure solver requires periodic axes")
        if not g.uniform:
            raise ValueError("spectral pressure solver requires uniform axes")
        self.g = g
        lam = np.zeros(g.shape)
        for a, n in enumerate(g.shape):
            h = float(g.widths[a][0])
            k = np.arange(n)
            sym = (2.0 * np.cos(2.0 * np.pi * k / n) - 2.0) / h**2
            shp = [1] * g.dim
            shp[a] = n
            lam = lam + sym.reshape(shp)
        half = list(g.shape)
        half[-1] = g.shape[-1] // 2 + 1
        lam = lam[tuple(slice(0, m) for m in half)].copy()
        lam[(0,) * g.dim] = 1.0
        self.lam = lam.astype(g.dtype)

    def __call__(self, rhs):
        mean = float(np.mean(rhs))
        rh = _rfftn(rhs - mean)
        rh /= self.lam
        rh[(0,) * self.g.dim] = 0.0
        return _irfftn(rh, s=self.g.shape)


def homogeneous_bcs(bcs):
    """poisson.py:31-40: Dirichlet values -> 0, other kinds unchanged."""
    return [tuple(("D", 0.0) if _kind(c) == "D" else c for c in side) for side in bcs]


def laplacian_apply(g, bcs, p_int):
    """poisson.py:43-68: scalar fill, gradient on the velocity DOFs,
    homogeneous velocity fill, divergence; interior in, interior out."""
    pf = g.zeros()
    pf[g.pdof()] = p_int
    fill_scalar(g, bcs, pf)
    vf = g.zeros_vel()
    for a in range(g.dim):
        sl = g.udof(a)
        t = np.subtract(pf[_sh(sl, a, 1)], pf[sl])
        t /= g.col(g.du[a], a, sl[a])
        vf[a][sl] = t
    fill_velocity(g, homogeneous_bcs(bcs), vf)
    return divergence(g, vf)[g.pdof()]


class CGSolve:
    """poisson.py:232-308: matrix-free CG on -W L, same update order,
    gauge fixing and stopping test; records iterations and the residual
    history."""

    def __init__(self, g, bcs, tol=None, max_iter=None):
        self.g, self.bcs = g, bcs
        self.w = pressure_weights(g)
        self.wtot = float(np.sum(self.w))
        self.tol = (1e-10 if g.dtype == np.float64 else 1e-5) if tol is None else float(tol)
        n_dof = int(np.prod(g.shape))
        self.max_iter = min(10000, 10 * int(np.ceil(n_dof ** (1.0 / g.dim))) + 10) if max_iter is None else max_iter
        self.iterations = 0
        self.residual_history = []

    def _wmean(self, a):
        return float(np.dot(self.w.ravel(), a.ravel()) / self.wtot)

    def __call__(self, rhs):
        w = self.w
        r = np.array(rhs, dtype=self.g.dtype)
        r -= self._wmean(r)
        r *= w
        np.negative(r, out=r)
        b_norm = float(np.linalg.norm(r.ravel()))
        self.residual_history = [b_norm]
        x = np.zeros(self.g.shape, dtype=self.g.dtype)
        self.iterations = 0
        if b_norm == 0.0:
            return x
        p = r.copy()
        rs = float(np.dot(r.ravel(), r.ravel()))
        for it in range(1, self.max_iter + 1):
            ap = laplacian_apply(self.g, self.bcs, p)
            ap *= w
            np.negative(ap, out=ap)
            denom = float(np.dot(p.ravel(), ap.ravel()))
            if denom <= 0.0:
                raise FloatingPointError("pressure operator lost positive definiteness")
            alpha = rs / denom
            x += p * alpha
            x -= self._wmean(x)
            ap *= alpha
            r -= ap
            r -= np.mean(r)
            res = float(np.linalg.norm(r.ravel()))
            self.residual_history.append(res)
            self.iterations = it
            if res <= self.tol * b_norm:
                return x
            rs_new = float(np.dot(r.ravel(), r.ravel()))
            beta = rs_new / rs
            rs = rs_new
            p *= beta
            p += r
        raise RuntimeError(f"pressure CG did not reach tol={self.tol} in {self.max_iter} iterations")


def project_into(g, bcs, solve, u):
    """poisson.py:321-341; returns the ghost-filled pressure."""
    fill_velocity(g, bcs, u)
    phi = divergence(g, u)
    p = g.zeros()
    p[g.pdof()] = solve(phi[g.pdof()])
    fill_scalar(g, bcs, p)
    for a in range(g.dim):
        sl = g.udof(a)
        t = np.subtract(p[_sh(sl, a, 1)], p[sl])
        t /= g.col(g.du[a], a, sl[a])
        u[a][sl] -= t
    fill_velocity(g, bcs, u)
    return p


# --------------------------------------------------------------------------
# time stepping  (timestep.py:21-337)
# --------------------------------------------------------------------------

class Tableau:
    """timestep.py:21-45 (explicit Butcher tableau, validated)."""

    def __init__(self, a, b, c):
        s = len(b)
        for i, row in enumerate(a):
            if any(row[j] != 0.0 for j in range(i, s)):
                raise ValueError("tableau must be strictly lower triangular")
            if abs(sum(row) - c[i]) > 1e-12:
                raise ValueError("c must be the row sums of a")
        if abs(sum(b) - 1.0) > 1e-12:
            raise ValueError("b must sum to one")
        self.a, self.b, self.c = tuple(map(tuple, a)), tuple(b), tuple(c)

    @property
    def stages(self):
        return len(self.b)


SSP33 = Tableau(((0.0, 0.0, 0.0), (1.0, 0.0, 0.0), (0.25, 0.25, 0.0)),
                (1.0 / 6.0, 1.0 / 6.0, 2.0 / 3.0), (0.0, 1.0, 0.5))        # timestep.py:48-52
WRAY3_GAMMA = (8.0 / 15.0, 5.0 / 12.0, 3.0 / 4.0)                           # timestep.py:56
WRAY3_ZETA = (0.0, -17.0 / 60.0, -5.0 / 12.0)                               # timestep.py:57
WRAY3 = Tableau(((0.0, 0.0, 0.0), (8.0 / 15.0, 0.0, 0.0), (0.25, 5.0 / 12.0, 0.0)),
                (0.25, 0.0, 0.75), (0.0, 8.0 / 15.0, 2.0 / 3.0))           # timestep.py:58-62
# classic RK4: not registered by the reference; injected through the generic
# rk_step (timestep.py:175) exactly as SURVEY.md section 0 describes.
RK4 = Tableau(((0.0, 0.0, 0.0, 0.0), (0.5, 0.0, 0.0, 0.0), (0.0, 0.5, 0.0, 0.0), (0.0, 0.0, 1.0, 0.0)),
              (1.0 / 6.0, 1.0 / 3.0, 1.0 / 3.0, 1.0 / 6.0), (0.0, 0.5, 0.5, 1.0))


def _axpy(g, dst, src, coef):
    """timestep.py:166-172"""
    for a in range(g.dim):
        sl = g.udof(a)
        dst[a][sl] += np.multiply(src[a][sl], coef)


def rk_step(g, bcs, solve, u0, dt, tab, nu, force=None, closure=None):
    """timestep.py:175-214; returns (u1, pressure).  ``u0`` must carry
    filled ghosts (the reference state always does)."""
    if dt <= 0:
        raise ValueError("time step must be positive")
    ks = []
    for j in range(tab.stages):
        if j == 0:
            y = u0
        else:
            y = [x.copy() for x in u0]
            for l in range(j):
                if tab.a[j][l] != 0.0:
                    _axpy(g, y, ks[l], dt * tab.a[j][l])
            project_into(g, bcs, solve, y)
        ks.append(momentum_rhs(g, y, nu, force, closure))
    acc = [x.copy() for x in u0]
    for l in range(tab.stages):
        if tab.b[l] != 0.0:
            _axpy(g, acc, ks[l], dt * tab.b[l])
    p = project_into(g, bcs, solve, acc)
    return acc, p


def wray3_step(g, bcs, solve, u, dt, nu, force=None):
    """timestep.py:217-250 (low-storage; updates ``u`` in place)."""
    fold = None
    p = None
    for i in range(3):
        fnew = momentum_rhs(g, u, nu, force)
        for a in range(g.dim):
            sl = g.udof(a)
            fnew[a][sl] *= dt * WRAY3_GAMMA[i]
            u[a][sl] += fnew[a][sl]
            if i > 0:
                fold[a][sl] *= WRAY3_ZETA[i] / WRAY3_GAMMA[i - 1]
                u[a][sl] += fold[a][sl]
        p = project_into(g, bcs, solve, u)
        fold = fnew
    return u, p


def cfl_dt(g, u, nu, c_conv, c_diff):
    """timestep.py:140-163"""
    if c_conv <= 0 or c_diff <= 0:
        raise ValueError("CFL safety factors must be positive")
    dt_conv = math.inf
    for a in range(g.dim):
        sl = g.udof(a)
        sp = np.abs(u[a][sl])
        wid = g.col(g.du[a], a, sl[a])
        with np.errstate(divide="ignore"):
            r = np.where(sp > 0, wid / sp, math.inf)
        dt_conv = min(dt_conv, float(np.min(r)))
    dt_diff = math.inf
    if nu > 0:
        h = min(float(np.min(w)) for w in g.widths)
        dt_diff = h * h / (2.0 * g.dim * nu)
    return min(c_conv * dt_conv, c_diff * dt_diff)


# --------------------------------------------------------------------------
# pullbacks  (adjoint.py:32-444), periodic boundaries
# --------------------------------------------------------------------------

def zero_ghosts_scalar(g, f):
    """adjoint.py:32-37"""
    for a, n in enumerate(g.shape):
        f[_plane(g.dim, a, 0)] = 0.0
        f[_plane(g.dim, a, n + 1)] = 0.0
    return f


def zero_non_dofs(g, v):
    """adjoint.py:40-50"""
    for c in range(g.dim):
        for a, n in enumerate(g.shape):
            v[c][_plane(g.dim, a, 0)] = 0.0
            v[c][_plane(g.dim, a, n + 1)] = 0.0
            if c == a and not g.periodic[a]:
                v[c][_plane(g.dim, a, n)] = 0.0
    return v


def fold_scalar(g, bcs, f):
    """adjoint.py:53-70"""
    d = g.dim
    for a in reversed(range(d)):
        n = g.shape[a]
        lo_g, hi_g = _plane(d, a, 0), _plane(d, a, n + 1)
        if _kind(bcs[a][0]) == "P":
            f[_plane(d, a, n)] += f[lo_g]
            f[_plane(d, a, 1)] += f[hi_g]
        else:
            f[_plane(d, a, 1)] += f[lo_g]
            f[_plane(d, a, n)] += f[hi_g]
        f[lo_g] = 0.0
        f[hi_g] = 0.0
    return f


def fold_velocity(g, bcs, v):
    """adjoint.py:73-111"""
    d = g.dim
    for a in reversed(range(d)):
        n = g.shape[a]
        lo, hi = bcs[a]
        lo_g, hi_g = _plane(d, a, 0), _plane(d, a, n + 1)
        for c in range(d):
            x = v[c]
            if _kind(lo) == "P":
                x[_plane(d, a, n)] += x[lo_g]
                x[_plane(d, a, 1)] += x[hi_g]
                x[lo_g] = 0.0
                x[hi_g] = 0.0
                continue
            normal = c == a
            if _kind(lo) == "D" and not normal:
                x[_plane(d, a, 1)] -= x[lo_g]
            elif _kind(lo) == "S" and not normal:
                x[_plane(d, a, 1)] += x[lo_g]
            x[lo_g] = 0.0
            if _kind(hi) in ("D", "S"):
                if normal:
                    x[_plane(d, a, n - 1)] -= x[hi_g]
                    x[_plane(d, a, n)] = 0.0
                elif _kind(hi) == "D":
                    x[_plane(d, a, n)] -= x[hi_g]
                else:
                    x[_plane(d, a, n)] += x[hi_g]
            x[hi_g] = 0.0
    return v


def divergence_pullback(g, bcs, pbar):
    """adjoint.py:114-128 (zeroes the ghosts of ``pbar`` in place)."""
    zero_ghosts_scalar(g, pbar)
    out = g.zeros_vel()
    p = g.pdof()
    for a in range(g.dim):
        t = pbar[p] / g.col(g.dx[a], a, p[a])
        out[a][p] += t
        out[a][_sh(p, a, -1)] -= t
    fold_velocity(g, bcs, out)
    return zero_non_dofs(g, out)


def pressure_gradient_pullback(g, bcs, vbar):
    """adjoint.py:131-145 (zeroes non-DOFs of ``vbar`` in place)."""
    zero_non_dofs(g, vbar)
    out = g.zeros()
    for a in range(g.dim):
        sl = g.udof(a)
        t = vbar[a][sl] / g.col(g.du[a], a, sl[a])
        out[_sh(sl, a, 1)] += t
        out[sl] -= t
    fold_scalar(g, bcs, out)
    return zero_ghosts_scalar(g, out)


def diffusion_pullback(g, bcs, vbar, nu):
    """adjoint.py:148-173"""
    zero_non_dofs(g, vbar)
    out = g.zeros_vel()
    for a in range(g.dim):
        sl = g.udof(a)
        for b in range(g.dim):
            if a == b:
                khi, klo = g.col(g.own_hi[a], a, sl[a]), g.col(g.own_lo[a], a, sl[a])
            else:
                khi, klo = g.col(g.tan_hi[b], b, sl[b]), g.col(g.tan_lo[b], b, sl[b])
            th = nu * vbar[a][sl] * khi
            tl = nu * vbar[a][sl] * klo
            out[a][_sh(sl, b, 1)] += th
            out[a][sl] -= th
            out[a][sl] -= tl
            out[a][_sh(sl, b, -1)] += tl
    fold_velocity(g, bcs, out)
    return zero_non_dofs(g, out)


def convection_pullback(g, bcs, vbar, u):
    """adjoint.py:176-227 (scatter form; refills the primal's ghosts)."""
    out = g.zeros_vel()
    zero_non_dofs(g, vbar)
    fill_velocity(g, bcs, u)
    for a in range(g.dim):
        sl = g.udof(a)
        ua = u[a]
        for b in range(g.dim):
            tp = 0.5 * (ua[sl] + ua[_sh(sl, b, 1)])
            tm = 0.5 * (ua[_sh(sl, b, -1)] + ua[sl])
            if a == b:
                gg = vbar[a][sl] / g.col(g.du[a], a, sl[a])
                gp, gm = gg * tp, gg * tm
                out[a][sl] -= gp
                out[a][_sh(sl, a, 1)] -= gp
                out[a][_sh(sl, a, -1)] += gm
                out[a][sl] += gm
            else:
                ub = u[b]
                wl = g.col(g.w_lo[a], a, sl[a])
                wh = g.col(g.w_hi[a], a, sl[a])
                sm = _sh(sl, b, -1)
                vp = wl * ub[sl] + wh * ub[_sh(sl, a, 1)]
                vm = wl * ub[sm] + wh * ub[_sh(sm, a, 1)]
                gg = vbar[a][sl] / g.col(g.dx[b], b, sl[b])
                h = 0.5 * gg * vp
                out[a][sl] -= h
                out[a][_sh(sl, b, 1)] -= h
                h = 0.5 * gg * vm
                out[a][sm] += h
                out[a][sl] += h
                r = gg * tp
                out[b][sl] -= wl * r
                out[b][_sh(sl, a, 1)] -= wh * r
                r = gg * tm
                out[b][sm] += wl * r
                out[b][_sh(sm, a, 1)] += wh * r
    fold_velocity(g, bcs, out)
    return zero_non_dofs(g, out)


def rhs_pullback(g, bcs, vbar, u, nu):
    """adjoint.py:253-261"""
    out = convection_pullback(g, bcs, vbar, u)
    if nu != 0.0:
        dif = diffusion_pullback(g, bcs, vbar, nu)
        for a in range(g.dim):
            out[a] += dif[a]
    return out


def poisson_solve_transpose(g, solve, pbar):
    """adjoint.py:236-250"""
    w = pressure_weights(g)
    out = g.zeros()
    out[g.pdof()] = solve(pbar[g.pdof()] / w) * w
    return out


def kinetic_energy_pullback(g, u):
    """adjoint.py:264-273"""
    out = g.zeros_vel()
    for a, w in enumerate(velocity_weights(g)):
        sl = g.udof(a)
        out[a][sl] = w * u[a][sl]
    return out


def project_pullback(g, bcs, solve, vbar):
    """adjoint.py:335-349"""
    zero_non_dofs(g, vbar)
    gbar = g.zeros_vel()
    for a in range(g.dim):
        gbar[a][g.udof(a)] = -vbar[a][g.udof(a)]
    pbar = pressure_gradient_pullback(g, bcs, gbar)
    sbar = poisson_solve_transpose(g, solve, pbar)
    dbar = divergence_pullback(g, bcs, sbar)
    out = g.zeros_vel()
    for a in range(g.dim):
        sl = g.udof(a)
        out[a][sl] = vbar[a][sl] + dbar[a][sl]
    return out


def project_with_tape(g, bcs, solve, u):
    """adjoint.py:319-332"""
    fill_velocity(g, bcs, u)
    p = g.zeros()
    p[g.pdof()] = solve(divergence(g, u)[g.pdof()])
    fill_scalar(g, bcs, p)
    gr = pressure_gradient(g, p)
    out = [x.copy() for x in u]
    for a in range(g.dim):
        sl = g.udof(a)
        out[a][sl] -= gr[a][sl]
    return fill_velocity(g, bcs, out)


def step_forward_tape(g, bcs, solve, u0, dt, tab, nu, force=None):
    """adjoint.py:352-384"""
    fill_velocity(g, bcs, u0)
    stages, ks = [], []
    for j in range(tab.stages):
        if j == 0:
            y = u0
        else:
            acc = [x.copy() for x in u0]
            for a in range(g.dim):
                sl = g.udof(a)
                for l in range(j):
                    if tab.a[j][l] != 0.0:
                        acc[a][sl] += (dt * tab.a[j][l]) * ks[l][a][sl]
            y = project_with_tape(g, bcs, solve, acc)
        stages.append(y)
        ks.append(momentum_rhs(g, y, nu, force))  # the tape excludes closures (adjoint.py:374)
    acc = [x.copy() for x in u0]
    for a in range(g.dim):
        sl = g.udof(a)
        for l in range(tab.stages):
            if tab.b[l] != 0.0:
                acc[a][sl] += (dt * tab.b[l]) * ks[l][a][sl]
    return project_with_tape(g, bcs, solve, acc), (stages, dt, tab)


def step_backward(g, bcs, solve, tape, ubar, nu):
    """adjoint.py:387-422"""
    stages, dt, tab = tape
    s = tab.stages
    ybar = project_pullback(g, bcs, solve, ubar)
    g0 = [x.copy() for x in ybar]
    kbars = [None] * s
    for l in range(s):
        if tab.b[l] != 0.0:
            kb = g.zeros_vel()
            for a in range(g.dim):
                sl = g.udof(a)
                kb[a][sl] = (dt * tab.b[l]) * ybar[a][sl]
            kbars[l] = kb
    for j in reversed(range(s)):
        if kbars[j] is None:
            continue
        fb = rhs_pullback(g, bcs, kbars[j], stages[j], nu)
        if j == 0:
            for a in range(g.dim):
                sl = g.udof(a)
                g0[a][sl] += fb[a][sl]
            continue
        yb = project_pullback(g, bcs, solve, fb)
        for a in range(g.dim):
            sl = g.udof(a)
            g0[a][sl] += yb[a][sl]
            for l in range(j):
                if tab.a[j][l] != 0.0:
                    if kbars[l] is None:
                        kbars[l] = g.zeros_vel()
                    kbars[l][a][sl] += (dt * tab.a[j][l]) * yb[a][sl]
    return g0


def unrolled_gradient_ke(g, bcs, solve, u0, n_steps, dt, tab, nu, force=None):
    """adjoint.py:425-444 with ``KineticEnergyLoss`` (adjoint.py:276-285)."""
    if not all(g.periodic):
        raise ValueError("periodic boundaries only")
    u = [x.copy() for x in u0]
    tapes = []
    for _ in range(n_steps):
        u, tape = step_forward_tape(g, bcs, solve, u, dt, tab, nu, force)
        tapes.append(tape)
    ubar = kinetic_energy_pullback(g, u)
    for tape in reversed(tapes):
        ubar = step_backward(g, bcs, solve, tape, ubar, nu)
    return zero_non_dofs(g, ubar)
