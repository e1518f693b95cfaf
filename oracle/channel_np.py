"""Channel pressure solve restated as FFT(x,z) x tridiagonal(y)
(TEST INFRASTRUCTURE ONLY).

The reference solves the channel pressure with ``DirectPoissonSolver``
(``poisson.py:203-229``): the volume-weighted operator W*D(G p) of
``_LaplacianApply`` (``poisson.py:43-68``, homogeneous wall conditions from
``poisson.py:31-40``) bordered by the weight vector, i.e.

    L p + mu = rhs,   sum(W p) = 0     =>   mu = wmean(rhs).

On a grid that is periodic and uniform in x (axis 0) and z (axis 2) with
walls on y (axis 1) that operator separates exactly: Fourier modes in x/z
times a per-mode tridiagonal along y with

    up_j = 1/(du[j] dx[j])   (j < n),   lo_j = 1/(du[j-1] dx[j])   (j > 1),
    di_j = -(up_j + lo_j) + lam_x(kx) + lam_z(kz),

and the singular (0,0) mode is closed by the weighted gauge
sum_j dx[j] q_j = 0 (the bordered system restricted to that mode).
``tests/test_oracle_golden.py`` pins this against the reference's direct
solver output stored in the golden fixtures.
"""

import numpy as np


class ChannelSolve:
    def __init__(self, g, wall_axis=1):
        if g.dim != 3 or wall_axis != 1:
            raise ValueError("channel solve needs a 3D grid with walls on axis 1")
        if not (g.periodic[0] and g.periodic[2] and not g.periodic[1]):
            raise ValueError("channel solve needs periodic x/z and walls on y")
        for a in (0, 2):
            w = g.widths[a]
            if not np.allclose(w, w[0], rtol=1e-12, atol=0.0):
                raise ValueError("channel solve needs uniform x/z")
        self.g = g
        n0, n1, n2 = g.shape
        dx = g.dx[1].astype(np.float64)
        du = g.du[1].astype(np.float64)
        up = np.zeros(n1 + 2)
        lo = np.zeros(n1 + 2)
        j = np.arange(1, n1 + 1)
        up[1:n1] = 1.0 / (du[1:n1] * dx[1:n1])
        lo[2:n1 + 1] = 1.0 / (du[1:n1] * dx[2:n1 + 1])
        self.up, self.lo = up, lo
        self.di = -(up + lo)
        self.dxy = dx[j]
        lam = []
        for a, m in ((0, n0), (2, n2)):
            h = float(g.widths[a][0])
            k = np.arange(m)
            lam.append((2.0 * np.cos(2.0 * np.pi * k / m) - 2.0) / h**2)
        self.lam_x = lam[0]
        self.lam_z = lam[1][: n2 // 2 + 1]
        w = np.ones((1, 1, 1))
        for a in range(3):
            shp = [1, 1, 1]
            shp[a] = g.shape[a]
            w = w * g.dx[a][1:g.shape[a] + 1].astype(np.float64).reshape(shp)
        self.w = np.broadcast_to(w, g.shape)
        self.wtot = float(np.sum(self.w))

    def __call__(self, rhs):
        g = self.g
        n0, n1, n2 = g.shape
        r = np.asarray(rhs, dtype=np.float64)
        r = r - float(np.sum(self.w * r)) / self.wtot
        rh = np.fft.fft(np.fft.rfft(r, axis=2), axis=0)  # (n0, n1, n2//2+1)
        shift = self.lam_x[:, None] + self.lam_z[None, :]  # (n0, nkz)
        # batched Thomas along axis 1 for every (kx, kz) except (0, 0)
        up, lo, di = self.up, self.lo, self.di
        cprime = np.zeros((n0, n1, shift.shape[1]))
        d = np.zeros_like(rh)
        piv = di[1] + shift
        piv[0, 0] = 1.0
        cprime[:, 0] = up[1] / piv
        d[:, 0] = rh[:, 0] / piv
        # the (0, 0) column of the sweep is singular and overflows harmlessly:
        # that mode is replaced by the bordered solve below
        err = np.seterr(over="ignore", invalid="ignore")
        for jj in range(1, n1):
            jext = jj + 1
            piv = di[jext] + shift - lo[jext] * cprime[:, jj - 1]
            piv[0, 0] = 1.0
            cprime[:, jj] = up[jext] / piv
            d[:, jj] = (rh[:, jj] - lo[jext] * d[:, jj - 1]) / piv
        x = np.zeros_like(rh)
        x[:, n1 - 1] = d[:, n1 - 1]
        for jj in range(n1 - 2, -1, -1):
            x[:, jj] = d[:, jj] - cprime[:, jj] * x[:, jj + 1]
        np.seterr(**err)
        # (0, 0): bordered system [[L_y, 1], [dx^T, 0]]
        a_mat = np.zeros((n1 + 1, n1 + 1))
        for jj in range(n1):
            jext = jj + 1
            a_mat[jj, jj] = di[jext]
            if jj + 1 < n1:
                a_mat[jj, jj + 1] = up[jext]
            if jj > 0:
                a_mat[jj, jj - 1] = lo[jext]
            a_mat[jj, n1] = 1.0
        a_mat[n1, :n1] = self.dxy
        b = np.zeros(n1 + 1, dtype=complex)
        b[:n1] = rh[0, :, 0]
        x[0, :, 0] = np.linalg.solve(a_mat, b)[:n1]
        out = np.fft.irfft(np.fft.ifft(x, axis=0), n=n2, axis=2)
        return out.astype(g.dtype)
