"""Test-only numpy backend for the slab-decomposed RK4 path
(paper_2604_18536_b200/distributed.py), so the multi-rank orchestration can be
exercised with gloo on CPU.  Local compute follows the oracle restatement of
the reference (oracle/stagflow_np.py); uniform periodic grids only."""

import numpy as np
import torch

from oracle import stagflow_np as O


class CpuField:
    def __init__(self, shape, dtype, dim=3):
        self.u = [torch.zeros(shape, dtype=dtype) for _ in range(dim)]


class CpuScalar:
    def __init__(self, shape, dtype):
        self.data = torch.zeros(shape, dtype=dtype)


class CpuSlabBackend:
    def __init__(self, global_bounds, layout, nu, force):
        self.lay = layout
        m, i0 = layout.m, layout.i0
        b0 = global_bounds[0][i0:i0 + m + 1]
        self.og = O.OGrid([b0, global_bounds[1], global_bounds[2]], (True, True, True))
        self.n0 = len(global_bounds[0]) - 1
        self.n1 = len(global_bounds[1]) - 1
        self.n2 = len(global_bounds[2]) - 1
        self.nu = nu
        self.force = force
        nh = self.n2 // 2 + 1
        P = layout.size
        self.spec = torch.zeros((m, self.n1, nh, 2), dtype=torch.float64)
        # one rank: the axis-0 pass works on the spectrum itself (no exchange)
        self.trans = torch.zeros((self.n0, self.n1 // P, nh, 2), dtype=torch.float64) if P > 1 else self.spec
        self.xchg = torch.zeros((P, m, self.n1 // P, nh, 2), dtype=torch.float64) if P > 1 else None
        self.p_slab = torch.zeros((m + 3, self.n1, self.n2), dtype=torch.float64)
        self.p_local = self.p_slab[1:m + 1]
        self.p_halo = self.p_slab[m + 1]
        lam = []
        for bnd, n in ((global_bounds[0], self.n0), (global_bounds[1], self.n1), (global_bounds[2], self.n2)):
            h = float(np.diff(bnd)[0])
            k = np.arange(n)
            lam.append((2.0 * np.cos(2.0 * np.pi * k / n) - 2.0) / h**2)
        self.lam = lam
        self.ext = self.og.ext_shape

    # -- fields
    def new_field(self):
        return CpuField(self.ext, torch.float64)

    def new_scalar(self):
        return CpuScalar(self.ext, torch.float64)

    def _np(self, f):
        return [t.numpy() for t in f.u]

    def _fill12(self, arrs):
        """periodic ghost fill of axes 1 and 2 (axis 0 ghosts come from the halo)."""
        for x in arrs:
            for a in (1, 2):
                n = x.shape[a] - 2
                sl = [slice(None)] * 3
                s2 = [slice(None)] * 3
                sl[a], s2[a] = 0, n
                x[tuple(sl)] = x[tuple(s2)]
                sl[a], s2[a] = n + 1, 1
                x[tuple(sl)] = x[tuple(s2)]

    # -- compute
    def _project_copy(self, y, p_slab):
        """y - G p on every plane the stencil reads (ghost planes included),
        from the slab pressure with the neighbours' planes."""
        og = self.og
        m = self.lay.m
        ys = [x.copy() for x in self._np(y)]
        self._fill12(ys)
        pe = np.zeros((m + 3,) + og.ext_shape[1:])
        pe[:, 1:-1, 1:-1] = p_slab.numpy()
        self._fill12([pe[:m + 2]])
        pe[m + 2, 1:-1, 1:-1] = p_slab.numpy()[m + 2]
        self._fill12([pe[m + 1:m + 3]])
        n1, n2 = self.n1, self.n2
        for a in range(3):
            sl = (slice(0, m + 2), slice(0, n1 + 2), slice(0, n2 + 2))
            hi = list(sl)
            if a == 0:
                hi[0] = slice(1, m + 3)
                pn = pe[tuple(hi)]
            else:
                # periodic wrap along axes 1, 2 for the +1 neighbour of the last ghost
                idx = np.arange(1, (n1 if a == 1 else n2) + 3)
                nn = n1 if a == 1 else n2
                idx = np.where(idx > nn + 1, idx - nn, idx)
                pn = np.take(pe[:m + 2], idx, axis=a)
            g = (pn - pe[:m + 2]) / og.col(og.du[a], a, slice(0, og.ext_shape[a]))
            ys[a] -= g
        return ys

    def stage(self, y, u0=None, s_in=None, s_out=None, y_next=None, cb=0.0, ca=0.0, p_slab=None, u0_out=None):
        og = self.og
        yv = self._np(y) if p_slab is None else self._project_copy(y, p_slab)
        k = O.momentum_rhs(og, yv, self.nu, self.force)
        for a in range(3):
            sl = og.udof(a)
            # u0_out (u0 is y, deferred projection): the combines use projected y
            u0v = yv[a] if u0_out is not None else (u0.u[a].numpy() if u0 is not None else None)
            if u0_out is not None:
                u0_out.u[a].numpy()[sl] = yv[a][sl]
            if s_out is not None:
                base = s_in.u[a].numpy() if s_in is not None else u0v
                s_out.u[a].numpy()[sl] = base[sl] + k[a][sl] * cb
            if y_next is not None:
                y_next.u[a].numpy()[sl] = u0v[sl] + k[a][sl] * ca

    # -- spectral solve in column chunks (the CUDA backend's interface)
    def max_chunks(self):
        return self.n2 // 2 + 1

    def _chunk(self, k, K):
        nh = self.n2 // 2 + 1
        base = (nh + K - 1) // K
        c0 = k * base
        return c0, min(base, nh - c0)

    def _blocks(self, k, K):
        """xchg block k as (P, m, c, w) and trans block k as (n0, c, w), complex."""
        P, m = self.lay.size, self.lay.m
        c = self.n1 // P
        c0, w = self._chunk(k, K)
        off, n = 2 * P * m * c * c0, 2 * P * m * c * w
        xb = self.xchg.reshape(-1)[off:off + n].view(P, m, c, w, 2)
        tb = self.trans.reshape(-1)[off:off + n].view(self.n0, c, w, 2)
        return xb, tb, c0, w

    def r2c(self, u):
        arrs = self._np(u)
        self._fill12(arrs)
        div = O.divergence(self.og, arrs)[self.og.pdof()]
        self.spec.copy_(torch.view_as_real(torch.from_numpy(np.fft.rfft(div, axis=2))))

    def axis1(self, k, K, inverse=False):
        s = torch.view_as_complex(self.spec).numpy()
        if self.xchg is None:
            s[...] = np.fft.ifft(s, axis=1) if inverse else np.fft.fft(s, axis=1)
            return
        P, m = self.lay.size, self.lay.m
        c = self.n1 // P
        xb, _, c0, w = self._blocks(k, K)
        if w <= 0:
            return
        if inverse:
            blk = torch.view_as_complex(xb.contiguous()).numpy()  # (P, m, c, w)
            nat = blk.transpose(1, 0, 2, 3).reshape(m, self.n1, w)
            s[:, :, c0:c0 + w] = np.fft.ifft(nat, axis=1)
        else:
            f = np.fft.fft(s[:, :, c0:c0 + w], axis=1).reshape(m, P, c, w).transpose(1, 0, 2, 3)
            xb.copy_(torch.view_as_real(torch.from_numpy(np.ascontiguousarray(f))))

    def axis0(self, k=0, K=1):
        P, q = self.lay.size, self.lay.rank
        c = self.n1 // P
        nh = self.n2 // 2 + 1
        if self.xchg is None:
            tb, c0, w = self.trans, 0, nh
        else:
            _, tb, c0, w = self._blocks(k, K)
            if w <= 0:
                return
        t = torch.view_as_complex(tb.contiguous()).numpy()
        f = np.fft.fft(t, axis=0)
        k1 = np.arange(q * c, (q + 1) * c)
        lam = (self.lam[0][:, None, None] + self.lam[1][k1][None, :, None]) + self.lam[2][c0:c0 + w][None, None, :]
        zero = q == 0 and c0 == 0
        if zero:
            lam[0, 0, 0] = 1.0
        f = f / lam
        if zero:
            f[0, 0, 0] = 0.0
        tb.copy_(torch.view_as_real(torch.from_numpy(np.fft.ifft(f, axis=0))))

    def c2r(self):
        s = torch.view_as_complex(self.spec).numpy()
        p = np.fft.irfft(s, n=self.n2, axis=2)
        self.p_local.copy_(torch.from_numpy(np.ascontiguousarray(p)))

    def correct(self, u, p_ext=None):
        og = self.og
        m = self.lay.m
        pe = np.zeros(og.ext_shape)
        pe[1:m + 1, 1:-1, 1:-1] = self.p_local.numpy()
        pe[m + 1, 1:-1, 1:-1] = self.p_halo.numpy()
        self._fill12([pe])
        arrs = self._np(u)
        for a in range(3):
            sl = og.udof(a)
            t = np.subtract(pe[O._sh(sl, a, 1)], pe[sl])
            t /= og.col(og.du[a], a, sl[a])
            arrs[a][sl] -= t
        self._fill12(arrs)
        if p_ext is not None:
            p_ext.data.numpy()[1:] = pe[1:]

    def kinetic_energy_local(self, u):
        return O.kinetic_energy(self.og, self._np(u))
