"""Pressure Poisson solvers and the projection on the GPU
(mirror of poisson.py:1-348).

Backends (same duck-typed interface as the reference: ``kind``,
``tolerance``, ``iterations``, ``grid``, ``bcs``, ``weights``, ``wtot``,
``solve(ScalarField)``, ``solve_interior(rhs, out)``):

* ``spectral``   -- cuFFT D2Z/Z2D + hand-written eigenvalue scaling;
  periodic uniform grids only (poisson.py:167-200).
* ``fft-tridiag`` -- channel grids (periodic uniform x/z, walls on y, any
  y stretching): batched 2D FFT over x/z + per-mode Thomas along y with the
  weighted zero-mean gauge.  It solves exactly the system of the reference's
  ``DirectPoissonSolver`` (poisson.py:203-229), so ``make_solver("direct")``
  returns it on such grids.
* ``cg``         -- matrix-free conjugate gradient on the weighted operator
  (poisson.py:232-308; csrc/cg.cu): any boundary conditions and stretching,
  the reference's defaults, ``residual_history`` and ``ConvergenceError``.
"""

import ctypes

import numpy as np
import torch

from . import _native as N
from .bcs import BoundarySpec, Dirichlet
from .errors import ConfigurationError, ConvergenceError
from .fields import ScalarField
from .operators import pressure_weights
from .plan import get_plan, set_time, stream_ptr


def homogeneous(bcs):
    """poisson.py:31-40"""
    return BoundarySpec([
        tuple(Dirichlet(0.0) if isinstance(c, Dirichlet) else c for c in side) for side in bcs.sides
    ])


class _GpuSolver:
    kind = "base"
    tolerance = 1e-12
    _native_kind = None

    def __init__(self, grid, bcs):
        self.grid = grid
        self.bcs = bcs
        self.weights = pressure_weights(grid)
        self.wtot = float(np.sum(self.weights))
        self.iterations = 0
        self.plan = get_plan(grid, bcs)
        h = ctypes.c_void_p()
        N.call("sfb_solver_create", self.plan.handle, self._native_kind, ctypes.byref(h))
        self.handle = h
        self._buf = None

    def __del__(self):
        h = getattr(self, "handle", None)
        if h is not None and h.value:
            try:
                N.lib.sfb_solver_destroy(h)
            except Exception:  # pragma: no cover
                pass

    def solve(self, rhs):
        out = ScalarField(self.grid)
        self.solve_interior(rhs.interior, out.interior)
        return out

    def solve_interior(self, rhs, out):
        """rhs/out: interior views (any strides) of shape grid.shape."""
        if self._buf is None:
            self._buf = torch.empty(self.grid.shape, dtype=out.dtype, device=out.device)
        buf = self._buf
        buf.copy_(rhs)
        N.call("sfb_solver_solve", self.handle, buf.data_ptr(), buf.data_ptr(), stream_ptr())
        out.copy_(buf)
        self.iterations = 1


class SpectralPoissonSolver(_GpuSolver):
    """FFT diagonalization; requires all axes periodic and uniform."""

    kind = "spectral"
    _native_kind = N.SFB_SOLVER_SPECTRAL

    def __init__(self, grid, bcs):
        if not all(grid.periodic):
            raise ConfigurationError("spectral pressure solver requires periodic axes")
        if not grid.uniform:
            raise ConfigurationError("spectral pressure solver requires uniform axes")
        super().__init__(grid, bcs)


def _separable_channel(grid):
    if grid.dim != 3 or grid.periodic != (True, False, True):
        return False
    return all(np.allclose(grid.axes[a].widths, grid.axes[a].widths[0], rtol=1e-12, atol=0.0) for a in (0, 2))


class ChannelPoissonSolver(_GpuSolver):
    """FFT(x,z) x batched tridiagonal(y) solve of the weighted channel
    operator with the weighted zero-mean gauge (exact replacement of the
    reference's augmented direct solve, poisson.py:203-229)."""

    kind = "fft-tridiag"
    _native_kind = N.SFB_SOLVER_CHANNEL

    def __init__(self, grid, bcs):
        if not _separable_channel(grid):
            raise ConfigurationError(
                "fft-tridiag pressure solver requires periodic uniform x/z and walls on y (3D)"
            )
        super().__init__(grid, bcs)


class CGPoissonSolver(_GpuSolver):
    """Matrix-free conjugate gradient on the weighted operator
    (poisson.py:232-308): b = -W (rhs - wmean), CG on -W L with the weighted
    mean of the iterate and the mean of the residual removed every step,
    stop at |r| <= tol |b|."""

    kind = "cg"
    _native_kind = N.SFB_SOLVER_CG

    def __init__(self, grid, bcs, tol=None, max_iter=None):
        if tol is None:
            tol = 1e-10 if np.dtype(grid.dtype) == np.float64 else 1e-5
        if tol <= 0:
            raise ValueError(f"tolerance must be positive, got {tol}")
        n_dof = int(np.prod(grid.shape))
        if max_iter is None:
            max_iter = min(10000, 10 * int(np.ceil(n_dof ** (1.0 / grid.dim))) + 10)
        super().__init__(grid, bcs)
        self.tol = float(tol)
        self.max_iter = int(max_iter)
        N.call("sfb_cg_configure", self.handle, self.tol, self.max_iter)
        self.residual_history = []

    @property
    def tolerance(self):
        return self.tol

    def _after_solve(self, failed=None):
        """Pull the iteration count and residual history of the last solve;
        attach them to a ConvergenceError."""
        it = ctypes.c_int()
        cnt = ctypes.c_int()
        N.call("sfb_cg_info", self.handle, ctypes.byref(it), None, 0, ctypes.byref(cnt))
        hist = (ctypes.c_double * max(cnt.value, 1))()
        N.call("sfb_cg_info", self.handle, ctypes.byref(it), hist, cnt.value, ctypes.byref(cnt))
        self.residual_history = list(hist[: cnt.value])
        self.iterations = it.value if failed is None else self.max_iter
        if failed is not None:
            b = self.residual_history[0] if self.residual_history else 1.0
            failed.residual = self.residual_history[-1] / b if b else None
            failed.iterations = self.max_iter

    def solve_interior(self, rhs, out):
        try:
            super().solve_interior(rhs, out)
        except ConvergenceError as e:
            self._after_solve(failed=e)
            raise
        self._after_solve()


def _periodic_uniform(grid):
    return all(grid.periodic) and grid.uniform


class DirectPoissonSolver(_GpuSolver):
    """``solver="direct"`` (poisson.py:203-229): the augmented system
    [[W L, w], [w^T, 0]] -- L p = rhs - wmean with the weighted zero-mean
    gauge w^T p = 0 -- on any grid, as the reference's sparse LU is.  The GPU
    path picks the exact solver for the layout:

    * separable channel (periodic uniform x/z, walls on y, 3D): FFT(x,z) x
      batched tridiagonal(y), exact (``backend == "fft-tridiag"``);
    * all-periodic uniform grids: the spectral solve -- on uniform grids W is
      constant, so rhs - wmean is rhs - mean and w^T p = 0 is the zero-mean
      gauge of the FFT diagonalisation (``backend == "spectral"``);
    * anything else (stretching along a periodic axis, walls on other axes,
      symmetric sides, 2D channels): the matrix-free CG on the same weighted
      operator and gauge, run to a relative residual of 1e-12 (fp64) /
      1e-6 (fp32) with up to 10000 iterations (``backend == "cg"``); a solve
      that does not get there raises ConvergenceError instead of returning a
      less accurate pressure.
    """

    kind = "direct"
    tolerance = 1e-12

    def __init__(self, grid, bcs):
        if _separable_channel(grid):
            self.backend, self._native_kind = "fft-tridiag", N.SFB_SOLVER_CHANNEL
        elif _periodic_uniform(grid):
            self.backend, self._native_kind = "spectral", N.SFB_SOLVER_SPECTRAL
        else:
            self.backend, self._native_kind = "cg", N.SFB_SOLVER_CG
        super().__init__(grid, bcs)
        if self.backend == "cg":
            self.tol = 1e-12 if np.dtype(grid.dtype) == np.float64 else 1e-6
            self.max_iter = 10000
            N.call("sfb_cg_configure", self.handle, self.tol, self.max_iter)
            self.residual_history = []

    def _after_solve(self, failed=None):
        if self.backend == "cg":
            CGPoissonSolver._after_solve(self, failed)
        else:
            self.iterations = 1

    def solve_interior(self, rhs, out):
        try:
            super().solve_interior(rhs, out)
        except ConvergenceError as e:
            self._after_solve(failed=e)
            raise
        self._after_solve()


def make_solver(kind, grid, bcs, tol=None, max_iter=None):
    """poisson.py:311-318"""
    if kind == "spectral":
        return SpectralPoissonSolver(grid, bcs)
    if kind == "direct":
        return DirectPoissonSolver(grid, bcs)
    if kind == "fft-tridiag":
        return ChannelPoissonSolver(grid, bcs)
    if kind == "cg":
        return CGPoissonSolver(grid, bcs, tol=tol, max_iter=max_iter)
    raise ConfigurationError(f"unknown pressure solver kind: {kind!r}")


def _native_solver(solver, bcs):
    if not isinstance(solver, _GpuSolver):
        raise ConfigurationError("project_into needs a GPU pressure solver from make_solver()")
    if bcs is not solver.bcs:
        from .plan import bcs_signature

        if bcs_signature(bcs) != bcs_signature(solver.bcs):
            raise ConfigurationError("projection boundary conditions differ from the solver's")
    return solver


def project_into(u, solver, bcs, t=0.0, scratch=None, p_div=None, p_out=None):
    """poisson.py:321-341: make ``u`` discretely divergence-free in place
    (one fused native call); returns the ghost-filled pressure."""
    set_time(u.grid, bcs, t)  # callable (moving) Dirichlet walls at the fill time
    s = _native_solver(solver, bcs)
    if p_out is None:
        p_out = ScalarField(u.grid)
    call_solver(s, "sfb_project", s.handle, N.ptr3(u.u), p_out.data.data_ptr(), stream_ptr())
    return p_out


def call_solver(s, name, *args):
    """One native call that runs the solver; keeps the solver's iteration
    bookkeeping (and a ConvergenceError's residual) up to date."""
    after = getattr(s, "_after_solve", None)
    try:
        N.call(name, *args)
    except ConvergenceError as e:
        if after is not None:
            after(failed=e)
        raise
    if after is not None:
        after()
    else:
        s.iterations = 1


def project(u, solver, bcs, t=0.0):
    """poisson.py:344-348"""
    v = u.copy()
    p = project_into(v, solver, bcs, t=t)
    return v, p
