"""Eddy-viscosity closures on the GPU (mirror of les.py:58-434).

``ClosureModel(kind, c, filter_rule, p)`` keeps the reference's interface
(``kind``, ``c``, ``filter_rule``, ``p``, ``KINDS``, ``nu_t(u)``,
``add_rhs(u, out, scratch)``); ``nu_t`` and ``eddy_stress_divergence`` are one
kernel each (csrc/les.cu).  The models' constants are the reference's
``MODEL_CONSTANTS``.
"""

import ctypes

import numpy as np

from . import _native as N
from .bcs import BoundarySpec
from .errors import ConfigurationError
from .fields import ScalarField, VelocityField
from .operators import _plan
from .plan import stream_ptr

MODEL_CONSTANTS = {
    "smagorinsky": 0.17,
    "vreman": float(np.sqrt(2.5 * 0.17 ** 2)),
    "qr": float(np.sqrt(1.5) / np.pi),
    "wale": float(np.sqrt(2.5 * 0.17)),
    "sigma": 1.35,
    "s3pqr": 0.762,
}

_KIND_CODE = {"smagorinsky": 1, "vreman": 2, "qr": 3, "wale": 4, "sigma": 5, "s3pqr": 6}


def filter_width(grid, rule="geometric"):
    """les.py:297-305: local filter width (prod of the cell widths)^(1/d) at the
    pressure points (host array; the kernels form it per cell)."""
    if rule != "geometric":
        raise ConfigurationError(f"unknown filter width rule: {rule!r}")
    prod = np.ones((1,) * grid.dim, dtype=grid.dtype)
    for a in range(grid.dim):
        w = np.asarray(grid.axes[a].widths, dtype=grid.dtype)
        shp = [1] * grid.dim
        shp[a] = w.size
        prod = prod * w.reshape(shp)
    return np.ascontiguousarray(np.broadcast_to(prod, grid.shape)) ** (1.0 / grid.dim)


def axis_widths(grid):
    """les.py:308-318: per-axis local widths at the pressure points."""
    out = []
    for a in range(grid.dim):
        w = np.asarray(grid.axes[a].widths, dtype=grid.dtype)
        shp = [1] * grid.dim
        shp[a] = w.size
        out.append(np.ascontiguousarray(np.broadcast_to(w.reshape(shp), grid.shape)))
    return out


class ClosureModel:
    """les.py:332-383: eddy-viscosity closure (kind, constant, filter rule,
    s3pqr exponent)."""

    KINDS = ("none", "smagorinsky", "vreman", "qr", "wale", "sigma", "s3pqr")

    def __init__(self, kind="none", c=None, filter_rule="geometric", p=-2.5):
        if kind not in self.KINDS:
            raise ConfigurationError(f"unknown closure kind: {kind!r}")
        self.kind = kind
        self.c = float(MODEL_CONSTANTS.get(kind, 0.0) if c is None else c)
        if self.c < 0:
            raise ValueError("closure constant must be nonnegative")
        self.filter_rule = filter_rule
        self.p = float(p)

    def nu_t(self, u):
        """Eddy viscosity at the pressure points from the current velocity
        (filled ghosts); ghosts of the result are zero, as in the reference."""
        grid = u.grid
        out = ScalarField(grid)
        if self.kind == "none":
            return out
        if self.filter_rule != "geometric":
            raise ConfigurationError(f"unknown filter width rule: {self.filter_rule!r}")
        N.call("sfb_closure_nut", _plan(grid), _KIND_CODE[self.kind], self.c, self.p, N.ptr3(u.u),
               out.data.data_ptr(), stream_ptr())
        return out

    def nu_t_into(self, u, out):
        """nu_t into an existing scalar field (no allocation)."""
        if self.filter_rule != "geometric":
            raise ConfigurationError(f"unknown filter width rule: {self.filter_rule!r}")
        N.call("sfb_closure_nut", _plan(u.grid), _KIND_CODE[self.kind], self.c, self.p, N.ptr3(u.u),
               out.data.data_ptr(), stream_ptr())
        return out

    def rhs_into(self, u, out, nut):
        """The closure's RHS term alone (out = div 2 nu_t S on the DOFs),
        with nu_t in the caller's buffer: the fused stage adds it after the
        force, like add_rhs does onto the assembled RHS."""
        self.nu_t_into(u, nut)
        _eddy(u, nut, out, accumulate=False)

    def add_rhs(self, u, out, scratch=None):
        if self.kind == "none":
            return
        nut = self.nu_t(u)
        _eddy(u, nut, out, accumulate=True)


def active(closure):
    return closure is not None and getattr(closure, "kind", "none") != "none"


def _eddy(u, nut, out, accumulate):
    grid = u.grid
    plan = _plan(grid)
    N.call("sfb_fill_ghosts_scalar", plan, nut.data.data_ptr(), stream_ptr())
    N.call("sfb_eddy_stress_divergence", plan, N.ptr3(u.u), nut.data.data_ptr(), N.ptr3(out.u),
           1 if accumulate else 0, stream_ptr())


def closure_pullback(closure, u, vbar, out=None, accumulate=False):
    """VJP of the closure's RHS term u -> div(2 nu_t(u) S(u)) at ``u``:
    (dE/du)^T vbar, nu_t's dependence on u included (Smagorinsky; periodic
    3D).  Fills the ghosts of ``u`` and ``vbar`` (periodic images).  The
    reference has no closure adjoint (its tape omits closures,
    adjoint.py:374); this is the training extension of SURVEY 8(f2)."""
    import torch

    from .fields import fill_ghosts_velocity

    if closure.kind != "smagorinsky":
        raise ConfigurationError("closure pullback: Smagorinsky only")
    grid = u.grid
    if out is None:
        out = VelocityField(grid)
    elif not accumulate:
        for c in out.u:
            c.zero_()
    bcs = BoundarySpec.all_periodic(grid.dim)
    fill_ghosts_velocity(u, bcs)
    fill_ghosts_velocity(vbar, bcs)
    nut = closure.nu_t_into(u, ScalarField(grid))
    N.call("sfb_fill_ghosts_scalar", _plan(grid), nut.data.data_ptr(), stream_ptr())
    scratch = torch.empty((16,) + tuple(u.u[0].shape), dtype=u.u[0].dtype, device=u.u[0].device)
    N.call("sfb_closure_pullback", _plan(grid), _KIND_CODE[closure.kind], closure.c, N.ptr3(u.u),
           nut.data.data_ptr(), N.ptr3(vbar.u), N.ptr3(out.u), scratch.data_ptr(), stream_ptr())
    return out


def scalar_max(f):
    mn, mx = ctypes.c_double(), ctypes.c_double()
    N.call("sfb_scalar_minmax", _plan(f.grid), f.data.data_ptr(), ctypes.byref(mn), ctypes.byref(mx), stream_ptr())
    return mn.value, mx.value


def eddy_stress_divergence(u, nut, out=None, scratch=None, accumulate=False):
    """les.py:343-417: divergence of the modelled stress 2 nu_t S on the
    velocity DOFs; fills nut's ghosts in place like the reference."""
    if out is None:
        out = VelocityField(u.grid)
    mn, _ = scalar_max(nut)
    if mn < 0:
        raise ValueError("eddy viscosity must be nonnegative")
    _eddy(u, nut, out, accumulate)
    return out
