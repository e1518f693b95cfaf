"""Matrix-free staggered stencils on the GPU (mirror of operators.py:1-301).

Same call signatures as the reference: pure forms allocate their output,
in-place forms take ``out=`` (and a ``scratch`` argument kept for signature
compatibility -- the CUDA kernels need no work arrays).  Inputs must carry
filled ghosts; outputs are whole extended arrays with only DOF ranges
written and everything else zeroed unless ``accumulate=True``.

The ghost fills of the *inputs* follow the boundary conditions of the plan
the field was last filled with; operators that need a plan but no BCs
(divergence, convection, ...) use the grid's periodic/wall layout with
homogeneous values, which only affects how *outputs* are bounded -- the
stencils themselves read the ghosts from memory, as the reference does.
"""

import numpy as np
import torch

from . import _native as N
from . import alloc
from .bcs import BoundarySpec, Dirichlet, Periodic
from .errors import ConfigurationError
from .fields import ScalarField, VelocityField
from .plan import get_plan, stream_ptr


class KernelScratch:
    """Signature-compatible stand-in for the reference's four work arrays
    (operators.py:93-100); the fused kernels need none."""

    def __init__(self, grid):
        self.grid = grid


def default_bcs(grid):
    """Periodic axes stay periodic, wall axes get homogeneous Dirichlet."""
    return BoundarySpec([
        (Periodic(), Periodic()) if p else (Dirichlet(0.0), Dirichlet(0.0)) for p in grid.periodic
    ])


def _plan(grid):
    return get_plan(grid, default_bcs(grid)).handle


def divergence(u, out=None, scratch=None):
    """operators.py:108-122"""
    grid = u.grid
    if out is None:
        out = ScalarField(grid)
    N.call("sfb_divergence", _plan(grid), N.ptr3(u.u), out.data.data_ptr(), stream_ptr())
    return out


def pressure_gradient(pf, out=None):
    """operators.py:125-137"""
    grid = pf.grid
    if out is None:
        out = VelocityField(grid)
    N.call("sfb_pressure_gradient", _plan(grid), pf.data.data_ptr(), N.ptr3(out.u), stream_ptr())
    return out


def diffusion(u, nu, out=None, scratch=None, accumulate=False):
    """operators.py:140-170"""
    if nu < 0:
        raise ValueError(f"viscosity must be nonnegative, got {nu}")
    grid = u.grid
    if out is None:
        out = VelocityField(grid)
    N.call("sfb_diffusion", _plan(grid), N.ptr3(u.u), float(nu), N.ptr3(out.u), int(bool(accumulate)), stream_ptr())
    return out


def convection(u, out=None, scratch=None, accumulate=False):
    """operators.py:173-215"""
    grid = u.grid
    if out is None:
        out = VelocityField(grid)
    N.call("sfb_convection", _plan(grid), N.ptr3(u.u), N.ptr3(out.u), int(bool(accumulate)), stream_ptr())
    return out


def _is_constant(f):
    return np.isscalar(f) or (isinstance(f, np.ndarray) and f.ndim == 0) or (
        isinstance(f, torch.Tensor) and f.dim() == 0)


def constant_force(grid, force):
    """Per-component constants for the fused kernels (0.0 for components
    given as fields), or None."""
    if force is None:
        return None
    return [float(grid.dtype.type(float(f))) if _is_constant(f) else 0.0 for f in force]


def force_fields(grid, force):
    """Per-DOF force components as extended device arrays (zero off the DOFs),
    or None when every component is a constant.  Accepts the reference's
    sampled arrays (DOF-shaped, operators.py:249-258), extended arrays, or
    tensors of either shape; constants in a mixed list become constant
    fields.  Cached on the list object for repeated stage launches."""
    if force is None or all(_is_constant(f) for f in force):
        return None
    cached = getattr(force, "_sfb_fields", None) if isinstance(force, ForceList) else None
    if cached is not None:
        return cached
    out = []
    for a in range(grid.dim):
        f = force[a]
        full = alloc.zeros(grid.ext_shape, grid.dtype)
        sl = grid.u_slices(a)
        if _is_constant(f):
            full[sl] = float(grid.dtype.type(float(f)))
        else:
            t = f if isinstance(f, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(np.asarray(f, dtype=grid.dtype)))
            t = t.to(device=full.device, dtype=full.dtype)
            if tuple(t.shape) == tuple(grid.ext_shape):
                full[sl] = t[sl]
            else:
                full[sl] = t
        out.append(full)
    if isinstance(force, ForceList):
        force._sfb_fields = out
    return out


class ForceList(list):
    """sample_force's result: a list (as the reference returns) that caches
    its device fields."""


def momentum_rhs(u, nu, force=None, closure=None, t=0.0, out=None, scratch=None):
    """operators.py:218-238: convection + diffusion + force in one kernel,
    then the closure's eddy-stress term (operators.py:236-237)."""
    if nu < 0:
        raise ValueError(f"viscosity must be nonnegative, got {nu}")
    grid = u.grid
    if out is None:
        out = VelocityField(grid)
    fv = constant_force(grid, force)
    fp = None
    if fv is not None:
        fp = (N.ctypes.c_double * 3)(*(fv + [0.0] * (3 - len(fv))))
    ff = force_fields(grid, force)
    ffp = N.ctypes.byref(N.ptr3(ff)) if ff is not None else None
    N.call("sfb_momentum_rhs", _plan(grid), N.ptr3(u.u), float(nu), fp, ffp, N.ptr3(out.u), stream_ptr())
    if closure is not None:
        closure.add_rhs(u, out, scratch)
    return out


def sample_force(grid, force):
    """operators.py:241-259: None, a d-vector of constants, or a callable
    ``f(component, *coords)`` sampled once at the velocity points (the
    reference's broadcast and dtype cast, kept on the host as DOF-shaped
    arrays; the stage kernels read them as device fields)."""
    if force is None:
        return None
    if callable(force):
        out = ForceList()
        for a in range(grid.dim):
            coords = [grid.broadcast(c, g) for g, c in enumerate(grid.face_coords(a))]
            full = np.broadcast_to(force(a, *coords), grid.ext_shape)
            out.append(np.array(full[grid.u_slices(a)], dtype=grid.dtype))
        return out
    return [grid.dtype.type(f) for f in force]


def _table(grid, values, axis, s):
    return grid.broadcast(values[s], axis)


def velocity_weights(grid):
    """operators.py:262-272 (host arrays)."""
    out = []
    for a in range(grid.dim):
        sl = grid.u_slices(a)
        w = np.ones((1,) * grid.dim, dtype=grid.dtype)
        for g in range(grid.dim):
            w = w * _table(grid, grid.du[g] if g == a else grid.dx[g], g, sl[g])
        out.append(np.ascontiguousarray(np.broadcast_to(w, tuple(s.stop - s.start for s in sl))))
    return out


def pressure_weights(grid):
    """operators.py:275-281 (host array)."""
    p = grid.p_slices()
    w = np.ones((1,) * grid.dim, dtype=grid.dtype)
    for g in range(grid.dim):
        w = w * _table(grid, grid.dx[g], g, p[g])
    return np.ascontiguousarray(np.broadcast_to(w, grid.shape))


def kinetic_energy(u):
    """operators.py:284-291 (device reduction, fp64 accumulation)."""
    out = N.ctypes.c_double()
    N.call("sfb_kinetic_energy", _plan(u.grid), N.ptr3(u.u), N.ctypes.byref(out), stream_ptr())
    return out.value


def weighted_inner(u, v):
    """operators.py:294-301"""
    out = N.ctypes.c_double()
    N.call("sfb_weighted_inner", _plan(u.grid), N.ptr3(u.u), N.ptr3(v.u), N.ctypes.byref(out), stream_ptr())
    return out.value


__all__ = [
    "KernelScratch", "divergence", "pressure_gradient", "diffusion", "convection", "momentum_rhs",
    "sample_force", "velocity_weights", "pressure_weights", "kinetic_energy", "weighted_inner",
]

_ = (torch, alloc)
