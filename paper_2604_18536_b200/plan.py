"""Device plans: one native ``sfb_plan`` per (grid, boundary conditions).

A plan owns the grid tables on the device and the boundary metadata the
fused ghost handling needs (bcs.py:47-83, fields.py:96-140).  Plans are
cached on the grid object; after creation no call allocates device memory.
"""

import ctypes

import numpy as np
import torch

from . import _native as N
from .bcs import Dirichlet, Periodic, Symmetric
from .errors import ConfigurationError


def _bc_code(c):
    if isinstance(c, Periodic):
        return N.SFB_BC_PERIODIC
    if isinstance(c, Dirichlet):
        return N.SFB_BC_DIRICHLET
    if isinstance(c, Symmetric):
        return N.SFB_BC_SYMMETRIC
    raise ConfigurationError(f"unsupported boundary condition {c!r}")


def _axslice(ndim, axis, idx):
    sl = [slice(None)] * ndim
    sl[axis] = idx
    return tuple(sl)


def _wall_coords(grid, component, axis, wall_x):
    """fields.py:62-69: coordinate arrays at the wall (broadcastable over a
    ghost slice), in the grid dtype."""
    coords = []
    for g in range(grid.dim):
        if g == axis:
            coords.append(np.asarray(wall_x, dtype=grid.dtype))
        else:
            c = grid.face_coords(component)[g]
            coords.append(grid.broadcast(c, g)[_axslice(grid.dim, axis, 0)])
    return coords


def wall_value(grid, c, comp, axis, side, t=0.0):
    """fields.py:72-76: a Dirichlet value of one component on one wall at time
    ``t``.  A callable is evaluated on the wall's face coordinates; the device
    path needs it uniform over the wall (a moving or oscillating wall), else
    ConfigurationError."""
    if not callable(c.values):
        return float(c.component_value(comp))
    wall_x = grid.xb[axis][0] if side == 0 else grid.xb[axis][grid.shape[axis]]
    v = np.asarray(c.values(comp, *_wall_coords(grid, comp, axis, wall_x), t), dtype=np.float64)
    flat = v.reshape(-1)
    if flat.size == 0:
        raise ConfigurationError("callable Dirichlet value returned no values")
    if not np.all(flat == flat[0]):
        raise ConfigurationError("callable Dirichlet values must be uniform over the wall on the GPU path "
                                 "(time-dependent, spatially constant walls are supported)")
    return float(flat[0])


def _dirichlet_values(c, dim):
    return [float(c.component_value(k)) for k in range(dim)]


def bcs_signature(bcs):
    sig = []
    for lo, hi in bcs.sides:
        for c in (lo, hi):
            code = _bc_code(c)
            if code != N.SFB_BC_DIRICHLET:
                vals = ()
            elif callable(c.values):
                vals = ("callable", id(c))
            else:
                vals = tuple(_dirichlet_values(c, bcs.dim))
            sig.append((code, vals))
    return tuple(sig)


class Plan:
    def __init__(self, grid, bcs, halo_axis0=False):
        if bcs.dim != grid.dim:
            raise ValueError("axis count and boundary spec dimension differ")
        if tuple(bcs.periodic) != tuple(grid.periodic):
            raise ValueError("boundary periodicity does not match the grid")
        if not torch.cuda.is_available():
            raise RuntimeError("paper_2604_18536_b200 needs a CUDA device (B200); there is no CPU path")
        self.grid = grid
        self.bcs = bcs
        self.device = torch.device("cuda", torch.cuda.current_device())
        d = N.GridDesc()
        d.dim = grid.dim
        d.dtype = N.SFB_F64 if grid.dtype == np.float64 else N.SFB_F32
        for a in range(grid.dim):
            d.n[a] = grid.shape[a]
            lo, hi = bcs.sides[a]
            d.bc_lo[a] = _bc_code(lo)
            d.bc_hi[a] = _bc_code(hi)
            for side, c, vals in ((0, lo, d.val_lo), (1, hi, d.val_hi)):
                if _bc_code(c) == N.SFB_BC_DIRICHLET:
                    for k in range(grid.dim):
                        vals[a][k] = wall_value(grid, c, k, a, side, 0.0)
            d.width0[a] = float(grid.axes[a].widths[0])
        if halo_axis0:
            # ghost planes of axis 0 come from the neighbouring slab (distributed.py)
            d.bc_lo[0] = d.bc_hi[0] = N.SFB_BC_HALO
        # callable Dirichlet walls: re-evaluated at every fill time (set_time)
        self.moving = any(isinstance(c, Dirichlet) and callable(c.values) for sides in bcs.sides for c in sides)
        self._t = 0.0
        self._tables = grid.packed_tables()
        d.tables = self._tables.ctypes.data_as(ctypes.POINTER(ctypes.c_double))
        h = ctypes.c_void_p()
        with torch.cuda.device(self.device):
            N.call("sfb_plan_create", ctypes.byref(d), ctypes.byref(h))
        self.handle = h

    def __del__(self):
        h = getattr(self, "handle", None)
        if h is not None and h.value:
            try:
                N.lib.sfb_plan_destroy(h)
            except Exception:  # pragma: no cover - interpreter shutdown
                pass


    def set_time(self, t):
        """Evaluate callable Dirichlet walls at time ``t`` (fields.py:72-76)
        for the fills and projections that follow; constant walls: no-op."""
        if not self.moving or t == self._t:
            return
        lo, hi = (ctypes.c_double * 9)(), (ctypes.c_double * 9)()
        for a, (clo, chi) in enumerate(self.bcs.sides):
            for side, c, arr in ((0, clo, lo), (1, chi, hi)):
                if isinstance(c, Dirichlet):
                    for k in range(self.grid.dim):
                        arr[3 * a + k] = wall_value(self.grid, c, k, a, side, t)
        N.call("sfb_plan_set_walls", self.handle, lo, hi)
        self._t = t


def set_time(grid, bcs, t):
    """Plan.set_time for (grid, bcs) when its walls move."""
    p = get_plan(grid, bcs)
    if p.moving:
        p.set_time(float(t))


def get_plan(grid, bcs):
    key = bcs_signature(bcs)
    p = grid._plans.get(key)
    if p is None:
        p = Plan(grid, bcs)
        grid._plans[key] = p
    return p


def stream_ptr():
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
