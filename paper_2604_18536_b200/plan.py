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


def _dirichlet_values(c, dim):
    if callable(c.values):
        raise ConfigurationError("callable (space/time-varying) Dirichlet values are not supported on the GPU path")
    return [float(c.component_value(k)) for k in range(dim)]


def bcs_signature(bcs):
    sig = []
    for lo, hi in bcs.sides:
        for c in (lo, hi):
            code = _bc_code(c)
            vals = tuple(_dirichlet_values(c, bcs.dim)) if code == N.SFB_BC_DIRICHLET else ()
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
            if d.bc_lo[a] == N.SFB_BC_DIRICHLET:
                for k, v in enumerate(_dirichlet_values(lo, grid.dim)):
                    d.val_lo[a][k] = v
            if d.bc_hi[a] == N.SFB_BC_DIRICHLET:
                for k, v in enumerate(_dirichlet_values(hi, grid.dim)):
                    d.val_hi[a][k] = v
            d.width0[a] = float(grid.axes[a].widths[0])
        if halo_axis0:
            # ghost planes of axis 0 come from the neighbouring slab (distributed.py)
            d.bc_lo[0] = d.bc_hi[0] = N.SFB_BC_HALO
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


def get_plan(grid, bcs):
    key = bcs_signature(bcs)
    p = grid._plans.get(key)
    if p is None:
        p = Plan(grid, bcs)
        grid._plans[key] = p
    return p


def stream_ptr():
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
