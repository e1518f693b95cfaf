"""Staggered field containers on the GPU and ghost filling.

Mirror of the reference's ``fields.py`` (fields.py:16-157): same classes and
extended C-order layout (one ghost layer per side, axis 0 slowest), with
storage in CUDA tensors.  ``VelocityField.u[a]`` is a ``torch.Tensor`` of
``grid.ext_shape``; ``.numpy()`` / ``from_numpy`` convert at the API edge.
"""

import numpy as np
import torch

from . import _native as N
from . import alloc
from .plan import get_plan, stream_ptr


def _as_device(grid, arr):
    if isinstance(arr, torch.Tensor):
        if tuple(arr.shape) != tuple(grid.ext_shape):
            raise ValueError("array shape does not match the grid's extended shape")
        if arr.dtype != alloc.torch_dtype(grid.dtype) or not arr.is_cuda or not arr.is_contiguous():
            raise ValueError("field arrays must be contiguous CUDA tensors of the grid dtype")
        return arr
    a = np.ascontiguousarray(np.asarray(arr, dtype=grid.dtype))
    if a.shape != tuple(grid.ext_shape):
        raise ValueError("array shape does not match the grid's extended shape")
    t = alloc.zeros(grid.ext_shape, grid.dtype)
    t.copy_(torch.from_numpy(a))
    return t


class ScalarField:
    """Volume-centred scalar with ghost layer (fields.py:16-30)."""

    def __init__(self, grid, data=None, empty=False):
        self.grid = grid
        if data is None:
            self.data = (alloc.empty if empty else alloc.zeros)(grid.ext_shape, grid.dtype)
        else:
            self.data = _as_device(grid, data)

    @property
    def interior(self):
        return self.data[self.grid.p_slices()]

    def copy(self):
        f = ScalarField(self.grid)
        f.data.copy_(self.data)
        return f

    def numpy(self):
        return self.data.cpu().numpy()


class VelocityField:
    """d staggered components on the GPU (fields.py:33-53)."""

    def __init__(self, grid, components=None, empty=False):
        self.grid = grid
        if components is None:
            mk = alloc.empty if empty else alloc.zeros
            self.u = [mk(grid.ext_shape, grid.dtype) for _ in range(grid.dim)]
        else:
            self.u = [_as_device(grid, c) for c in components]

    def copy(self):
        v = VelocityField(self.grid)
        v.copy_from(self)
        return v

    def copy_from(self, other):
        for dst, src in zip(self.u, other.u):
            dst.copy_(src if isinstance(src, torch.Tensor) else torch.from_numpy(np.asarray(src, dtype=self.grid.dtype)))

    def interiors(self):
        return [self.u[a][self.grid.u_slices(a)] for a in range(self.grid.dim)]

    def numpy(self):
        return [c.cpu().numpy() for c in self.u]

    @classmethod
    def from_numpy(cls, grid, arrays):
        return cls(grid, [np.asarray(a) for a in arrays])


def fill_ghosts_scalar(f, bcs):
    """fields.py:81-93"""
    N.call("sfb_fill_ghosts_scalar", get_plan(f.grid, bcs).handle, f.data.data_ptr(), stream_ptr())
    return f


def fill_ghosts_velocity(v, bcs, t=0.0):
    """fields.py:96-140; callable Dirichlet walls are evaluated at ``t``
    (spatially uniform ones on the device path)."""
    plan = get_plan(v.grid, bcs)
    if plan.moving:
        plan.set_time(float(t))
    N.call("sfb_fill_ghosts_velocity", plan.handle, N.ptr3(v.u), stream_ptr())
    return v


def interpolate_to_centers(v):
    """fields.py:143-157: two-point average of each component to the centres
    (requires filled ghosts).  Returns interior tensors."""
    grid = v.grid
    p = grid.p_slices()
    out = []
    for a in range(grid.dim):
        lo = list(p)
        lo[a] = slice(0, grid.shape[a])
        out.append(0.5 * (v.u[a][tuple(lo)] + v.u[a][p]))
    return out
