"""Staggered grids (host side): 1D profiles and the extended width tables.

Mirror of the reference's ``grid.py`` API (grid.py:26-223).  The tables are
built on the host once per grid, in the grid dtype exactly as the reference
builds them, and uploaded bit-for-bit into a device plan (``plan.py``); the
kernels never recompute geometry.
"""

from dataclasses import dataclass

import numpy as np

from .errors import ConfigurationError


@dataclass(frozen=True)
class AxisCoords:
    """Strictly increasing volume boundaries of one axis (grid.py:26-58)."""

    boundaries: np.ndarray

    def __post_init__(self):
        b = np.asarray(self.boundaries, dtype=float)
        if b.ndim != 1 or b.size < 2:
            raise ValueError("need at least two boundary coordinates")
        if not np.all(np.diff(b) > 0):
            raise ValueError("boundaries must be strictly increasing")
        object.__setattr__(self, "boundaries", b)

    n = property(lambda self: self.boundaries.size - 1)
    widths = property(lambda self: np.diff(self.boundaries))
    centers = property(lambda self: 0.5 * (self.boundaries[:-1] + self.boundaries[1:]))
    a = property(lambda self: self.boundaries[0])
    b = property(lambda self: self.boundaries[-1])


def _interval(a, b, n):
    if n < 1:
        raise ValueError(f"need at least one volume, got n={n}")
    if not a < b:
        raise ValueError(f"invalid interval: a={a} must be < b={b}")


def _pin(x, a, b):
    x[0], x[-1] = a, b
    return AxisCoords(x)


def uniform_grid(a, b, n):
    """grid.py:68-71"""
    _interval(a, b, n)
    return AxisCoords(np.linspace(a, b, n + 1))


def cosine_grid(a, b, n):
    """grid.py:74-80"""
    _interval(a, b, n)
    t = np.arange(n + 1)
    return _pin(a + (1.0 - np.cos(np.pi * t / n)) / 2.0 * (b - a), a, b)


def tanh_grid(a, b, n, gamma):
    """grid.py:83-91"""
    _interval(a, b, n)
    if gamma <= 0:
        raise ValueError(f"stretching parameter must be positive, got {gamma}")
    xi = np.arange(n + 1) / n
    return _pin(a + (b - a) / 2.0 * (1.0 + np.tanh(gamma * (2.0 * xi - 1.0)) / np.tanh(gamma)), a, b)


def stretched_grid(a, b, n, s):
    """grid.py:94-104"""
    _interval(a, b, n)
    if s <= 0:
        raise ValueError(f"stretch ratio must be positive, got {s}")
    if s == 1.0:
        return uniform_grid(a, b, n)
    t = np.arange(n + 1)
    return _pin(a + (b - a) * (1.0 - s ** t) / (1.0 - float(s) ** n), a, b)


PROFILES = {"uniform": uniform_grid, "cosine": cosine_grid, "tanh": tanh_grid, "stretched": stretched_grid}


def _axis_tables(ax, periodic):
    """Extended dx/du/xb/xc of one axis, float64 (grid.py:143-166)."""
    w = ax.widths
    n = w.size
    dx = np.concatenate(([w[-1] if periodic else w[0]], w, [w[0] if periodic else w[-1]]))
    beyond = w[1 % n] if periodic else w[-1]
    du = np.empty(n + 2)
    du[: n + 1] = 0.5 * (dx[: n + 1] + dx[1:])
    du[n + 1] = 0.5 * (dx[n + 1] + beyond)
    xb = np.append(ax.boundaries, ax.boundaries[-1] + dx[n + 1])
    xc = np.concatenate(([ax.boundaries[0] - 0.5 * dx[0]], ax.centers, [ax.boundaries[-1] + 0.5 * dx[n + 1]]))
    return dx, du, xb, xc


class Grid:
    """Immutable 2D/3D staggered grid (grid.py:115-216).

    ``dx``, ``du``, ``xb``, ``xc`` are host numpy tables (length n+2 per axis,
    grid dtype, read-only).  Field storage lives on the GPU (fields.py).
    """

    def __init__(self, axes, periodic, dtype=np.float64):
        if not 2 <= len(axes) <= 3:
            raise ConfigurationError(f"unsupported dimension {len(axes)}; need 2 or 3")
        if len(periodic) != len(axes):
            raise ValueError("one periodic flag per axis required")
        self.dtype = np.dtype(dtype)
        if self.dtype not in (np.dtype(np.float64), np.dtype(np.float32)):
            raise ConfigurationError(f"unsupported dtype {self.dtype}; need float64 or float32")
        self.axes = tuple(axes)
        self.periodic = tuple(bool(p) for p in periodic)
        self.dim = len(axes)
        self.shape = tuple(ax.n for ax in axes)
        self.ext_shape = tuple(n + 2 for n in self.shape)
        tabs = [_axis_tables(ax, p) for ax, p in zip(self.axes, self.periodic)]
        self.dx, self.du, self.xb, self.xc = ([t[i].astype(self.dtype) for t in tabs] for i in range(4))
        for arr in (*self.dx, *self.du, *self.xb, *self.xc):
            arr.flags.writeable = False
        self._packed = None
        self._plans = {}

    @property
    def uniform(self):
        """grid.py:177-183"""
        return all(np.allclose(ax.widths, ax.widths[0], rtol=1e-12, atol=0.0) for ax in self.axes)

    def broadcast(self, values, axis):
        shape = [1] * self.dim
        shape[axis] = values.shape[0]
        return values.reshape(shape)

    def p_slices(self):
        return tuple(slice(1, n + 1) for n in self.shape)

    def u_slices(self, component):
        return tuple(
            slice(1, n) if (a == component and not self.periodic[a]) else slice(1, n + 1)
            for a, n in enumerate(self.shape)
        )

    def face_coords(self, component):
        return [self.xb[a] if a == component else self.xc[a] for a in range(self.dim)]

    def packed_tables(self):
        """The SFB_NTAB per-axis tables of the C ABI, in the grid dtype
        (operators.py:47-84 formulas), packed as float64 for transport."""
        if self._packed is None:
            parts = []
            for a, n in enumerate(self.shape):
                dx, du = self.dx[a], self.du[a]
                one = self.dtype.type(1.0)
                w_lo = dx / (2.0 * du)
                w_hi = 1.0 - w_lo
                own_hi = np.zeros(n + 2, self.dtype)
                own_lo = np.zeros(n + 2, self.dtype)
                tan_hi = np.zeros(n + 2, self.dtype)
                tan_lo = np.zeros(n + 2, self.dtype)
                own_hi[: n + 1] = 1.0 / (du[: n + 1] * dx[1:])
                own_lo[: n + 1] = 1.0 / (du[: n + 1] * dx[: n + 1])
                tan_hi[: n + 1] = 1.0 / (dx[: n + 1] * du[: n + 1])
                tan_lo[1:] = 1.0 / (dx[1:] * du[:-1])
                for t in (dx, du, one / dx, one / du, w_lo, w_hi, own_hi, own_lo, tan_hi, tan_lo):
                    parts.append(np.asarray(t, dtype=self.dtype).astype(np.float64))
            self._packed = np.ascontiguousarray(np.concatenate(parts))
        return self._packed


def build_grid(axes, bcs, dtype=np.float64):
    """grid.py:219-223"""
    if len(axes) != bcs.dim:
        raise ValueError("axis count and boundary spec dimension differ")
    return Grid(axes, bcs.periodic, dtype=dtype)
