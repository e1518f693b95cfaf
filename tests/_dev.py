"""Helpers shared by the GPU parity tests: build matching product/oracle
grids and move fields between them."""

import numpy as np

from oracle import stagflow_np as O


def pgrid_from_bounds(P, bounds, periodic, dtype=np.float64):
    return P.Grid(tuple(P.AxisCoords(np.asarray(b)) for b in bounds), periodic, dtype=dtype)


def grids(P, bounds, periodic, dtype=np.float64):
    return pgrid_from_bounds(P, bounds, periodic, dtype), O.OGrid(bounds, periodic, dtype)


def grids_from_case(P, case):
    dim = int(case["dim"])
    bounds = [case[f"bounds{a}"] for a in range(dim)]
    per = tuple(bool(p) for p in case["periodic"])
    return grids(P, bounds, per, np.dtype(str(case["dtype"])))


def pbcs(P, periodic, value=0.0):
    return P.BoundarySpec([
        (P.Periodic(), P.Periodic()) if p else (P.Dirichlet(value), P.Dirichlet(value)) for p in periodic
    ])


def obcs(periodic, value=0.0):
    return [("P", "P") if p else (("D", value), ("D", value)) for p in periodic]


def vel(P, grid, arrays):
    return P.VelocityField(grid, [np.array(a) for a in arrays])


def rel(got, ref):
    got = np.asarray(got, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    den = float(np.max(np.abs(ref)))
    if den == 0.0:
        return float(np.max(np.abs(got)))
    return float(np.max(np.abs(got - ref))) / den


def tol(dtype):
    return 1e-12 if np.dtype(dtype) == np.float64 else 1e-5


def random_vel(og, rng):
    u = og.zeros_vel()
    for a in range(og.dim):
        sl = og.udof(a)
        u[a][sl] = rng.standard_normal(u[a][sl].shape)
    return u


def cube_bounds(n, lengths=None, stretched=False, gamma=1.4):
    ns = (n,) * 3 if np.isscalar(n) else n
    out = []
    for a, m in enumerate(ns):
        ln = 1.0 + 0.3 * a if lengths is None else lengths[a]
        out.append(O.tanh_bounds(0.0, ln, m, gamma) if stretched else O.uniform_bounds(0.0, ln, m))
    return out
