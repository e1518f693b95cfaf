"""Pin the CPU oracle against the round-2 golden vectors produced by the
reference itself (tests/golden/make_golden_r2.py).  CPU only."""

import numpy as np

from _golden import load, ogrid, sides_bcs, vel
from oracle import stagflow_np as O


def _rel(a, b):
    den = max(float(np.max(np.abs(b))), 1e-300)
    return float(np.max(np.abs(np.asarray(a, dtype=np.float64) - b))) / den


def test_fold_ghosts_bitwise():
    """adjoint.py:53-111 with periodic / Dirichlet / symmetric sides mixed."""
    for name in ("folds3d", "folds2d"):
        c = load(name)
        g = ogrid(c)
        bcs = sides_bcs(c)
        fv = O.fold_velocity(g, bcs, vel(c, "v", g.dim))
        for a in range(g.dim):
            assert np.array_equal(fv[a], c[f"fv{a}"])
        assert np.array_equal(O.fold_scalar(g, bcs, c["f"].copy()), c["ff"])


def test_force_field_rhs_and_steps():
    """sample_force of a callable: momentum_rhs bitwise, RK4 / SSP33 steps."""
    c = load("force_field")
    g = ogrid(c)
    force = [c[f"force{a}"] for a in range(3)]
    u0 = vel(c, "u0", 3)
    rh = O.momentum_rhs(g, u0, float(c["nu"]), force)
    for a in range(3):
        assert np.array_equal(rh[a], c[f"rhs{a}"])
    bcs = O.periodic_bcs(3)
    solve = O.SpectralSolve(g)
    for meth, tab in (("rk4", O.RK4), ("ssp33", O.SSP33)):
        u, p = O.rk_step(g, bcs, solve, vel(c, "u0", 3), float(c["dt"]), tab, float(c["nu"]), force)
        for a in range(3):
            assert np.array_equal(u[a], c[f"{meth}_u{a}"])
        assert np.array_equal(p, c[f"{meth}_p"])


def test_direct_periodic_box_equals_spectral_gauge():
    """The reference's augmented direct solve on a periodic uniform box and
    the spectral solve agree (same weighted zero-mean gauge): the basis of
    mapping solver="direct" to the FFT kernels on such grids."""
    c = load("direct_any")
    cc = {k[4:]: v for k, v in c.items() if k.startswith("box_")}
    g = ogrid(cc)
    u = vel(cc, "u", 3)
    O.project_into(g, O.periodic_bcs(3), O.SpectralSolve(g), u)
    for a in range(3):
        assert _rel(u[a], cc[f"v{a}"]) <= 1e-12


def test_solve_transpose_uniform_bitwise():
    c = load("solve_transpose")
    cc = {k[4:]: v for k, v in c.items() if k.startswith("uni_")}
    g = ogrid(cc)
    got = O.poisson_solve_transpose(g, O.SpectralSolve(g), cc["pbar"].copy())
    assert _rel(got, cc["out"]) <= 1e-14
