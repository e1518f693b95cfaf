"""GPU matrix-free CG pressure solver (poisson.py:232-308, csrc/cg.cu) against
golden vectors produced by the reference's own CGPoissonSolver
(tests/golden/make_golden.py) and against the CPU oracle's restatement:
stretched grids with periodic, Dirichlet (non-zero wall values) and symmetric
sides; solve, projection and an SSP33 step; the reference's error behaviour.

CG iterates are rounding-sensitive, so the bar is the solver tolerance
scale (1e-8 relative, the reference's own cross-solver bar,
test_poisson.py:186-199), not bitwise."""

import numpy as np
import pytest

from _dev import grids, rel, vel
from _golden import load, sides_bcs
from oracle import stagflow_np as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_2604_18536_b200 as P

    return P


def _pbcs(P, obcs):
    def one(c):
        if c == "P":
            return P.Periodic()
        if c == "S":
            return P.Symmetric()
        return P.Dirichlet(c[1])

    return P.BoundarySpec([tuple(one(c) for c in side) for side in obcs])


def _case(P, name):
    c = load(name)
    dim = int(c["dim"])
    bounds = [c[f"bounds{a}"] for a in range(dim)]
    pg, og = grids(P, bounds, tuple(bool(p) for p in c["periodic"]))
    ob = sides_bcs(c)
    return c, pg, og, ob, _pbcs(P, ob)


@pytest.mark.parametrize("name", ["cg3d_mixed", "cg2d_stretched"])
def test_cg_vs_reference_golden(P, name):
    c, pg, og, ob, bcs = _case(P, name)
    d = pg.dim
    solver = P.make_solver("cg", pg, bcs, max_iter=1000)
    assert solver.kind == "cg" and solver.tolerance == 1e-10
    sol = solver.solve(P.ScalarField(pg, c["rhs"])).numpy()
    assert rel(sol[pg.p_slices()], c["sol"][og.pdof()]) <= 1e-8
    assert abs(solver.iterations - int(c["iterations"])) <= 3
    h = solver.residual_history
    assert len(h) == solver.iterations + 1
    assert h[-1] <= 1e-10 * h[0] and abs(h[0] - float(c["residual_history"][0])) <= 1e-12 * h[0]
    u = vel(P, pg, [c[f"u{a}"] for a in range(d)])
    p = P.project_into(u, solver, bcs)
    got = u.numpy()
    for a in range(d):
        assert rel(got[a], c[f"uproj{a}"]) <= 1e-8
    assert rel(p.numpy(), c["pproj"]) <= 1e-8
    setup = P.Setup(pg, bcs, nu=float(c["nu"]), solver=solver)
    st = setup.new_state(u0=vel(P, pg, [c[f"uproj{a}"] for a in range(d)]))
    P.rk_step(st, float(c["dt"]), P.SSP33, setup.solver, setup)
    got = st.u.numpy()
    for a in range(d):
        assert rel(got[a], c[f"ssp33_u{a}"]) <= 1e-8
    assert rel(st.pressure.numpy(), c["ssp33_p"]) <= 1e-7


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_cg_vs_oracle_larger(P, dtype):
    """40 x 24 x 20, tanh-stretched in y and z, periodic / walls / symmetric+wall."""
    bounds = [O.uniform_bounds(0.0, 2.0, 40), O.tanh_bounds(0.0, 1.0, 24, 1.6), O.tanh_bounds(0.0, 0.7, 20, 1.2)]
    ob = [("P", "P"), (("D", 0.0), ("D", 0.0)), ("S", ("D", 0.1))]
    pg, og = grids(P, bounds, (True, False, False), dtype)
    bcs = _pbcs(P, ob)
    rng = np.random.default_rng(4)
    rhs = og.zeros()
    rhs[og.pdof()] = rng.standard_normal(og.shape)
    solver = P.make_solver("cg", pg, bcs, max_iter=2000)
    got = solver.solve(P.ScalarField(pg, rhs)).numpy()[pg.p_slices()]
    og64 = O.OGrid(bounds, (True, False, False), np.float64)
    ref = O.CGSolve(og64, ob, tol=1e-12, max_iter=4000)(rhs[og.pdof()].astype(np.float64))
    # fp32: the reference default tol 1e-5 on |r|, times the operator condition
    assert rel(got, ref) <= (1e-8 if dtype == np.float64 else 1e-3)


def test_cg_errors(P):
    c, pg, og, ob, bcs = _case(P, "cg3d_mixed")
    with pytest.raises(ValueError):
        P.make_solver("cg", pg, bcs, tol=0.0)
    solver = P.make_solver("cg", pg, bcs, max_iter=3)
    with pytest.raises(P.ConvergenceError) as e:
        solver.solve(P.ScalarField(pg, c["rhs"]))
    assert e.value.iterations == 3 and e.value.residual > 1e-10
    assert len(solver.residual_history) == 4
