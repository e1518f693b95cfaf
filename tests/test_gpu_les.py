"""GPU eddy-viscosity closures (les.py, csrc/les.cu) against golden vectors
produced by the reference itself: every model's nu_t, the eddy-stress
divergence, the closure in momentum_rhs, SSP33 / RK4 steps with a closure and
the closure-tightened adaptive step, on stretched periodic grids (2D, 3D) and
the channel (walls on y)."""

import numpy as np
import pytest

from _dev import grids, rel, vel
from _golden import load, ogrid
from _golden import vel as ovel
from oracle import les_np as LES

pytestmark = pytest.mark.gpu

MODELS = ["smagorinsky", "vreman", "qr", "wale", "sigma", "s3pqr"]


@pytest.fixture(scope="module")
def P():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_2604_18536_b200 as P

    return P


def _case(P, name):
    c = load(name)
    dim = int(c["dim"])
    bounds = [c[f"bounds{a}"] for a in range(dim)]
    per = tuple(bool(p) for p in c["periodic"])
    pg, og = grids(P, bounds, per)
    if all(per):
        bcs = P.BoundarySpec.all_periodic(dim)
        solver = P.make_solver("cg", pg, bcs, tol=1e-13, max_iter=5000)
        tol = 1e-8  # CG-limited (the reference ran CG at tol 1e-13)
    else:
        bcs = P.BoundarySpec.channel(dim=3, wall_axis=1)
        solver = P.make_solver("direct", pg, bcs)
        tol = 1e-12
    return c, pg, bcs, solver, tol


@pytest.mark.parametrize("name", ["les3d", "les2d", "les_channel"])
def test_closures_vs_reference_golden(P, name):
    c, pg, bcs, solver, tol = _case(P, name)
    d = pg.dim
    u = vel(P, pg, [c[f"u{a}"] for a in range(d)])
    for kind in MODELS:
        nut = P.ClosureModel(kind).nu_t(u).numpy()
        if kind == "sigma":
            # the reference's longdouble closed form loses ~1e-7 relative on
            # the second singular value of nearly two-component gradients
            # (channel IC); the kernel's invariant form is checked against the
            # same form in longdouble, and against the reference at 1e-5
            og = ogrid(c)
            acc = LES.nu_t_sigma_accurate(og, ovel(c, "u", d))
            assert rel(nut[og.pdof()], acc) <= 1e-12
            assert rel(nut, c["nut_sigma"]) <= 1e-5
        else:
            assert rel(nut, c[f"nut_{kind}"]) <= 1e-12, kind
    esd = P.eddy_stress_divergence(u, P.ScalarField(pg, c["nut_in"])).numpy()
    for a in range(d):
        assert rel(esd[a], c[f"esd{a}"]) <= 1e-12
    force = [0.5] + [0.0] * (d - 1)
    rhs = P.momentum_rhs(u, 0.01, force=force, closure=P.ClosureModel("vreman")).numpy()
    for a in range(d):
        assert rel(rhs[a], c[f"rhs_cl{a}"]) <= 1e-12
    for tag, tab, kind in (("ssp33", P.SSP33, "wale"), ("rk4", P.RK4, "smagorinsky")):
        setup = P.Setup(pg, bcs, nu=0.01, solver=solver, closure=P.ClosureModel(kind))
        st = setup.new_state(u0=vel(P, pg, [c[f"u{a}"] for a in range(d)]))
        st.workspace = P.Workspace(pg, tab.stages + 1)
        P.rk_step(st, 0.003, tab, setup.solver, setup)
        got = st.u.numpy()
        for a in range(d):
            assert rel(got[a], c[f"{tag}_u{a}"]) <= tol, (tag, a)
        assert rel(st.pressure.numpy(), c[f"{tag}_p"]) <= 10 * tol
    from paper_2604_18536_b200.timestep import _adaptive_dt

    setup = P.Setup(pg, bcs, nu=0.01, solver=solver, closure=P.ClosureModel("qr"), dt_max=1.0)
    st = setup.new_state(u0=vel(P, pg, [c[f"u{a}"] for a in range(d)]))
    assert abs(_adaptive_dt(st, setup) - float(c["adaptive_dt"])) <= 1e-13 * float(c["adaptive_dt"])


def test_closure_errors(P):
    c, pg, bcs, solver, tol = _case(P, "les3d")
    with pytest.raises(P.ConfigurationError):
        P.ClosureModel("nope")
    with pytest.raises(ValueError):
        P.ClosureModel("smagorinsky", c=-1.0)
    u = vel(P, pg, [c[f"u{a}"] for a in range(3)])
    neg = P.ScalarField(pg, -np.abs(c["nut_in"]) - 1.0)
    with pytest.raises(ValueError):
        P.eddy_stress_divergence(u, neg)
    none = P.ClosureModel("none")
    assert float(np.abs(none.nu_t(u).numpy()).max()) == 0.0
