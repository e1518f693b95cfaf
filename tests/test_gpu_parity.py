"""GPU parity: CUDA path (through the C ABI) vs the CPU oracle and the
reference's golden vectors.  Tolerances (BASELINE.json north star): relative
max-abs 1e-12 in fp64, 1e-5 in fp32, per call / per step from a shared state.
"""

import math

import numpy as np
import pytest

from _dev import cube_bounds, grids, grids_from_case, obcs, pbcs, random_vel, rel, tol, vel
from _golden import load
from oracle import stagflow_np as O
from oracle.channel_np import ChannelSolve

pytestmark = pytest.mark.gpu

OPS = ["ops3d_stretched", "ops3d_uniform", "ops2d_stretched", "ops3d_stretched_f32"]


@pytest.fixture(scope="module")
def P():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    import paper_2604_18536_b200 as P

    return P


# ------------------------------------------------------------------ operators
@pytest.mark.parametrize("name", OPS)
def test_operators_match_reference_golden(P, name):
    c = load(name)
    pg, og = grids_from_case(P, c)
    d = pg.dim
    t = tol(pg.dtype)
    u = vel(P, pg, [c[f"u{a}"] for a in range(d)])
    nu = float(c["nu"])
    assert rel(P.divergence(u).numpy(), c["div"]) <= t
    pf = P.ScalarField(pg, c["p"])
    gr = P.pressure_gradient(pf).numpy()
    df = P.diffusion(u, nu).numpy()
    cv = P.convection(u).numpy()
    rh = P.momentum_rhs(u, nu, force=P.operators.sample_force(pg, c["force"])).numpy()
    for a in range(d):
        assert rel(gr[a], c[f"grad{a}"]) <= t
        assert rel(df[a], c[f"diff{a}"]) <= t
        assert rel(cv[a], c[f"conv{a}"]) <= t
        assert rel(rh[a], c[f"rhs{a}"]) <= t
        # non-DOF entries are exactly zero, as in the reference
        assert np.array_equal(rh[a] == 0, c[f"rhs{a}"] == 0) or rel(rh[a], c[f"rhs{a}"]) <= t
    assert abs(P.kinetic_energy(u) - float(c["ke"])) <= t * abs(float(c["ke"]))
    cfl = P.cfl_dt(u, nu, pg, 0.85, 0.85)
    assert abs(cfl - float(c["cfl"])) <= t * float(c["cfl"])


@pytest.mark.parametrize("stretched", [False, True])
@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_momentum_rhs_random_3d(P, stretched, dtype):
    rng = np.random.default_rng(1)
    bounds = cube_bounds((24, 20, 28), stretched=stretched)
    pg, og = grids(P, bounds, (True,) * 3, dtype)
    u = random_vel(og, rng)
    O.fill_velocity(og, O.periodic_bcs(3), u)
    ref = O.momentum_rhs(og, u, 0.013, (0.5, -0.25, 0.125))
    got = P.momentum_rhs(vel(P, pg, u), 0.013, force=(0.5, -0.25, 0.125)).numpy()
    for a in range(3):
        assert rel(got[a], ref[a]) <= tol(dtype)


def test_operators_channel_walls(P):
    """Stencils and fills on a wall-bounded (Dirichlet y, nonzero value) grid."""
    rng = np.random.default_rng(2)
    bounds = [O.uniform_bounds(0, 2.0, 12), O.tanh_bounds(0, 2.0, 10, 2.0), O.uniform_bounds(0, 1.0, 8)]
    per = (True, False, True)
    pg, og = grids(P, bounds, per)
    ob = [("P", "P"), (("D", (0.3, -0.2, 0.1)), ("D", (-0.1, 0.0, 0.25))), ("P", "P")]
    pb = P.BoundarySpec([(P.Periodic(), P.Periodic()),
                         (P.Dirichlet((0.3, -0.2, 0.1)), P.Dirichlet((-0.1, 0.0, 0.25))),
                         (P.Periodic(), P.Periodic())])
    u = [rng.standard_normal(og.ext_shape) for _ in range(3)]  # garbage ghosts
    ud = vel(P, pg, u)
    O.fill_velocity(og, ob, u)
    P.fill_ghosts_velocity(ud, pb)
    got = ud.numpy()
    for a in range(3):
        assert np.array_equal(got[a], u[a])
    ref = O.momentum_rhs(og, u, 0.02, (1.0, 0.0, 0.0))
    rh = P.momentum_rhs(ud, 0.02, force=(1.0, 0.0, 0.0)).numpy()
    for a in range(3):
        assert rel(rh[a], ref[a]) <= 1e-12
    assert rel(P.divergence(ud).numpy(), O.divergence(og, u)) <= 1e-12


def test_fill_symmetric_and_mixed(P):
    rng = np.random.default_rng(3)
    bounds = [O.uniform_bounds(0, 1.0, 6), O.uniform_bounds(0, 1.0, 7), O.uniform_bounds(0, 1.0, 5)]
    per = (False, False, True)
    pg, og = grids(P, bounds, per)
    ob = [("S", ("D", 0.4)), (("D", (0.1, 0.2, 0.3)), "S"), ("P", "P")]
    pb = P.BoundarySpec([(P.Symmetric(), P.Dirichlet(0.4)),
                         (P.Dirichlet((0.1, 0.2, 0.3)), P.Symmetric()),
                         (P.Periodic(), P.Periodic())])
    u = [rng.standard_normal(og.ext_shape) for _ in range(3)]
    ud = vel(P, pg, u)
    O.fill_velocity(og, ob, u)
    P.fill_ghosts_velocity(ud, pb)
    got = ud.numpy()
    for a in range(3):
        np.testing.assert_array_equal(got[a], u[a])
    s = rng.standard_normal(og.ext_shape)
    sd = P.ScalarField(pg, s)
    O.fill_scalar(og, ob, s)
    P.fill_ghosts_scalar(sd, pb)
    np.testing.assert_array_equal(sd.numpy(), s)


# ------------------------------------------------------------------ pressure
@pytest.mark.parametrize("name", ["steps3d", "steps3d_f32"])
def test_spectral_projection_and_steps_golden(P, name):
    c = load(name)
    pg, og = grids_from_case(P, c)
    t = tol(pg.dtype)
    bcs = P.BoundarySpec.all_periodic(3)
    setup = P.Setup(pg, bcs, nu=float(c["nu"]), force=tuple(c["force"]), solver="spectral", method="rk4")
    sol = setup.solver.solve(P.ScalarField(pg, c["rhs"]))
    assert rel(sol.numpy()[pg.p_slices()], c["sol"][pg.p_slices()]) <= t
    u = vel(P, pg, [c[f"u{a}"] for a in range(3)])
    pp = P.project_into(u, setup.solver, bcs)
    got = u.numpy()
    for a in range(3):
        assert rel(got[a], c[f"uproj{a}"]) <= t
    assert rel(pp.numpy(), c["pproj"]) <= t
    dt = float(c["dt"])
    for tag, tab, meth in (("rk4", P.RK4, "rk4"), ("ssp33", P.SSP33, "ssp33"), ("wray3", P.WRAY3, "wray3")):
        setup.method, setup.tableau = meth, tab
        st = setup.new_state(u0=vel(P, pg, [c[f"uproj{a}"] for a in range(3)]))
        if meth == "wray3":
            P.wray3_step(st, dt, setup.solver, setup)
        else:
            P.rk_step(st, dt, tab, setup.solver, setup)
        got = st.u.numpy()
        for a in range(3):
            assert rel(got[a], c[f"{tag}_u{a}"]) <= t, (tag, a)
        if pg.dtype == np.float64:
            assert rel(st.pressure.numpy(), c[f"{tag}_p"]) <= t, tag
        else:
            # fp32: this pressure is ~1e-3 of the velocity (a nearly projected
            # field), so the reference's own fp32 rounding puts it 6.4e-6 (wray3)
            # from the exact result; two fp32 implementations can then differ
            # by ~2x that.  The north-star bar is applied against the reference
            # evaluated in fp64 on the same fp32 initial field.
            truth = _fp64_truth(c, tag, og)
            assert rel(st.pressure.numpy(), truth) <= t, tag
            assert rel(st.pressure.numpy(), c[f"{tag}_p"]) <= 2 * t, tag


def _fp64_truth(c, tag, og):
    g64 = O.OGrid([np.asarray(c[f"bounds{a}"]) for a in range(3)], (True,) * 3, np.float64)
    bcs = O.periodic_bcs(3)
    u = [np.asarray(c[f"uproj{a}"], dtype=np.float64) for a in range(3)]
    args = (float(c["dt"]),)
    if tag == "wray3":
        _, p = O.wray3_step(g64, bcs, O.SpectralSolve(g64), u, *args, float(c["nu"]), tuple(c["force"]))
    else:
        _, p = O.rk_step(g64, bcs, O.SpectralSolve(g64), u, *args, O.RK4 if tag == "rk4" else O.SSP33,
                         float(c["nu"]), tuple(c["force"]))
    return p


@pytest.mark.parametrize("shape", [(6, 10, 14), (20, 12, 30), (42, 8, 16), (64, 64, 64), (7, 9, 5),
                                   (105, 6, 8), (48, 40, 840), (40, 30), (56, 22)])
@pytest.mark.parametrize("force_cufft", [False, True])
def test_spectral_solve_sizes(P, shape, force_cufft, monkeypatch):
    """Hand-written FFT engine (radices 8/4/2/7/5/3, real trick on the last
    axis) and the cuFFT fallback against scipy's rfftn solve (poisson.py:194-200)."""
    if force_cufft:
        monkeypatch.setenv("SFB_FORCE_CUFFT", "1")
    rng = np.random.default_rng(sum(shape))
    bounds = [O.uniform_bounds(0, 1.0 + 0.2 * a, n) for a, n in enumerate(shape)]
    pg, og = grids(P, bounds, (True,) * len(shape))
    solver = P.make_solver("spectral", pg, P.BoundarySpec.all_periodic(len(shape)))
    rhs = og.zeros()
    rhs[og.pdof()] = rng.standard_normal(og.shape)
    rhs[og.pdof()] -= rhs[og.pdof()].mean()
    ref = O.SpectralSolve(og)(rhs[og.pdof()])
    got = solver.solve(P.ScalarField(pg, rhs)).numpy()[pg.p_slices()]
    assert rel(got, ref) <= 1e-12


def test_taylor_green_2d_rk4_golden(P):
    c = load("tg2d_rk4")
    pg, og = grids_from_case(P, c)
    bcs = P.BoundarySpec.all_periodic(2)
    setup = P.Setup(pg, bcs, nu=float(c["nu"]), solver="spectral", method="rk4")
    st = setup.new_state(u0=vel(P, pg, [c["u00"], c["u01"]]))
    P.run_steps(setup, int(c["n_steps"]), dt=float(c["dt"]), state=st)
    got = st.u.numpy()
    for a in range(2):
        assert rel(got[a], c[f"u{a}"]) <= 1e-12
    assert rel(st.pressure.numpy(), c["p"]) <= 1e-12


def test_taylor_green_2d_64_analytic_decay(P):
    """BASELINE config 1: 2D TG 64^2, RK4, 100 steps -> analytic decay."""
    from paper_2604_18536_b200 import cases

    g = cases.taylor_green_grid(64)
    bcs = P.BoundarySpec.all_periodic(2)
    nu = 2e-3
    setup = P.Setup(g, bcs, nu=nu, solver="spectral", method="rk4")
    u0, _ = cases.taylor_green(g, nu, 0.0)
    e0 = P.kinetic_energy(u0)
    st = P.simulate(setup, 1.0, dt=0.01, u0=u0)
    ue, _ = cases.taylor_green(g, nu, 1.0)
    err = cases.l2_error(st.u, ue)
    assert err < 2e-5  # reference measures 1.42e-5
    ratio = P.kinetic_energy(st.u) / e0
    assert abs(ratio - math.exp(-4 * nu)) < 2e-5


def test_channel_golden_direct_solver(P):
    c = load("channel")
    pg, og = grids_from_case(P, c)
    bcs = P.BoundarySpec.channel()
    setup = P.Setup(pg, bcs, nu=float(c["nu"]), force=(1.0, 0.0, 0.0), solver="direct", method="rk4")
    sol = setup.solver.solve(P.ScalarField(pg, c["rhs"]))
    assert rel(sol.numpy()[pg.p_slices()], c["sol"][pg.p_slices()]) <= 1e-12
    u = vel(P, pg, [c[f"u{a}"] for a in range(3)])
    P.fill_ghosts_velocity(u, bcs)
    pp = P.project_into(u, setup.solver, bcs)
    got = u.numpy()
    for a in range(3):
        assert rel(got[a], c[f"uproj{a}"]) <= 1e-12
    assert rel(pp.numpy(), c["pproj"]) <= 1e-12
    for tag, tab, meth in (("rk4", P.RK4, "rk4"), ("ssp33", P.SSP33, "ssp33")):
        setup.method, setup.tableau = meth, tab
        st = setup.new_state(u0=vel(P, pg, [c[f"uproj{a}"] for a in range(3)]))
        P.rk_step(st, float(c["dt"]), tab, setup.solver, setup)
        got = st.u.numpy()
        for a in range(3):
            assert rel(got[a], c[f"{tag}_u{a}"]) <= 1e-12, (tag, a)
        assert rel(st.pressure.numpy(), c[f"{tag}_p"]) <= 1e-12


@pytest.mark.parametrize("shape", [(32, 48, 16), (64, 48, 32), (128, 64, 64)])
def test_channel_step_vs_oracle(P, shape):
    """BASELINE config 4 (reduced): stretched channel, RK4 step vs the
    FFT x tridiagonal oracle."""
    nx, ny, nz = shape
    bounds = [O.uniform_bounds(0, 4 * math.pi, nx), O.tanh_bounds(0, 2.0, ny, 2.0),
              O.uniform_bounds(0, 4 * math.pi / 3, nz)]
    pg, og = grids(P, bounds, (True, False, True))
    ob = O.channel_bcs()
    from paper_2604_18536_b200 import cases

    u0d = cases.channel_ic(pg, 1 / 180.0)
    bcs = P.BoundarySpec.channel()
    P.fill_ghosts_velocity(u0d, bcs)
    setup = P.Setup(pg, bcs, nu=1 / 180.0, force=(1.0, 0.0, 0.0), solver="direct", method="rk4")
    P.project_into(u0d, setup.solver, bcs)
    u0 = u0d.numpy()
    st = setup.new_state(u0=u0d)
    P.rk_step(st, 2e-3, P.RK4, setup.solver, setup)
    ru, rp = O.rk_step(og, ob, ChannelSolve(og), [x.copy() for x in u0], 2e-3, O.RK4, 1 / 180.0, (1.0, 0.0, 0.0))
    got = st.u.numpy()
    for a in range(3):
        assert rel(got[a], ru[a]) <= 1e-12
    assert rel(st.pressure.numpy(), rp) <= 1e-12


# ------------------------------------------------------------------ 3D configs
def test_tgv_128_rhs_and_projection(P):
    """BASELINE config 2: 3D TGV 128^3 fp64, forward RHS + projection."""
    from paper_2604_18536_b200 import cases

    n = 128
    pg = cases.periodic_box(n)
    og = O.OGrid([ax.boundaries for ax in pg.axes], (True,) * 3)
    u = cases.taylor_green_3d(pg)
    un = u.numpy()
    bcs = P.BoundarySpec.all_periodic(3)
    solver = P.make_solver("spectral", pg, bcs)
    nu = 1 / 1600
    ref = O.momentum_rhs(og, un, nu)
    got = P.momentum_rhs(u, nu).numpy()
    for a in range(3):
        assert rel(got[a], ref[a]) <= 1e-12
    rp = O.project_into(og, O.periodic_bcs(3), O.SpectralSolve(og), [x.copy() for x in un])
    pp = P.project_into(u, solver, bcs)
    # TGV is discretely divergence-free: pressure ~ 0; compare velocity
    gu = u.numpy()
    for a in range(3):
        assert rel(gu[a], un[a]) <= 1e-12
    assert np.max(np.abs(pp.numpy() - rp)) <= 1e-12


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_isotropic_rk4_step_vs_oracle(P, dtype):
    """BASELINE config 3 (reduced to 64^3): one RK4 step, u / p / KE."""
    from paper_2604_18536_b200 import cases

    n = 64
    pg = cases.periodic_box(n, dtype=dtype)
    og = O.OGrid([ax.boundaries for ax in pg.axes], (True,) * 3, dtype)
    bcs = P.BoundarySpec.all_periodic(3)
    setup = P.Setup(pg, bcs, nu=1 / 1600, solver="spectral", method="rk4")
    u0d = cases.isotropic(pg, setup.solver, seed=0)
    u0 = u0d.numpy()
    st = setup.new_state(u0=u0d)
    dt = 2e-3
    P.rk_step(st, dt, P.RK4, setup.solver, setup)
    ru, rp = O.rk_step(og, O.periodic_bcs(3), O.SpectralSolve(og), [x.copy() for x in u0], dt, O.RK4, 1 / 1600)
    got = st.u.numpy()
    t = tol(dtype)
    for a in range(3):
        assert rel(got[a], ru[a]) <= t
    assert rel(st.pressure.numpy(), rp) <= t
    ke_ref = O.kinetic_energy(og, ru)
    assert abs(P.kinetic_energy(st.u) - ke_ref) <= t * ke_ref


def test_properties_at_256(P):
    """Size-independent properties at a size the oracle would take minutes:
    projection leaves max|div| at round-off and is idempotent; convection is
    skew-symmetric on the projected field; KE decays under viscosity."""
    import torch
    from paper_2604_18536_b200 import cases

    n = 256
    pg = cases.periodic_box(n)
    bcs = P.BoundarySpec.all_periodic(3)
    setup = P.Setup(pg, bcs, nu=1 / 1600, solver="spectral", method="rk4")
    u = cases.isotropic(pg, setup.solver, seed=1)
    div = P.divergence(u).data
    assert float(div.abs().max()) < 1e-10
    v = u.copy()
    p2 = P.project_into(v, setup.solver, bcs)
    assert float(p2.data.abs().max()) < 1e-12
    conv = P.convection(u)
    skew = P.weighted_inner(u, conv)
    assert abs(skew) <= 1e-12 * P.weighted_inner(u, u) * n
    e0 = P.kinetic_energy(u)
    st = setup.new_state(u0=u)
    P.rk_step(st, 1e-3, P.RK4, setup.solver, setup)
    assert P.kinetic_energy(st.u) < e0
    assert float(P.divergence(st.u).data.abs().max()) < 1e-10
    torch.cuda.synchronize()


# ------------------------------------------------------------------ adjoint
@pytest.mark.parametrize("name", ["ops3d_stretched", "ops3d_uniform", "ops2d_stretched", "ops3d_stretched_f32"])
def test_pullbacks_match_reference_golden(P, name):
    c = load(name)
    pg, og = grids_from_case(P, c)
    d = pg.dim
    t = tol(pg.dtype)
    bcs = P.BoundarySpec.all_periodic(d)
    nu = float(c["nu"])
    cv = lambda: vel(P, pg, [c[f"cv{a}"] for a in range(d)])  # noqa: E731
    dp = P.divergence_pullback(P.ScalarField(pg, c["cs"]), bcs).numpy()
    gp = P.pressure_gradient_pullback(cv(), bcs).numpy()
    fp = P.diffusion_pullback(cv(), nu, bcs).numpy()
    cp = P.convection_pullback(cv(), vel(P, pg, [c[f"u{a}"] for a in range(d)]), bcs).numpy()
    assert rel(gp, c["gradpb"]) <= t
    for a in range(d):
        assert rel(dp[a], c[f"divpb{a}"]) <= t
        assert rel(fp[a], c[f"diffpb{a}"]) <= t
        assert rel(cp[a], c[f"convpb{a}"]) <= t


def test_project_pullback_and_unrolled_gradient_golden(P):
    c = load("adjoint3d")
    pg, og = grids_from_case(P, c)
    bcs = P.BoundarySpec.all_periodic(3)
    setup = P.Setup(pg, bcs, nu=float(c["nu"]), solver="spectral", method="rk4")
    pb = P.project_pullback(vel(P, pg, [c[f"cot{a}"] for a in range(3)]), setup.solver, bcs).numpy()
    for a in range(3):
        assert rel(pb[a], c[f"projpb{a}"]) <= 1e-12
    for n in (1, 2):
        gr = P.unrolled_gradient(P.KineticEnergyLoss(), vel(P, pg, [c[f"u0{a}"] for a in range(3)]), n,
                                 float(c["dt"]), setup).numpy()
        for a in range(3):
            assert rel(gr[a], c[f"grad{n}_{a}"]) <= 1e-12


@pytest.mark.parametrize("n", [32, 128])
@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_unrolled_gradient_vs_oracle(P, dtype, n):
    """BASELINE config 3 VJP (32^3 and 128^3; 512^3 in
    profiles/r2/parity_vjp_512.json): RK4 unrolled gradient of KE, tape +
    reverse sweep, against the oracle's restatement of adjoint.py:425-444."""
    from paper_2604_18536_b200 import cases

    pg = cases.periodic_box(n, dtype=dtype)
    og = O.OGrid([ax.boundaries for ax in pg.axes], (True,) * 3, dtype)
    bcs = P.BoundarySpec.all_periodic(3)
    setup = P.Setup(pg, bcs, nu=1 / 1600, solver="spectral", method="rk4")
    u0d = cases.isotropic(pg, setup.solver, seed=2)
    u0 = u0d.numpy()
    gr = P.unrolled_gradient(P.KineticEnergyLoss(), u0d, 1, 2e-3, setup).numpy()
    ref = O.unrolled_gradient_ke(og, O.periodic_bcs(3), O.SpectralSolve(og), u0, 1, 2e-3, O.RK4, 1 / 1600)
    for a in range(3):
        assert rel(gr[a], ref[a]) <= tol(dtype)


def test_fd_identity_unrolled_gradient(P):
    """checks.py:72-126 protocol: <grad, du> vs centred FD of the loss."""
    from paper_2604_18536_b200 import cases

    pg = cases.periodic_box(16)
    bcs = P.BoundarySpec.all_periodic(3)
    setup = P.Setup(pg, bcs, nu=0.01, solver="spectral", method="rk4")
    u0 = cases.isotropic(pg, setup.solver, seed=4)
    du = cases.isotropic(pg, setup.solver, seed=5)
    loss = P.KineticEnergyLoss()
    g = P.unrolled_gradient(loss, u0, 2, 5e-3, setup)

    def value(eps):
        v = u0.copy()
        for a in range(3):
            v.u[a].add_(du.u[a], alpha=eps)
        st = setup.new_state(u0=v)
        for _ in range(2):
            P.rk_step(st, 5e-3, P.RK4, setup.solver, setup)
        return loss.value(st.u)

    eps = 1e-6
    lhs = (value(eps) - value(-eps)) / (2 * eps)
    rhs = sum(float((g.u[a][pg.u_slices(a)] * du.u[a][pg.u_slices(a)]).sum()) for a in range(3))
    assert abs(lhs - rhs) / abs(rhs) <= 1e-5


def test_tape_primal_matches_in_place_step(P):
    from paper_2604_18536_b200 import cases

    pg = cases.periodic_box(24)
    bcs = P.BoundarySpec.all_periodic(3)
    setup = P.Setup(pg, bcs, nu=0.01, solver="spectral", method="rk4")
    u0 = cases.isotropic(pg, setup.solver, seed=6)
    u1, _ = P.step_forward_tape(u0.copy(), 3e-3, P.RK4, setup.solver, setup)
    st = setup.new_state(u0=u0)
    P.rk_step(st, 3e-3, P.RK4, setup.solver, setup)
    for a in range(3):
        assert rel(u1.numpy()[a], st.u.numpy()[a]) <= 1e-14


def test_no_allocations_per_step(P):
    """Acceptance 11 analogue (test_acceptance.py:407-428)."""
    from paper_2604_18536_b200 import alloc, cases

    pg = cases.periodic_box(16)
    bcs = P.BoundarySpec.all_periodic(3)
    setup = P.Setup(pg, bcs, nu=0.01, solver="spectral", method="rk4")
    st = setup.new_state(u0=cases.taylor_green_3d(pg))
    P.run_steps(setup, 2, dt=1e-3, state=st)
    before = alloc.allocation_count()
    P.run_steps(setup, 50, dt=1e-3, state=st, project_initial=False)
    assert alloc.allocation_count() == before


def test_determinism(P):
    from paper_2604_18536_b200 import cases

    pg = cases.periodic_box(32)
    bcs = P.BoundarySpec.all_periodic(3)
    setup = P.Setup(pg, bcs, nu=0.01, solver="spectral", method="rk4")
    u0 = cases.isotropic(pg, setup.solver, seed=7)
    outs = []
    for _ in range(2):
        st = setup.new_state(u0=u0)
        P.run_steps(setup, 3, dt=2e-3, state=st)
        outs.append(st.u.numpy())
    for a in range(3):
        assert np.array_equal(outs[0][a], outs[1][a])


def test_errors_map_to_reference_exceptions(P):
    g = P.Grid([P.tanh_grid(0, 1, 8, 1.4)] * 3, (True,) * 3)
    bcs = P.BoundarySpec.all_periodic(3)
    with pytest.raises(P.ConfigurationError):
        P.make_solver("spectral", g, bcs)
    with pytest.raises(ValueError):
        P.diffusion(P.VelocityField(g), -1.0)
    assert P.make_solver("cg", g, bcs).kind == "cg"  # stretched periodic: the CG path (row f1)
    with pytest.raises(P.ConfigurationError):
        P.make_solver("nope", g, bcs)
    wall = P.BoundarySpec.channel()
    gw = P.Grid([P.uniform_grid(0, 1, 8), P.uniform_grid(0, 1, 6), P.uniform_grid(0, 1, 4)], (True, False, True))
    setup = P.Setup(gw, wall, nu=0.01, solver="direct", method="rk4")
    with pytest.raises(P.ConfigurationError):
        P.unrolled_gradient(P.KineticEnergyLoss(), P.VelocityField(gw), 1, 0.01, setup)


@pytest.mark.parametrize("shape", [(20, 13, 37), (9, 40, 33), (64, 8, 96)])
@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_rhs_pullback_ragged_tiles_garbage_ghosts(P, shape, dtype):
    """The marching rhs pullback (TMA ring in fp64, wrapped cp.async in fp32)
    on stretched periodic grids whose sizes are not multiples of the tile,
    with random values in the ghost layers of vbar and u: equal to the
    oracle's rhs_pullback (adjoint.py:253-261); vbar's ghosts come back zero
    (adjoint.py:119-136), u keeps its interior."""
    import torch

    rng = np.random.default_rng(sum(shape))
    bounds = [O.tanh_bounds(0.0, 1.0 + 0.2 * a, n, 1.3) for a, n in enumerate(shape)]
    pg, og = grids(P, bounds, (True,) * 3, dtype)
    bcs = P.BoundarySpec.all_periodic(3)
    vb = [rng.standard_normal(og.ext_shape).astype(dtype) for _ in range(3)]
    u = [rng.standard_normal(og.ext_shape).astype(dtype) for _ in range(3)]
    ref = O.rhs_pullback(og, O.periodic_bcs(3), [x.copy() for x in vb], [x.copy() for x in u], 0.013)
    vbd, ud = vel(P, pg, vb), vel(P, pg, u)
    got = P.rhs_pullback(vbd, ud, 0.013, bcs).numpy()
    torch.cuda.synchronize()
    for a in range(3):
        assert rel(got[a], ref[a]) <= tol(dtype)
    vbo, uo = vbd.numpy(), ud.numpy()
    for a in range(3):
        ghost = np.ones(og.ext_shape, bool)
        ghost[1:-1, 1:-1, 1:-1] = False
        assert not np.any(vbo[a][ghost])
        assert np.array_equal(uo[a][1:-1, 1:-1, 1:-1], u[a][1:-1, 1:-1, 1:-1])
