"""Pin the CPU oracle against golden vectors produced by the reference itself
(tests/golden/make_golden.py).  CPU only."""

import math

import numpy as np
import pytest

from _golden import load, obcs, ogrid, sides_bcs, vel
from oracle import les_np as LES
from oracle import stagflow_np as O
from oracle.channel_np import ChannelSolve


def _rel(a, b):
    den = max(float(np.max(np.abs(b))), 1e-300)
    return float(np.max(np.abs(np.asarray(a, dtype=np.float64) - b))) / den


OPS = ["ops3d_stretched", "ops3d_uniform", "ops2d_stretched", "ops3d_stretched_f32"]


@pytest.mark.parametrize("name", OPS)
def test_forward_operators_bitwise(name):
    c = load(name)
    g = ogrid(c)
    d = g.dim
    u = vel(c, "u", d)
    nu = float(c["nu"])
    assert np.array_equal(O.divergence(g, u), c["div"])
    gr = O.pressure_gradient(g, c["p"].copy())
    df = O.diffusion(g, u, nu)
    cv = O.convection(g, u)
    rh = O.momentum_rhs(g, u, nu, c["force"])
    for a in range(d):
        assert np.array_equal(gr[a], c[f"grad{a}"])
        assert np.array_equal(df[a], c[f"diff{a}"])
        assert np.array_equal(cv[a], c[f"conv{a}"])
        assert np.array_equal(rh[a], c[f"rhs{a}"])
    assert O.kinetic_energy(g, u) == float(c["ke"])
    assert O.cfl_dt(g, u, nu, 0.85, 0.85) == float(c["cfl"])


@pytest.mark.parametrize("name", OPS)
def test_pullbacks_bitwise(name):
    c = load(name)
    g = ogrid(c)
    d = g.dim
    bcs = O.periodic_bcs(d)
    u = vel(c, "u", d)
    nu = float(c["nu"])
    dp = O.divergence_pullback(g, bcs, c["cs"].copy())
    gp = O.pressure_gradient_pullback(g, bcs, vel(c, "cv", d))
    fp = O.diffusion_pullback(g, bcs, vel(c, "cv", d), nu)
    cp = O.convection_pullback(g, bcs, vel(c, "cv", d), [x.copy() for x in u])
    assert np.array_equal(gp, c["gradpb"])
    for a in range(d):
        assert np.array_equal(dp[a], c[f"divpb{a}"])
        assert np.array_equal(fp[a], c[f"diffpb{a}"])
        assert np.array_equal(cp[a], c[f"convpb{a}"])


@pytest.mark.parametrize("name", ["steps3d", "steps3d_f32"])
def test_spectral_projection_and_steps(name):
    c = load(name)
    g = ogrid(c)
    bcs = O.periodic_bcs(3)
    solve = O.SpectralSolve(g)
    p = g.pdof()
    assert np.array_equal(solve(c["rhs"][p]), c["sol"][p])
    u = vel(c, "u", 3)
    pp = O.project_into(g, bcs, solve, u)
    for a in range(3):
        assert np.array_equal(u[a], c[f"uproj{a}"])
    assert np.array_equal(pp, c["pproj"])
    nu, dt, f = float(c["nu"]), float(c["dt"]), c["force"]
    for tag, tab in (("rk4", O.RK4), ("ssp33", O.SSP33)):
        u1, p1 = O.rk_step(g, bcs, solve, vel(c, "uproj", 3), dt, tab, nu, f)
        for a in range(3):
            assert np.array_equal(u1[a], c[f"{tag}_u{a}"]), tag
        assert np.array_equal(p1, c[f"{tag}_p"])
    u1, p1 = O.wray3_step(g, bcs, solve, vel(c, "uproj", 3), dt, nu, f)
    for a in range(3):
        assert np.array_equal(u1[a], c[f"wray3_u{a}"])
    assert np.array_equal(p1, c["wray3_p"])


def test_taylor_green_2d_rk4_five_steps():
    c = load("tg2d_rk4")
    g = ogrid(c)
    bcs = O.periodic_bcs(2)
    solve = O.SpectralSolve(g)
    u = vel(c, "u0", 2)
    O.fill_velocity(g, bcs, u)
    solve_p = O.project_into(g, bcs, solve, u)  # run_steps projects the IC first
    del solve_p
    for _ in range(int(c["n_steps"])):
        u, p = O.rk_step(g, bcs, solve, u, float(c["dt"]), O.RK4, float(c["nu"]))
    for a in range(2):
        assert np.array_equal(u[a], c[f"u{a}"])
    assert np.array_equal(p, c["p"])


def test_channel_fft_tridiag_matches_reference_direct_solver():
    c = load("channel")
    g = ogrid(c)
    bcs = obcs(g)
    solve = ChannelSolve(g)
    p = g.pdof()
    assert _rel(solve(c["rhs"][p]), c["sol"][p]) < 1e-12
    u = vel(c, "u", 3)
    pp = O.project_into(g, bcs, solve, u)
    for a in range(3):
        assert _rel(u[a], c[f"uproj{a}"]) < 1e-12
    assert _rel(pp, c["pproj"]) < 1e-11
    up = vel(c, "uproj", 3)
    rh = O.momentum_rhs(g, up, float(c["nu"]), c["force"])
    df = O.diffusion(g, up, float(c["nu"]))
    for a in range(3):
        assert np.array_equal(rh[a], c[f"rhs_u{a}"])
        assert np.array_equal(df[a], c[f"diff_u{a}"])
    for tag, tab in (("rk4", O.RK4), ("ssp33", O.SSP33)):
        u1, p1 = O.rk_step(g, bcs, solve, vel(c, "uproj", 3), float(c["dt"]), tab, float(c["nu"]), c["force"])
        for a in range(3):
            assert _rel(u1[a], c[f"{tag}_u{a}"]) < 1e-12
        assert _rel(p1, c[f"{tag}_p"]) < 1e-10


def test_adjoint_project_pullback_and_unrolled_gradient():
    c = load("adjoint3d")
    g = ogrid(c)
    bcs = O.periodic_bcs(3)
    solve = O.SpectralSolve(g)
    pb = O.project_pullback(g, bcs, solve, vel(c, "cot", 3))
    for a in range(3):
        assert np.array_equal(pb[a], c[f"projpb{a}"])
    for n in (1, 2):
        gr = O.unrolled_gradient_ke(g, bcs, solve, vel(c, "u0", 3), n, float(c["dt"]), O.RK4, float(c["nu"]))
        for a in range(3):
            assert np.array_equal(gr[a], c[f"grad{n}_{a}"])


def test_known_answer_stability_polynomial_rk4():
    """test_timestep.py:96-115 restated for RK4 (quartic polynomial)."""
    n, nu, k, dt = 16, 0.35, 2, 0.11
    b = O.uniform_bounds(0.0, 2 * math.pi, n)
    g = O.OGrid([b, b], (True, True))
    bcs = O.periodic_bcs(2)
    h = 2 * math.pi / n
    lam = (2 * math.cos(k * h) - 2) / h**2
    u0 = g.zeros_vel()
    u0[0][...] = np.sin(k * g.xc[1])[None, :]
    O.fill_velocity(g, bcs, u0)
    u1, _ = O.rk_step(g, bcs, O.SpectralSolve(g), u0, dt, O.RK4, nu)
    z = nu * lam * dt
    growth = 1 + z + z**2 / 2 + z**3 / 6 + z**4 / 24
    sl = g.udof(0)
    assert np.allclose(u1[0][sl], growth * u0[0][sl], rtol=1e-12, atol=1e-13)
    assert np.max(np.abs(u1[1][g.udof(1)])) <= 1e-13


def test_known_answer_channel_from_rest():
    """test_cases.py:145-155: channel from rest with nu=0: one step gives u = dt."""
    bx = O.uniform_bounds(0.0, 4 * math.pi, 8)
    by = O.tanh_bounds(0.0, 2.0, 6, 2.0)
    bz = O.uniform_bounds(0.0, 4 * math.pi / 3, 4)
    g = O.OGrid([bx, by, bz], (True, False, True))
    bcs = O.channel_bcs()
    u0 = g.zeros_vel()
    O.fill_velocity(g, bcs, u0)
    dt = 0.01
    u1, _ = O.rk_step(g, bcs, ChannelSolve(g), u0, dt, O.SSP33, 0.0, (1.0, 0.0, 0.0))
    assert np.allclose(u1[0][g.udof(0)], dt, rtol=1e-12)
    assert np.max(np.abs(u1[1][g.udof(1)])) < 1e-14


@pytest.mark.parametrize("name", ["cg3d_mixed", "cg2d_stretched"])
def test_cg_solver_projection_and_step(name):
    """CGSolve restates poisson.py:232-308 (and laplacian_apply poisson.py:43-68):
    same iterations and residual history, same solution, projection and SSP33
    step on a stretched grid with periodic, Dirichlet and symmetric sides."""
    c = load(name)
    g = ogrid(c)
    d = g.dim
    bcs = sides_bcs(c)
    cg = O.CGSolve(g, bcs, max_iter=1000)
    sol = cg(c["rhs"][g.pdof()])
    assert cg.iterations == int(c["iterations"])
    assert np.allclose(cg.residual_history, c["residual_history"], rtol=1e-12, atol=0)
    assert _rel(sol, c["sol"][g.pdof()]) <= 1e-13
    u = vel(c, "u", d)
    p = O.project_into(g, bcs, cg, u)
    for a in range(d):
        assert _rel(u[a], c[f"uproj{a}"]) <= 1e-12
    assert _rel(p, c["pproj"]) <= 1e-12
    u1, p1 = O.rk_step(g, bcs, cg, vel(c, "uproj", d), float(c["dt"]), O.SSP33, float(c["nu"]))
    for a in range(d):
        assert _rel(u1[a], c[f"ssp33_u{a}"]) <= 1e-12
    assert _rel(p1, c["ssp33_p"]) <= 1e-11


LES_MODELS = ["smagorinsky", "vreman", "qr", "wale", "sigma", "s3pqr"]


def _les_closure(kind):
    def add(g, u, out):
        LES.eddy_stress_divergence(g, u, _ext(g, LES.nu_t(g, u, kind)), out=out)

    return add


def _ext(g, interior):
    f = g.zeros()
    f[g.pdof()] = interior
    return f


@pytest.mark.parametrize("name", ["les3d", "les2d", "les_channel"])
def test_les_closures(name):
    """oracle/les_np.py restates les.py: every model's nu_t, the eddy-stress
    divergence, the closure in momentum_rhs and in SSP33 / RK4 steps, the
    closure-tightened adaptive step (timestep.py:259-270)."""
    c = load(name)
    g = ogrid(c)
    d = g.dim
    u = vel(c, "u", d)
    for kind in LES_MODELS:
        got = LES.nu_t(g, u, kind)
        assert _rel(got, c[f"nut_{kind}"][g.pdof()]) <= (1e-14 if kind != "sigma" else 1e-12), kind
    esd = LES.eddy_stress_divergence(g, u, c["nut_in"].copy())
    for a in range(d):
        assert _rel(esd[a], c[f"esd{a}"]) <= 1e-14
    force = [0.5] + [0.0] * (d - 1)
    rhs = O.momentum_rhs(g, u, 0.01, force, _les_closure("vreman"))
    for a in range(d):
        assert _rel(rhs[a], c[f"rhs_cl{a}"]) <= 1e-14
    bcs = obcs(g)
    if name == "les_channel":
        solve = ChannelSolve(g)
        tol = 1e-12
    else:
        solve = O.CGSolve(g, bcs, tol=1e-13, max_iter=5000)
        tol = 1e-9
    for tag, tab, kind in (("ssp33", O.SSP33, "wale"), ("rk4", O.RK4, "smagorinsky")):
        u1, p1 = O.rk_step(g, bcs, solve, vel(c, "u", d), 0.003, tab, 0.01, None, _les_closure(kind))
        for a in range(d):
            assert _rel(u1[a], c[f"{tag}_u{a}"]) <= tol, (tag, a)
    nut = LES.nu_t(g, u, "qr")
    dt = O.cfl_dt(g, u, 0.01 + float(np.max(nut)), 0.85, 0.85)
    assert abs(min(dt, 1.0) - float(c["adaptive_dt"])) <= 1e-15 * dt
