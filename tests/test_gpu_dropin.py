"""GPU parity of the round-2 drop-in surface against golden vectors written by
the reference itself (tests/golden/make_golden_r2.py) and the oracle:

* ``fold_ghosts_velocity`` / ``fold_ghosts_scalar`` (adjoint.py:53-111),
  ``zero_non_dofs_velocity`` / ``zero_ghosts_scalar`` (adjoint.py:32-50);
* spatially varying body forces (``sample_force`` of a callable,
  operators.py:241-259) in ``momentum_rhs`` and in the fused RK4 / generic
  SSP33 stage kernels;
* ``solver="direct"`` on every layout (poisson.py:203-229);
* ``poisson_solve_transpose`` (adjoint.py:236-250).
"""

import numpy as np
import pytest

from _dev import grids, rel, tol, vel
from _golden import load, sides_bcs
from oracle import stagflow_np as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    import paper_2604_18536_b200 as P

    return P


def _pbcs(P, case):
    out = []
    for lo, hi in sides_bcs(case):
        pair = []
        for s in (lo, hi):
            if s == "P":
                pair.append(P.Periodic())
            elif s == "S":
                pair.append(P.Symmetric())
            else:
                pair.append(P.Dirichlet(s[1]))
        out.append(tuple(pair))
    return P.BoundarySpec(out)


def _grid(P, case, prefix=""):
    dim = int(case[prefix + "dim"])
    bounds = [case[f"{prefix}bounds{a}"] for a in range(dim)]
    per = tuple(bool(p) for p in case[prefix + "periodic"])
    return grids(P, bounds, per, np.dtype(str(case[prefix + "dtype"])))


@pytest.mark.parametrize("name", ["folds3d", "folds2d"])
def test_fold_ghosts_golden_bitwise(P, name):
    c = load(name)
    pg, og = _grid(P, c)
    bcs = _pbcs(P, c)
    d = pg.dim
    v = vel(P, pg, [c[f"v{a}"] for a in range(d)])
    out = P.adjoint.fold_ghosts_velocity(v, bcs)
    assert out is v
    got = v.numpy()
    for a in range(d):
        np.testing.assert_array_equal(got[a], c[f"fv{a}"])
    f = P.ScalarField(pg, c["f"])
    P.adjoint.fold_ghosts_scalar(f, bcs)
    np.testing.assert_array_equal(f.numpy(), c["ff"])


def test_zero_non_dofs_and_ghosts_walls(P):
    rng = np.random.default_rng(21)
    bounds = [O.uniform_bounds(0, 1.0, 6), O.tanh_bounds(0, 2.0, 5, 1.5), O.uniform_bounds(0, 1.0, 4)]
    pg, og = grids(P, bounds, (True, False, True))
    u = [rng.standard_normal(og.ext_shape) for _ in range(3)]
    ud = vel(P, pg, u)
    P.adjoint.zero_non_dofs_velocity(ud)
    ref = O.zero_non_dofs(og, [x.copy() for x in u])
    got = ud.numpy()
    for a in range(3):
        np.testing.assert_array_equal(got[a], ref[a])
    s = rng.standard_normal(og.ext_shape)
    sd = P.ScalarField(pg, s)
    P.adjoint.zero_ghosts_scalar(sd)
    np.testing.assert_array_equal(sd.numpy(), O.zero_ghosts_scalar(og, s.copy()))


def _force_fn(c, *x):
    if c == 0:
        return 0.3 * np.sin(2.0 * np.pi * x[1]) + 0.1 * np.cos(x[0])
    if c == 1:
        return 0.2 * np.cos(2.0 * np.pi * x[0]) * (1.0 + 0.0 * x[1])
    return -0.15 * np.sin(x[0] + x[1]) * np.cos(x[2])


def test_force_field_golden(P):
    """Callable force: sampled arrays identical to the reference's, then
    momentum_rhs, the fused RK4 path and the generic SSP33 path."""
    c = load("force_field")
    pg, og = _grid(P, c)
    sampled = P.operators.sample_force(pg, _force_fn)
    for a in range(3):
        np.testing.assert_array_equal(sampled[a], c[f"force{a}"])
    nu, dt = float(c["nu"]), float(c["dt"])
    u0 = vel(P, pg, [c[f"u0{a}"] for a in range(3)])
    rh = P.momentum_rhs(u0, nu, force=sampled).numpy()
    for a in range(3):
        assert rel(rh[a], c[f"rhs{a}"]) <= 1e-12
    bcs = P.BoundarySpec.all_periodic(3)
    for meth, tab in (("rk4", P.RK4), ("ssp33", P.SSP33)):
        setup = P.Setup(pg, bcs, nu=nu, force=_force_fn, solver="spectral", method=meth)
        st = setup.new_state(u0=vel(P, pg, [c[f"u0{a}"] for a in range(3)]))
        P.rk_step(st, dt, tab, setup.solver, setup)
        got = st.u.numpy()
        for a in range(3):
            assert rel(got[a], c[f"{meth}_u{a}"]) <= 1e-12, (meth, a)
        assert rel(st.pressure.numpy(), c[f"{meth}_p"]) <= 1e-12, meth


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_force_field_rk4_vs_oracle_48(P, dtype):
    """Kolmogorov-type forcing on a 48^3 box through the fused (marching)
    stage kernels, every projection fused, against the oracle."""
    from paper_2604_18536_b200 import cases

    n = 48
    pg = cases.periodic_box(n, dtype=dtype)
    og = O.OGrid([ax.boundaries for ax in pg.axes], (True,) * 3, dtype)
    bcs = P.BoundarySpec.all_periodic(3)
    setup = P.Setup(pg, bcs, nu=1 / 400, force=_force_fn, solver="spectral", method="rk4")
    u0d = cases.isotropic(pg, setup.solver, seed=3)
    u0 = u0d.numpy()
    st = setup.new_state(u0=u0d)
    P.rk_step(st, 2e-3, P.RK4, setup.solver, setup)
    force = P.operators.sample_force(pg, _force_fn)
    ru, rp = O.rk_step(og, O.periodic_bcs(3), O.SpectralSolve(og), [x.copy() for x in u0], 2e-3, O.RK4, 1 / 400,
                       force)
    got = st.u.numpy()
    t = tol(dtype)
    for a in range(3):
        assert rel(got[a], ru[a]) <= t
    assert rel(st.pressure.numpy(), rp) <= t


def test_direct_solver_any_layout_golden(P):
    """solver="direct" on a periodic box (spectral backend: same gauge),
    a stretched periodic box and a 2D cavity with a symmetric side (CG to
    1e-12) against the reference's sparse-LU projection."""
    c = load("direct_any")
    for tag, backend, t in (("box", "spectral", 1e-12), ("strp", "cg", 1e-9), ("cav", "cg", 1e-9)):
        cc = {k[len(tag) + 1:]: v for k, v in c.items() if k.startswith(tag + "_")}
        pg, og = _grid(P, cc)
        bcs = _pbcs(P, cc)
        solver = P.make_solver("direct", pg, bcs)
        assert solver.kind == "direct" and solver.backend == backend
        d = pg.dim
        u = vel(P, pg, [cc[f"u{a}"] for a in range(d)])
        v, p = P.project(u, solver, bcs)
        got = v.numpy()
        for a in range(d):
            assert rel(got[a], cc[f"v{a}"]) <= t, (tag, a)
        assert rel(p.numpy(), cc["p"]) <= t, tag
    # Setup's default solver works on a plain periodic box, as in the reference
    g = P.Grid([P.uniform_grid(0.0, 1.0, 8)] * 3, (True,) * 3)
    assert P.Setup(g, P.BoundarySpec.all_periodic(3)).solver.backend == "spectral"


def test_solve_transpose_golden(P):
    c = load("solve_transpose")
    for tag, t in (("uni", 1e-12), ("str", 1e-9)):
        cc = {k[4:]: v for k, v in c.items() if k.startswith(tag + "_")}
        pg, og = _grid(P, cc)
        bcs = P.BoundarySpec.all_periodic(3)
        solver = P.make_solver(str(cc["kind"]), pg, bcs)
        out = P.adjoint.poisson_solve_transpose(P.ScalarField(pg, cc["pbar"]), solver)
        assert rel(out.numpy(), cc["out"]) <= t, tag


def test_config_build_setup_channel_rk4(P):
    """a configuration with the B200 keys (run.device,
    solver.kind = fft-tridiag, time.method = rk4) builds the channel setup on
    the device (cli.py:76-110) and steps it."""
    from paper_2604_18536_b200 import cases
    from paper_2604_18536_b200.config import build_setup, parse_config

    cfg = parse_config("[run]\nstudy = channel-smoke\ndevice = cuda:0\n[grid]\ndim = 3\nx_n = 16\ny_n = 24\n"
                       "z_n = 8\ny_kind = tanh\ny_a = 0\ny_b = 2\ny_gamma = 2.0\n[bc]\ny = dirichlet\n"
                       "[physics]\nnu = 0.0055\nforce = constant\n[solver]\nkind = fft-tridiag\n"
                       "[time]\nmethod = rk4\ndt = 0.001\n")
    setup = build_setup(cfg)
    assert setup.solver.kind == "fft-tridiag" and setup.method == "rk4"
    st = setup.new_state(u0=cases.channel_ic(setup.grid, 0.0055, seed=1))
    P.rk_step(st, 1e-3, P.RK4, setup.solver, setup)
    assert float(P.divergence(st.u).data.abs().max()) < 1e-10


def _lid_channel(c, *x):
    t = x[-1]
    return 0.7 * np.cos(3.0 * t) if c == 0 else 0.0 * x[0]


def _lid_cavity(c, *x):
    t = x[-1]
    return np.tanh(5.0 * t) + 0.0 * x[0] if c == 0 else 0.0


@pytest.mark.parametrize("meth", ["rk4", "ssp33", "wray3"])
def test_moving_wall_golden(P, meth):
    """Time-dependent, spatially uniform callable Dirichlet walls
    (fields.py:72-77), re-evaluated at every stage's fill time: an
    oscillating channel wall (direct solver = FFT x tridiagonal) and an
    accelerating cavity lid (direct solver = CG to 1e-12), three steps."""
    c = load("moving_wall")
    dt, nsteps = float(c["dt"]), int(c["nsteps"])
    for tag, lid, t in (("chan", _lid_channel, 1e-11), ("cav", _lid_cavity, 1e-8)):
        cc = {k[len(tag) + 1:]: v for k, v in c.items() if k.startswith(tag + "_")}
        pg, og = _grid(P, cc)
        if tag == "chan":
            bcs = P.BoundarySpec([(P.Periodic(), P.Periodic()), (P.Dirichlet(0.0), P.Dirichlet(lid)),
                                  (P.Periodic(), P.Periodic())])
        else:
            bcs = P.BoundarySpec([(P.Dirichlet(0.0), P.Dirichlet(0.0)), (P.Dirichlet(0.0), P.Dirichlet(lid))])
        d = pg.dim
        setup = P.Setup(pg, bcs, nu=0.05, solver="direct", method=meth)
        st = setup.new_state(u0=vel(P, pg, [cc[f"u0{a}"] for a in range(d)]))
        for _ in range(nsteps):
            if meth == "wray3":
                P.wray3_step(st, dt, setup.solver, setup)
            else:
                P.rk_step(st, dt, setup.tableau, setup.solver, setup)
        assert abs(st.t - float(cc[f"{meth}_t"])) <= 1e-15
        got = st.u.numpy()
        for a in range(d):
            assert rel(got[a], cc[f"{meth}_u{a}"]) <= t, (tag, meth, a)
        assert rel(st.pressure.numpy(), cc[f"{meth}_p"]) <= t, (tag, meth)


def test_moving_wall_simulate_matches_steps(P):
    """simulate/run_steps carry the wall time through (t advances with the
    state): run_steps(3) equals three rk_step calls bit for bit."""
    c = load("moving_wall")
    cc = {k[5:]: v for k, v in c.items() if k.startswith("chan_")}
    pg, og = _grid(P, cc)
    bcs = P.BoundarySpec([(P.Periodic(), P.Periodic()), (P.Dirichlet(0.0), P.Dirichlet(_lid_channel)),
                          (P.Periodic(), P.Periodic())])
    u0 = [cc[f"u0{a}"] for a in range(3)]
    setup = P.Setup(pg, bcs, nu=0.05, solver="direct", method="rk4")
    st = setup.new_state(u0=vel(P, pg, u0))
    for _ in range(3):
        P.rk_step(st, 0.02, setup.tableau, setup.solver, setup)
    st2 = P.run_steps(setup, 3, dt=0.02, u0=vel(P, pg, u0), project_initial=False)
    for x, y in zip(st.u.numpy(), st2.u.numpy()):
        assert np.array_equal(x, y)
    assert rel(st2.u.numpy()[0], cc["rk4_u0"]) <= 1e-11
    assert st2.t == st.t


def test_moving_wall_must_be_uniform(P):
    g = P.Grid([P.uniform_grid(0.0, 1.0, 8), P.tanh_grid(0.0, 1.0, 6, 1.4), P.uniform_grid(0.0, 1.0, 4)],
               (True, False, True))
    bcs = P.BoundarySpec([(P.Periodic(), P.Periodic()),
                          (P.Dirichlet(0.0), P.Dirichlet(lambda c, x, y, z, t: np.sin(x) * (1.0 + t))),
                          (P.Periodic(), P.Periodic())])
    with pytest.raises(P.ConfigurationError, match="uniform"):
        P.Setup(g, bcs, nu=0.05, solver="direct", method="rk4").new_state()
