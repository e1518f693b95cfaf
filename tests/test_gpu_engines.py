"""GPU tests of the fast paths behind the reference API, each against the CPU
oracle and against the slower path it replaces:

* the register-resident FFT engine (sfb_fft_reg.cuh) on every transform
  length class it instantiates, fp64 and fp32, including the 28 x 30 strided
  engine (840) and the 20 x 21 real-trick rows (840 reals);
* the divergence fused into the first FFT pass (poisson.py:321-333);
* the gradient subtract of the intermediate RK projections fused into the next
  stage kernel (timestep.py:198-199 + poisson.py:333-339), which never
  materialises the projected stage state.
"""

import numpy as np
import pytest

from _dev import grids, random_vel, rel, tol, vel
from oracle import stagflow_np as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_2604_18536_b200 as P

    return P


def _solve(P, shape, dtype, monkeypatch, stockham):
    if stockham:
        monkeypatch.setenv("SFB_FFT_STOCKHAM", "1")
    else:
        monkeypatch.delenv("SFB_FFT_STOCKHAM", raising=False)
    rng = np.random.default_rng(sum(shape))
    bounds = [O.uniform_bounds(0, 1.0 + 0.2 * a, n) for a, n in enumerate(shape)]
    pg, og = grids(P, bounds, (True,) * len(shape), dtype)
    solver = P.make_solver("spectral", pg, P.BoundarySpec.all_periodic(len(shape)))
    rhs = og.zeros()
    rhs[og.pdof()] = rng.standard_normal(og.shape)
    rhs[og.pdof()] -= rhs[og.pdof()].mean()
    got = solver.solve(P.ScalarField(pg, rhs)).numpy()[pg.p_slices()]
    og64 = O.OGrid(bounds, (True,) * len(shape), np.float64)
    ref = O.SpectralSolve(og64)(rhs[og.pdof()].astype(np.float64))
    return got, ref


# strided lengths 1680 (40x42), 840 (28x30), 512 (16x32), 420 (20x21), 256, 96, 64, 48, 40;
# real-trick half lengths 420, 256, 128, 48, 24, 20, 16
@pytest.mark.parametrize("shape", [(840, 6, 8), (6, 840, 40), (512, 4, 16), (4, 420, 48), (256, 8, 840),
                                   (96, 64, 512), (48, 40, 32), (840, 32), (1680, 4, 16), (6, 1680, 8)])
@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_register_fft_solve_vs_oracle_and_stockham(P, shape, dtype, monkeypatch):
    got, ref = _solve(P, shape, dtype, monkeypatch, stockham=False)
    assert rel(got, ref) <= (1e-12 if dtype == np.float64 else 1e-5)
    old, _ = _solve(P, shape, dtype, monkeypatch, stockham=True)
    assert rel(got, old) <= (1e-13 if dtype == np.float64 else 1e-5)


@pytest.mark.parametrize("shape", [(840, 6, 8), (6, 840, 40), (96, 64, 512), (48, 40, 32), (20, 24, 420)])
@pytest.mark.parametrize("dtype", [np.float64, np.float32])
@pytest.mark.parametrize("rows_tiled", [False, True])
def test_tiled_spectrum_bitwise_natural(P, shape, dtype, rows_tiled, monkeypatch):
    """The 3D solve's tiled half spectrum (column blocks, fft.cu) -- the
    default hybrid (tiled copy for the strided passes) and the all-tiled
    variant (SFB_FFT_TILED_ROWS) -- runs the same per-column arithmetic as the
    natural layout: bitwise-equal pressure, including ragged last blocks
    (n2/2+1 not a multiple of the block width)."""
    monkeypatch.delenv("SFB_FFT_NATURAL", raising=False)
    if rows_tiled:
        monkeypatch.setenv("SFB_FFT_TILED_ROWS", "1")
    else:
        monkeypatch.delenv("SFB_FFT_TILED_ROWS", raising=False)
    tiled, ref = _solve(P, shape, dtype, monkeypatch, stockham=False)
    monkeypatch.setenv("SFB_FFT_NATURAL", "1")
    nat, _ = _solve(P, shape, dtype, monkeypatch, stockham=False)
    assert np.array_equal(tiled, nat)
    assert rel(tiled, ref) <= (1e-12 if dtype == np.float64 else 1e-5)


def _rk4(P, n, dtype, monkeypatch, env):
    for k in ("SFB_NO_PROJFUSE", "SFB_NO_DIVFUSE"):
        monkeypatch.delenv(k, raising=False)
    for k in env:
        monkeypatch.setenv(k, "1")
    bounds = [O.uniform_bounds(0.0, 1.0 + 0.3 * a, m) for a, m in enumerate(n)]
    pg, og = grids(P, bounds, (True,) * 3, dtype)
    rng = np.random.default_rng(7)
    u0 = random_vel(og, rng)
    O.fill_velocity(og, O.periodic_bcs(3), u0)
    solve = O.SpectralSolve(og)
    O.project_into(og, O.periodic_bcs(3), solve, u0)
    setup = P.Setup(pg, P.BoundarySpec.all_periodic(3), nu=0.02, force=(0.3, 0.0, -0.1), solver="spectral",
                    method="rk4")
    st = setup.new_state(u0=vel(P, pg, u0))
    P.rk_step(st, 2e-3, P.RK4, setup.solver, setup)
    ref_u, ref_p = O.rk_step(og, O.periodic_bcs(3), solve, [x.copy() for x in u0], 2e-3, O.RK4, 0.02,
                             (0.3, 0.0, -0.1))
    return st.u.numpy(), st.pressure.numpy(), ref_u, ref_p


@pytest.mark.parametrize("n", [(24, 20, 40), (40, 33, 48), (16, 16, 840)])
@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_fused_projection_paths(P, n, dtype, monkeypatch):
    """RK4 step with (a) divergence fused into R2C + gradient subtract fused
    into the next stage (default), (b) no stage fusion, (c) no fusion at all:
    all equal the oracle within the north-star tolerance and each other."""
    t = tol(dtype)
    runs = [_rk4(P, n, dtype, monkeypatch, env) for env in ((), ("SFB_NO_PROJFUSE",),
                                                          ("SFB_NO_PROJFUSE", "SFB_NO_DIVFUSE"))]
    for u, p, ref_u, ref_p in runs:
        for a in range(3):
            assert rel(u[a], ref_u[a]) <= t, a
        assert rel(p, ref_p) <= t
    for a in range(3):
        assert rel(runs[0][0][a], runs[2][0][a]) <= t


def test_rk4_step_at_256_cubed_vs_oracle(P, monkeypatch):
    """One full RK4 step at 256^3 fp64 (16.8M cells, every default fusion on)
    against the CPU oracle, cell for cell: parity at a production-sized grid,
    not only at the small golden sizes (the oracle takes ~30 s here)."""
    u, p, ref_u, ref_p = _rk4(P, (256, 256, 256), np.float64, monkeypatch, ())
    for a in range(3):
        assert rel(u[a], ref_u[a]) <= 1e-12, a
    assert rel(p, ref_p) <= 1e-12


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_run_steps_deferred_last_projection(P, dtype):
    """run_steps with a fixed dt leaves each step's last projection to the
    next step's first stage kernel (u0 - G p formed in shared memory and
    written once): the trajectory equals rk_step called step by step and the
    oracle; observers and the returned state see fully projected fields."""
    n = (40, 36, 48)
    bounds = [O.uniform_bounds(0.0, 1.0 + 0.3 * a, m) for a, m in enumerate(n)]
    pg, og = grids(P, bounds, (True,) * 3, dtype)
    rng = np.random.default_rng(9)
    u0 = random_vel(og, rng)
    O.fill_velocity(og, O.periodic_bcs(3), u0)
    solve = O.SpectralSolve(og)
    O.project_into(og, O.periodic_bcs(3), solve, u0)
    setup = P.Setup(pg, P.BoundarySpec.all_periodic(3), nu=0.02, force=(0.3, 0.0, -0.1), solver="spectral",
                    method="rk4")
    dt, K = 2e-3, 4
    st_a = setup.new_state(u0=vel(P, pg, u0))
    for _ in range(K):
        P.rk_step(st_a, dt, P.RK4, setup.solver, setup)
    seen = []

    def obs(s):
        seen.append((s.step, [c.clone() for c in s.u.u], s.pressure.data.clone()))

    st_b = setup.new_state(u0=vel(P, pg, u0))
    P.run_steps(setup, K, dt=dt, state=st_b, project_initial=False, observers=[obs], observer_cadence=3)
    assert st_b._pending is None
    ru = [x.copy() for x in u0]
    t = tol(dtype)
    for k in range(K):
        ru, rp = O.rk_step(og, O.periodic_bcs(3), solve, ru, dt, O.RK4, 0.02, (0.3, 0.0, -0.1))
        if k == 2:
            assert seen and seen[0][0] == 3
            for a in range(3):
                assert rel(seen[0][1][a].cpu().numpy(), ru[a]) <= t
            assert rel(seen[0][2].cpu().numpy(), rp) <= t
    ga, gb = st_a.u.numpy(), st_b.u.numpy()
    for a in range(3):
        assert rel(gb[a], ga[a]) <= t
        assert rel(gb[a], ru[a]) <= t
    assert rel(st_b.pressure.numpy(), rp) <= t
    assert rel(st_b.pressure.numpy(), st_a.pressure.numpy()) <= t
    assert float(P.divergence(st_b.u).data.abs().max()) < (1e-10 if dtype == np.float64 else 1e-3)
    # simulate with a fixed step defers too; adaptive dt never does
    st_c = P.simulate(setup, K * dt, dt=dt, u0=vel(P, pg, u0), project_initial=False)
    for a in range(3):
        assert rel(st_c.u.numpy()[a], ga[a]) <= t
