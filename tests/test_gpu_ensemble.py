"""HostEnsemble (paper_2604_18536_b200/ensemble.py): trajectories held in
pinned host memory, uploaded before and read back after every step with the
copies overlapped across members.  Each member must end exactly where
chained ``rk_step`` calls on the device put it (bitwise: same kernels, same
order), and where the oracle's chained steps put it (1e-12)."""

import numpy as np
import pytest

from _dev import cube_bounds, grids, random_vel, rel
from oracle import stagflow_np as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_2604_18536_b200 as P

    return P


def _members(P, pg, og, n, seed):
    import torch

    solve = O.SpectralSolve(og)
    out = []
    for m in range(n):
        u = random_vel(og, np.random.default_rng(seed + m))
        O.fill_velocity(og, O.periodic_bcs(3), u)
        O.project_into(og, O.periodic_bcs(3), solve, u)
        out.append(u)
    host = [[torch.from_numpy(np.ascontiguousarray(c)).pin_memory() for c in u] for u in out]
    return out, host, solve


@pytest.mark.parametrize("n_members,method,dtype", [(1, "rk4", np.float64), (2, "rk4", np.float64),
                                                    (3, "rk4", np.float64), (2, "ssp33", np.float64),
                                                    (2, "wray3", np.float64), (2, "rk4", np.float32)])
def test_host_ensemble_matches_chained_steps(P, n_members, method, dtype):
    import torch

    pg, og = grids(P, cube_bounds(16), (True,) * 3, dtype)
    bcs = P.BoundarySpec.all_periodic(3)
    setup = P.Setup(pg, bcs, nu=0.05, force=(0.1, 0.0, 0.0), solver="spectral", method=method)
    us, host, _ = _members(P, pg, og, n_members, 7)
    dt, nsteps = 0.01, 3
    ens = P.HostEnsemble(setup, host, chunks=3)
    ens.run(nsteps, dt)
    ens.synchronize()
    for m, u in enumerate(us):
        st = setup.new_state(u0=P.VelocityField(pg, u))
        for _ in range(nsteps):
            P.rk_step(st, dt, setup.tableau, setup.solver, setup) if method != "wray3" else \
                P.wray3_step(st, dt, setup.solver, setup)
        torch.cuda.synchronize()
        ref = st.u.numpy()
        for a in range(3):
            got = host[m][a].numpy()
            assert np.array_equal(got[pg.u_slices(a)], ref[a][pg.u_slices(a)]), f"member {m} u{a}"
    assert ens.steps == nsteps


def test_host_ensemble_vs_oracle_and_host_edits(P):
    """Two RK4 members against the oracle; between two runs the host edits
    a member's interior (a scaled state), which the next upload must honour."""
    pg, og = grids(P, cube_bounds(16), (True,) * 3)
    bcs = P.BoundarySpec.all_periodic(3)
    setup = P.Setup(pg, bcs, nu=0.05, force=(0.1, 0.0, 0.0), solver="spectral", method="rk4")
    us, host, solve = _members(P, pg, og, 2, 11)
    dt = 0.01
    ens = P.HostEnsemble(setup, host, chunks=4)
    ens.run(2, dt)
    ens.synchronize()
    for c in host[1]:
        c.mul_(0.5)  # a host-side edit between runs; the oracle restarts from it
    ref1 = [c.numpy().copy() for c in host[1]]
    ens.run(1, dt)
    ens.synchronize()
    # member 0: three chained oracle steps
    u = [x.copy() for x in us[0]]
    for _ in range(3):
        u, _ = O.rk_step(og, O.periodic_bcs(3), solve, u, dt, O.RK4, 0.05, (0.1, 0.0, 0.0))
    for a in range(3):
        assert rel(host[0][a].numpy()[pg.u_slices(a)], u[a][pg.u_slices(a)]) <= 1e-12
    # member 1: one oracle step from the edited host state (ghosts refilled)
    O.fill_velocity(og, O.periodic_bcs(3), ref1)
    v, _ = O.rk_step(og, O.periodic_bcs(3), solve, ref1, dt, O.RK4, 0.05, (0.1, 0.0, 0.0))
    for a in range(3):
        assert rel(host[1][a].numpy()[pg.u_slices(a)], v[a][pg.u_slices(a)]) <= 1e-12


def test_host_ensemble_rejects_pageable_and_bad_shapes(P):
    import torch

    pg, og = grids(P, cube_bounds(8), (True,) * 3)
    setup = P.Setup(pg, P.BoundarySpec.all_periodic(3), nu=0.01, solver="spectral", method="rk4")
    ext = tuple(pg.ext_shape)
    with pytest.raises(P.ConfigurationError):
        P.HostEnsemble(setup, [[torch.zeros(ext, dtype=torch.float64) for _ in range(3)]])
    with pytest.raises(ValueError):
        P.HostEnsemble(setup, [[torch.zeros(ext, dtype=torch.float64).pin_memory() for _ in range(2)]])
    with pytest.raises(ValueError):
        P.HostEnsemble(setup, [[torch.zeros(ext, dtype=torch.float32).pin_memory() for _ in range(3)]])
    with pytest.raises(ValueError):
        P.HostEnsemble(setup, [])


def test_host_ensemble_channel_walls(P):
    """Wall-bounded members (channel, FFT x tridiagonal solver, RK4): the
    ghost refill after each upload applies the wall conditions; equal bit for
    bit to chained rk_step calls."""
    import torch

    from paper_2604_18536_b200 import cases

    setup = cases.channel_setup(16, 12, 8, solver="direct", method="rk4")
    pg = setup.grid
    host = []
    for seed in (1, 2):
        v = cases.channel_ic(pg, setup.nu, force_x=1.0, perturbation=0.1, seed=seed)
        P.project_into(v, setup.solver, setup.bcs)
        host.append([c.cpu().pin_memory() for c in v.u])
    ref_in = [[c.clone() for c in m] for m in host]
    ens = P.HostEnsemble(setup, host, chunks=2)
    ens.run(2, 0.01)
    ens.synchronize()
    for m in range(2):
        st = setup.new_state(u0=P.VelocityField(pg, [c.numpy() for c in ref_in[m]]))
        for _ in range(2):
            P.rk_step(st, 0.01, setup.tableau, setup.solver, setup)
        torch.cuda.synchronize()
        ref = st.u.numpy()
        for a in range(3):
            sl = pg.u_slices(a)
            assert np.array_equal(host[m][a].numpy()[sl], ref[a][sl]), f"member {m} u{a}"
