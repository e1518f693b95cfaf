"""Generate golden vectors by running the reference ``stagflow`` itself.

Run in the build container (where ``/root/reference`` exists):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

Writes ``tests/golden/<case>.npz``.  Each file holds the inputs (grid
boundaries, periodic flags, dtype, fields, scalars) and the reference's
outputs for that case.  The fixtures are small (<= 8^3) so they travel with
the repo; the GPU box never needs ``/root/reference``.

RK4 is injected through the generic ``rk_step`` with a ``ButcherTableau``
and a 5-register ``Workspace``, no source edits.
"""

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
OUT = os.path.dirname(os.path.abspath(__file__))


def _import():
    sys.path.insert(0, REF)
    import stagflow  # noqa: F401

    return stagflow


def main():
    _import()
    from stagflow import adjoint as adj
    from stagflow import cases, operators as ops, poisson, timestep as ts
    from stagflow.bcs import BoundarySpec
    from stagflow.fields import ScalarField, VelocityField, fill_ghosts_scalar, fill_ghosts_velocity
    from stagflow.grid import Grid, tanh_grid, uniform_grid

    rk4 = ts.ButcherTableau(
        a=((0.0, 0.0, 0.0, 0.0), (0.5, 0.0, 0.0, 0.0), (0.0, 0.5, 0.0, 0.0), (0.0, 0.0, 1.0, 0.0)),
        b=(1.0 / 6.0, 1.0 / 3.0, 1.0 / 3.0, 1.0 / 6.0),
        c=(0.0, 0.5, 0.5, 1.0),
    )

    def mkgrid(shape, stretched, dtype=np.float64, lengths=None, periodic=None):
        axes = []
        for i, n in enumerate(shape):
            ln = 1.0 + 0.3 * i if lengths is None else lengths[i]
            axes.append(tanh_grid(0.0, ln, n, 1.4) if stretched else uniform_grid(0.0, ln, n))
        per = (True,) * len(shape) if periodic is None else periodic
        return Grid(tuple(axes), per, dtype=dtype)

    def rvel(grid, rng):
        v = VelocityField(grid)
        for a in range(grid.dim):
            sl = grid.u_slices(a)
            v.u[a][sl] = rng.standard_normal(v.u[a][sl].shape)
        return v

    def rsca(grid, rng):
        f = ScalarField(grid)
        f.interior[...] = rng.standard_normal(grid.shape)
        return f

    def grid_meta(grid):
        d = {"dim": grid.dim, "periodic": np.array(grid.periodic), "dtype": str(grid.dtype)}
        for a, ax in enumerate(grid.axes):
            d[f"bounds{a}"] = ax.boundaries
        return d

    def vel(prefix, v):
        return {f"{prefix}{a}": np.array(v.u[a]) for a in range(len(v.u))}

    def save(name, **kw):
        np.savez_compressed(os.path.join(OUT, name + ".npz"), **kw)
        print("wrote", name)

    # ---- operator cases (periodic, stretched and uniform, 2D and 3D, fp64/fp32)
    for name, shape, stretched, dtype in (
        ("ops3d_stretched", (6, 5, 4), True, np.float64),
        ("ops3d_uniform", (6, 5, 4), False, np.float64),
        ("ops2d_stretched", (8, 7), True, np.float64),
        ("ops3d_stretched_f32", (6, 5, 4), True, np.float32),
    ):
        rng = np.random.default_rng(7)
        g = mkgrid(shape, stretched, dtype)
        bcs = BoundarySpec.all_periodic(g.dim)
        u = rvel(g, rng)
        fill_ghosts_velocity(u, bcs)
        p = rsca(g, rng)
        fill_ghosts_scalar(p, bcs)
        nu = 0.37
        force = (0.3, -0.2, 0.1)[: g.dim]
        cot_v = rvel(g, rng)
        cot_s = rsca(g, rng)
        out = dict(grid_meta(g), nu=nu, force=np.array(force))
        out.update(vel("u", u))
        out["p"] = p.data.copy()
        out.update(vel("cv", cot_v))
        out["cs"] = cot_s.data.copy()
        out["div"] = ops.divergence(u).data
        out.update(vel("grad", ops.pressure_gradient(p)))
        out.update(vel("diff", ops.diffusion(u, nu)))
        out.update(vel("conv", ops.convection(u)))
        out.update(vel("rhs", ops.momentum_rhs(u, nu, force=ops.sample_force(g, force))))
        out["ke"] = ops.kinetic_energy(u)
        out["cfl"] = ts.cfl_dt(u, nu, g, 0.85, 0.85)
        out.update(vel("divpb", adj.divergence_pullback(ScalarField(g, cot_s.data.copy()), bcs)))
        out["gradpb"] = adj.pressure_gradient_pullback(cot_v.copy(), bcs).data.copy()
        out.update(vel("diffpb", adj.diffusion_pullback(cot_v.copy(), nu, bcs)))
        uc = u.copy()
        out.update(vel("convpb", adj.convection_pullback(cot_v.copy(), uc, bcs)))
        save(name, **out)

    # ---- spectral solve, projection and full steps (uniform periodic 3D)
    for name, dtype in (("steps3d", np.float64), ("steps3d_f32", np.float32)):
        rng = np.random.default_rng(11)
        g = mkgrid((8, 6, 4), False, dtype)
        bcs = BoundarySpec.all_periodic(3)
        nu = 0.05
        force = (0.2, 0.0, -0.1)
        setup = ts.Setup(g, bcs, nu=nu, force=force, solver="spectral", method="ssp33")
        rhs = rsca(g, rng)
        sol = setup.solver.solve(rhs)
        u = rvel(g, rng)
        fill_ghosts_velocity(u, bcs)
        uproj = u.copy()
        pproj = poisson.project_into(uproj, setup.solver, bcs)
        out = dict(grid_meta(g), nu=nu, force=np.array(force), dt=0.01)
        out["rhs"] = rhs.data.copy()
        out["sol"] = sol.data.copy()
        out.update(vel("u", u))
        out.update(vel("uproj", uproj))
        out["pproj"] = pproj.data.copy()
        # one step of each scheme from the projected state
        for tag, meth, tab in (("rk4", "ssp33", rk4), ("ssp33", "ssp33", ts.SSP33), ("wray3", "wray3", None)):
            st = setup.new_state(u0=uproj)
            if tab is rk4:
                st.workspace = ts.Workspace(g, 5)
            if meth == "wray3":
                setup.method = "wray3"
                ts.wray3_step(st, 0.01, setup.solver, setup)
                setup.method = "ssp33"
            else:
                ts.rk_step(st, 0.01, tab, setup.solver, setup)
            out.update(vel(f"{tag}_u", st.u))
            out[f"{tag}_p"] = st.pressure.data.copy()
        save(name, **out)

    # ---- 2D Taylor-Green RK4 steps (config 1 of BASELINE.json, reduced)
    g = cases.taylor_green_grid(16)
    bcs = BoundarySpec.all_periodic(2)
    setup = ts.Setup(g, bcs, nu=2e-3, solver="spectral")
    setup.tableau = rk4
    u0, _ = cases.taylor_green(g, 2e-3, 0.0)
    st = setup.new_state(u0=u0)
    st.workspace = ts.Workspace(g, 5)
    ts.run_steps(setup, 5, dt=0.01, state=st)
    out = dict(grid_meta(g), nu=2e-3, dt=0.01, n_steps=5)
    out.update(vel("u0", u0))
    out.update(vel("u", st.u))
    out["p"] = st.pressure.data.copy()
    save("tg2d_rk4", **out)

    # ---- channel (walls on y): direct solver solve, projection, steps
    setup = cases.channel_setup(8, 6, 4, gamma=2.0, solver="direct")
    g = setup.grid
    bcs = setup.bcs
    rng = np.random.default_rng(5)
    rhs = rsca(g, rng)
    sol = setup.solver.solve(rhs)
    st = setup.new_state()
    u_ic = st.u.copy()
    uproj = st.u.copy()
    pproj = poisson.project_into(uproj, setup.solver, bcs)
    out = dict(grid_meta(g), nu=setup.nu, force=np.array([1.0, 0.0, 0.0]), dt=0.005)
    out["rhs"] = rhs.data.copy()
    out["sol"] = sol.data.copy()
    out.update(vel("u", u_ic))
    out.update(vel("uproj", uproj))
    out["pproj"] = pproj.data.copy()
    out.update(vel("rhs_u", ops.momentum_rhs(uproj, setup.nu, force=setup.force)))
    out.update(vel("diff_u", ops.diffusion(uproj, setup.nu)))
    for tag, tab in (("rk4", rk4), ("ssp33", ts.SSP33)):
        st2 = setup.new_state(u0=uproj)
        st2.workspace = ts.Workspace(g, tab.stages + 1)
        ts.rk_step(st2, 0.005, tab, setup.solver, setup)
        out.update(vel(f"{tag}_u", st2.u))
        out[f"{tag}_p"] = st2.pressure.data.copy()
    save("channel", **out)

    # ---- CG pressure solver (poisson.py:232-308): stretched, mixed boundaries
    from stagflow.bcs import Dirichlet, Periodic, Symmetric

    for name, shape, per, sides in (
        ("cg3d_mixed", (8, 6, 5), (True, False, False),
         [(Periodic(), Periodic()), (Dirichlet(0.3), Dirichlet(-0.2)), (Symmetric(), Dirichlet(0.0))]),
        ("cg2d_stretched", (10, 7), (True, True), [(Periodic(), Periodic()), (Periodic(), Periodic())]),
    ):
        rng = np.random.default_rng(11)
        g = mkgrid(shape, True, periodic=per)
        bcs = BoundarySpec(sides)
        solver = poisson.make_solver("cg", g, bcs, max_iter=1000)
        rhs = rsca(g, rng)
        sol = solver.solve(rhs)
        out = dict(grid_meta(g), sides=np.array([[repr(c) for c in sd] for sd in sides]))
        out["rhs"] = rhs.data.copy()
        out["sol"] = sol.data.copy()
        out["iterations"] = solver.iterations
        out["residual_history"] = np.array(solver.residual_history)
        # one projection and one SSP33 step through the CG solver
        u = rvel(g, rng)
        uproj = u.copy()
        pproj = poisson.project_into(uproj, solver, bcs)
        out.update(vel("u", u))
        out.update(vel("uproj", uproj))
        out["pproj"] = pproj.data.copy()
        setup = ts.Setup(g, bcs, nu=0.03, solver=solver)
        st = setup.new_state(u0=uproj)
        ts.rk_step(st, 0.004, ts.SSP33, setup.solver, setup)
        out.update(vel("ssp33_u", st.u))
        out["ssp33_p"] = st.pressure.data.copy()
        out["nu"] = 0.03
        out["dt"] = 0.004
        save(name, **out)

    # ---- LES closures (les.py): nu_t of every model, eddy-stress divergence,
    # closure in the momentum RHS and in RK steps (periodic and channel walls)
    from stagflow import les

    def les_case(name, g, bcs, solver, u):
        out = dict(grid_meta(g))
        out.update(vel("u", u))
        for kind in les.ClosureModel.KINDS[1:]:
            out[f"nut_{kind}"] = les.ClosureModel(kind).nu_t(u).data.copy()
        nut = les.ClosureModel("smagorinsky", c=0.3).nu_t(u)
        out["nut_in"] = nut.data.copy()
        out.update(vel("esd", les.eddy_stress_divergence(u, nut)))
        cl = les.ClosureModel("vreman")
        out.update(vel("rhs_cl", ops.momentum_rhs(u, 0.01, force=np.array([0.5] + [0.0] * (g.dim - 1)), closure=cl)))
        for tag, tab, kind in (("ssp33", ts.SSP33, "wale"), ("rk4", rk4, "smagorinsky")):
            setup = ts.Setup(g, bcs, nu=0.01, solver=solver, closure=les.ClosureModel(kind))
            st = setup.new_state(u0=u)
            st.workspace = ts.Workspace(g, tab.stages + 1)
            ts.rk_step(st, 0.003, tab, setup.solver, setup)
            out.update(vel(f"{tag}_u", st.u))
            out[f"{tag}_p"] = st.pressure.data.copy()
        st = ts.Setup(g, bcs, nu=0.01, solver=solver, closure=les.ClosureModel("qr"), dt_max=1.0).new_state(u0=u)
        out["adaptive_dt"] = ts._adaptive_dt(st, ts.Setup(g, bcs, nu=0.01, solver=solver,
                                                         closure=les.ClosureModel("qr"), dt_max=1.0))
        save(name, **out)

    for name, shape in (("les3d", (7, 6, 5)), ("les2d", (9, 8))):
        rng = np.random.default_rng(21)
        g = mkgrid(shape, True)
        bcs = BoundarySpec.all_periodic(len(shape))
        u = rvel(g, rng)
        fill_ghosts_velocity(u, bcs)
        les_case(name, g, bcs, poisson.make_solver("cg", g, bcs, tol=1e-13, max_iter=5000), u)
    setup = cases.channel_setup(8, 6, 4, gamma=2.0, solver="direct")
    g = setup.grid
    u = setup.new_state().u.copy()
    poisson.project_into(u, setup.solver, setup.bcs)
    les_case("les_channel", g, setup.bcs, setup.solver, u)

    # ---- channel statistics (stats.py): three snapshots of a channel run
    # with a closure, with and without eddy-viscosity profiles
    from stagflow import stats

    setup = cases.channel_setup(8, 6, 4, gamma=2.0, solver="direct", closure=les.ClosureModel("smagorinsky"))
    st = setup.new_state()
    poisson.project_into(st.u, setup.solver, setup.bcs)
    snaps, nuts = [], []
    for _ in range(3):
        ts.run_steps(setup, 2, dt=0.002, state=st)
        snaps.append(st.u.copy())
        nuts.append(setup.closure.nu_t(st.u))
    out = dict(grid_meta(setup.grid), nu=setup.nu)
    for i, sn in enumerate(snaps):
        out.update(vel(f"snap{i}_", sn))
        out[f"nut{i}"] = nuts[i].data.copy()
    for tag, ns in (("plain", None), ("nut", nuts)):
        prof = stats.accumulate_stats(snaps, setup.bcs, setup.nu, nut_snapshots=ns)
        out[f"{tag}_rows"] = prof.rows()
        out[f"{tag}_u_tau"] = prof.u_tau
    save("stats_channel", **out)
    # the reference's file formats for the same profile / snapshot
    stats.write_profile_csv(os.path.join(OUT, "stats_profile_ref.csv"), prof)
    stats.write_snapshot(os.path.join(OUT, "snapshot_ref"), snaps[0], 0.125)

    # ---- adjoint: project pullback and unrolled gradient (RK4, 1 and 2 steps)
    rng = np.random.default_rng(3)
    g = mkgrid((6, 5, 4), False)
    bcs = BoundarySpec.all_periodic(3)
    setup = ts.Setup(g, bcs, nu=0.05, solver="spectral")
    setup.tableau = rk4
    u = rvel(g, rng)
    fill_ghosts_velocity(u, bcs)
    u0, _ = poisson.project(u, setup.solver, bcs)
    cot = rvel(g, rng)
    out = dict(grid_meta(g), nu=0.05, dt=0.02)
    out.update(vel("u0", u0))
    out.update(vel("cot", cot))
    out.update(vel("projpb", adj.project_pullback(cot.copy(), setup.solver, bcs)))
    for n in (1, 2):
        gr = adj.unrolled_gradient(adj.KineticEnergyLoss(), u0.copy(), n, 0.02, setup)
        out.update(vel(f"grad{n}_", gr))
    save("adjoint3d", **out)


if __name__ == "__main__":
    main()
