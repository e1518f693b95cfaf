"""Round-2 golden vectors, produced by running the reference ``stagflow``
(imported from /root/reference/pkg/src) -- run here, in the build container:

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden_r2.py

Cases (each a small .npz next to this script):

* ``folds3d`` / ``folds2d``: ``fold_ghosts_velocity`` / ``fold_ghosts_scalar``
  (adjoint.py:53-111) on random extended arrays (ghosts included) with
  periodic, Dirichlet and symmetric sides mixed per axis.
* ``force_field``: ``sample_force`` of a callable (operators.py:241-259),
  ``momentum_rhs`` with the sampled arrays, and one RK4 / one SSP33 step of a
  ``Setup(force=<callable>)`` (timestep.py:97-137, 175-214).
* ``direct_any``: ``DirectPoissonSolver`` (poisson.py:203-229) on layouts the
  FFT x tridiagonal solver does not cover -- a periodic uniform box, a
  stretched periodic box, a 2D lid-free cavity -- as projections.
* ``solve_transpose``: ``poisson_solve_transpose`` (adjoint.py:236-250) with
  the spectral solver on a uniform box and the direct solver on a stretched
  periodic box.
* ``moving_wall``: time-dependent callable Dirichlet walls (fields.py:72-77,
  evaluated at every stage's fill time, timestep.py:189-209/232-245) -- a 3D
  channel whose top wall oscillates in x and a 2D cavity whose lid
  accelerates -- three RK4, SSP33 and Wray3 steps each.
"""

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
OUT = os.path.dirname(os.path.abspath(__file__))


def force_fn(c, *x):
    """A smooth, spatially varying body force (Kolmogorov-like), component c."""
    if c == 0:
        return 0.3 * np.sin(2.0 * np.pi * x[1]) + 0.1 * np.cos(x[0])
    if c == 1:
        return 0.2 * np.cos(2.0 * np.pi * x[0]) * (1.0 + 0.0 * x[1])
    return -0.15 * np.sin(x[0] + x[1]) * np.cos(x[2])


def lid_channel(c, *x):
    """Top wall of the channel: oscillating streamwise velocity, uniform
    over the wall (last positional argument is the time)."""
    t = x[-1]
    return 0.7 * np.cos(3.0 * t) if c == 0 else 0.0 * x[0]


def lid_cavity(c, *x):
    """Lid of the cavity: a smoothly accelerating tangential velocity."""
    t = x[-1]
    return np.tanh(5.0 * t) + 0.0 * x[0] if c == 0 else 0.0


def main():
    sys.path.insert(0, REF)
    from stagflow import adjoint as adj
    from stagflow import operators as ops, poisson, timestep as ts
    from stagflow.bcs import BoundarySpec, Dirichlet, Periodic, Symmetric
    from stagflow.fields import ScalarField, VelocityField, fill_ghosts_velocity
    from stagflow.grid import Grid, tanh_grid, uniform_grid

    rk4 = ts.ButcherTableau(
        a=((0.0, 0.0, 0.0, 0.0), (0.5, 0.0, 0.0, 0.0), (0.0, 0.5, 0.0, 0.0), (0.0, 0.0, 1.0, 0.0)),
        b=(1.0 / 6.0, 1.0 / 3.0, 1.0 / 3.0, 1.0 / 6.0),
        c=(0.0, 0.5, 0.5, 1.0),
    )

    def grid_meta(grid):
        d = {"dim": grid.dim, "periodic": np.array(grid.periodic), "dtype": str(grid.dtype)}
        for a, ax in enumerate(grid.axes):
            d[f"bounds{a}"] = ax.boundaries
        return d

    def sides(bcs):
        return np.array([[repr(c) for c in sd] for sd in bcs.sides])

    def vel(prefix, v):
        return {f"{prefix}{a}": np.array(v.u[a]) for a in range(len(v.u))}

    def rvel(grid, rng):
        v = VelocityField(grid)
        for a in range(grid.dim):
            sl = grid.u_slices(a)
            v.u[a][sl] = rng.standard_normal(v.u[a][sl].shape)
        return v

    def save(name, **kw):
        np.savez_compressed(os.path.join(OUT, name + ".npz"), **kw)
        print("wrote", name)

    # ---- ghost-fill adjoints, mixed sides
    rng = np.random.default_rng(11)
    for name, shape, bcs in (
        ("folds3d", (6, 5, 4), BoundarySpec([(Periodic(), Periodic()), (Dirichlet(0.0), Symmetric()),
                                             (Symmetric(), Dirichlet(0.0))])),
        ("folds2d", (5, 4), BoundarySpec([(Dirichlet(0.0), Dirichlet(0.0)), (Periodic(), Periodic())])),
    ):
        g = Grid(tuple(tanh_grid(0.0, 1.0 + 0.2 * a, n, 1.3) for a, n in enumerate(shape)), bcs.periodic)
        v = VelocityField(g)
        for a in range(g.dim):
            v.u[a][...] = rng.standard_normal(g.ext_shape)
        f = ScalarField(g)
        f.data[...] = rng.standard_normal(g.ext_shape)
        out = dict(grid_meta(g), sides=sides(bcs))
        out.update(vel("v", v))
        out["f"] = f.data.copy()
        out.update(vel("fv", adj.fold_ghosts_velocity(v, bcs)))
        out["ff"] = adj.fold_ghosts_scalar(f, bcs).data.copy()
        save(name, **out)

    # ---- spatially varying body force
    rng = np.random.default_rng(12)
    g = Grid(tuple(uniform_grid(0.0, 1.0 + 0.3 * a, 8) for a in range(3)), (True,) * 3)
    bcs = BoundarySpec.all_periodic(3)
    sampled = ops.sample_force(g, force_fn)
    u = rvel(g, rng)
    fill_ghosts_velocity(u, bcs)
    solver = poisson.make_solver("spectral", g, bcs)
    u0, _ = poisson.project(u, solver, bcs)
    out = dict(grid_meta(g), nu=0.02, dt=0.01)
    out.update({f"force{a}": sampled[a] for a in range(3)})
    out.update(vel("u0", u0))
    out.update(vel("rhs", ops.momentum_rhs(u0, 0.02, force=sampled)))
    for meth, tab in (("rk4", rk4), ("ssp33", ts.SSP33)):
        setup = ts.Setup(g, bcs, nu=0.02, force=force_fn, solver="spectral", method="ssp33")
        setup.tableau = tab
        st = setup.new_state(u0=u0)
        ts.rk_step(st, 0.01, tab, setup.solver, setup)
        out.update(vel(f"{meth}_u", st.u))
        out[f"{meth}_p"] = st.pressure.data.copy()
    save("force_field", **out)

    # ---- the direct solver on layouts beyond the separable channel
    rng = np.random.default_rng(13)
    out = {}
    cases = (
        ("box", Grid(tuple(uniform_grid(0.0, 1.0 + 0.25 * a, 6) for a in range(3)), (True,) * 3),
         BoundarySpec.all_periodic(3)),
        ("strp", Grid(tuple(tanh_grid(0.0, 1.0 + 0.25 * a, n, 1.3) for a, n in enumerate((6, 5, 4))), (True,) * 3),
         BoundarySpec.all_periodic(3)),
        ("cav", Grid((tanh_grid(0.0, 1.0, 7, 1.5), uniform_grid(0.0, 1.2, 6)), (False, False)),
         BoundarySpec([(Dirichlet(0.0), Dirichlet(0.0)), (Symmetric(), Dirichlet(0.0))])),
    )
    for tag, g, bcs in cases:
        u = rvel(g, rng)
        fill_ghosts_velocity(u, bcs)
        solver = poisson.make_solver("direct", g, bcs)
        v, p = poisson.project(u, solver, bcs)
        out.update({f"{tag}_{k}": val for k, val in grid_meta(g).items()})
        out[f"{tag}_sides"] = sides(bcs)
        out.update(vel(f"{tag}_u", u))
        out.update(vel(f"{tag}_v", v))
        out[f"{tag}_p"] = p.data.copy()
    save("direct_any", **out)

    # ---- poisson_solve_transpose
    rng = np.random.default_rng(14)
    out = {}
    for tag, g, kind in (
        ("uni", Grid(tuple(uniform_grid(0.0, 1.0 + 0.25 * a, 6) for a in range(3)), (True,) * 3), "spectral"),
        ("str", Grid(tuple(tanh_grid(0.0, 1.0 + 0.25 * a, n, 1.3) for a, n in enumerate((6, 5, 4))), (True,) * 3),
         "direct"),
    ):
        bcs = BoundarySpec.all_periodic(3)
        solver = poisson.make_solver(kind, g, bcs)
        pb = ScalarField(g)
        pb.interior[...] = rng.standard_normal(g.shape)
        res = adj.poisson_solve_transpose(pb, solver)
        out.update({f"{tag}_{k}": val for k, val in grid_meta(g).items()})
        out[f"{tag}_kind"] = np.array(kind)
        out[f"{tag}_pbar"] = pb.data.copy()
        out[f"{tag}_out"] = res.data.copy()
    save("solve_transpose", **out)

    # ---- moving (time-dependent, spatially uniform) Dirichlet walls
    rng = np.random.default_rng(15)
    out = {"dt": 0.02, "nsteps": 3}
    cases = (
        ("chan", Grid((uniform_grid(0.0, 2.0, 8), tanh_grid(0.0, 1.0, 6, 1.4), uniform_grid(0.0, 1.0, 4)),
                      (True, False, True)),
         BoundarySpec([(Periodic(), Periodic()), (Dirichlet(0.0), Dirichlet(lid_channel)), (Periodic(), Periodic())])),
        ("cav", Grid((tanh_grid(0.0, 1.0, 7, 1.5), uniform_grid(0.0, 1.2, 6)), (False, False)),
         BoundarySpec([(Dirichlet(0.0), Dirichlet(0.0)), (Dirichlet(0.0), Dirichlet(lid_cavity))])),
    )
    for tag, g, bcs in cases:
        u = rvel(g, rng)
        solver = poisson.make_solver("direct", g, bcs)
        u0, _ = poisson.project(u, solver, bcs, t=0.0)
        out.update({f"{tag}_{k}": val for k, val in grid_meta(g).items()})
        out.update(vel(f"{tag}_u0", u0))
        for meth, tab in (("rk4", rk4), ("ssp33", ts.SSP33), ("wray3", None)):
            setup = ts.Setup(g, bcs, nu=0.05, solver="direct", method="ssp33")
            if tab is not None:
                setup.tableau = tab
            st = setup.new_state(u0=u0)
            for _ in range(out["nsteps"]):
                if tab is None:
                    ts.wray3_step(st, out["dt"], setup.solver, setup)
                else:
                    ts.rk_step(st, out["dt"], tab, setup.solver, setup)
            out.update(vel(f"{tag}_{meth}_u", st.u))
            out[f"{tag}_{meth}_p"] = st.pressure.data.copy()
            out[f"{tag}_{meth}_t"] = st.t
    save("moving_wall", **out)


if __name__ == "__main__":
    main()
