"""One-off parity check at a production size ("parity at 512^3"):
one RK4 step of the GPU path (fp64 and fp32) against the CPU oracle (fp64)
from the same seeded, projected random state.  Run on the GPU box:
    python scripts/parity_full.py 512 > profiles/<round>/parity_512.json
    python scripts/parity_full.py 512 vjp > profiles/<round>/parity_vjp_512.json
The oracle step takes minutes at 512^3 (numpy + scipy.fft on all cores).
The ``vjp`` mode is BASELINE config 3's adjoint: the RK4 unrolled gradient of
the kinetic energy (adjoint.py:425-444, KineticEnergyLoss adjoint.py:276-285)
over one step from an isotropic random-phase state, GPU fp64 and fp32 against
the fp64 oracle."""
import contextlib
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]

from _dev import grids, random_vel, rel, vel  # noqa: E402
from oracle import stagflow_np as O  # noqa: E402


def main_vjp(n):
    import scipy.fft as sfft

    import paper_2604_18536_b200 as P
    from paper_2604_18536_b200 import cases

    nu, dt = 1 / 1600, 2e-3
    out = {"grid": [n, n, n], "mode": "vjp", "method": "rk4", "solver": "spectral", "nu": nu, "dt": dt,
           "loss": "KineticEnergyLoss", "n_steps": 1}
    pg = cases.periodic_box(n)
    setup = P.Setup(pg, P.BoundarySpec.all_periodic(3), nu=nu, solver="spectral", method="rk4")
    u0 = cases.isotropic(pg, setup.solver, seed=2).numpy()
    del setup
    og = O.OGrid([ax.boundaries for ax in pg.axes], (True,) * 3)
    t0 = time.time()
    with sfft.set_workers(os.cpu_count() or 1) if hasattr(sfft, "set_workers") else contextlib.nullcontext():
        ref = O.unrolled_gradient_ke(og, O.periodic_bcs(3), O.SpectralSolve(og), [x.copy() for x in u0],
                                     1, dt, O.RK4, nu)
    out["oracle_s"] = time.time() - t0
    for dtype, tol in ((np.float64, 1e-12), (np.float32, 1e-5)):
        pgt = cases.periodic_box(n, dtype=dtype)
        setup = P.Setup(pgt, P.BoundarySpec.all_periodic(3), nu=nu, solver="spectral", method="rk4")
        gr = P.unrolled_gradient(P.KineticEnergyLoss(), vel(P, pgt, [x.astype(dtype) for x in u0]), 1, dt,
                                 setup).numpy()
        errs = [rel(gr[a][og.udof(a)], ref[a][og.udof(a)]) for a in range(3)]
        key = "f64" if dtype == np.float64 else "f32"
        out[key] = {"rel_err_grad": errs, "tolerance": tol, "pass": bool(max(errs) <= tol)}
        del gr, setup
    import resource

    out["host_peak_rss_gb"] = resource.getrusage(resource.RUSAGE_SELF).ru_maxrss / 1e6
    print(json.dumps(out))


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 512
    if len(sys.argv) > 2 and sys.argv[2] == "vjp":
        return main_vjp(n)
    import scipy.fft as sfft

    import paper_2604_18536_b200 as P

    nu, dt, force = 1 / 1600, 1e-3, (0.3, 0.0, -0.1)
    bounds = [O.uniform_bounds(0.0, 2 * np.pi, n) for _ in range(3)]
    out = {"grid": [n, n, n], "method": "rk4", "solver": "spectral", "nu": nu, "dt": dt, "force": force}
    pg, og = grids(P, bounds, (True,) * 3, np.float64)
    bcs = O.periodic_bcs(3)
    t0 = time.time()
    with sfft.set_workers(os.cpu_count() or 1) if hasattr(sfft, "set_workers") else contextlib.nullcontext():
        u0 = random_vel(og, np.random.default_rng(2024))
        O.fill_velocity(og, bcs, u0)
        solve = O.SpectralSolve(og)
        O.project_into(og, bcs, solve, u0)
        ref_u, ref_p = O.rk_step(og, bcs, solve, [x.copy() for x in u0], dt, O.RK4, nu, force)
    out["oracle_s"] = time.time() - t0
    ref_ke = O.kinetic_energy(og, ref_u) if hasattr(O, "kinetic_energy") else None
    for dtype, tol in ((np.float64, 1e-12), (np.float32, 1e-5)):
        pgt, _ = grids(P, bounds, (True,) * 3, dtype)
        setup = P.Setup(pgt, P.BoundarySpec.all_periodic(3), nu=nu, force=force, solver="spectral", method="rk4")
        st = setup.new_state(u0=vel(P, pgt, [x.astype(dtype) for x in u0]))
        P.rk_step(st, dt, P.RK4, setup.solver, setup)
        u = st.u.numpy()
        errs = [rel(u[a][og.udof(a)], ref_u[a][og.udof(a)]) for a in range(3)]
        ep = rel(st.pressure.numpy()[og.pdof()], ref_p[og.pdof()])
        key = "f64" if dtype == np.float64 else "f32"
        out[key] = {"rel_err_u": errs, "rel_err_p": ep, "tolerance": tol,
                    "pass": bool(max(errs) <= tol and ep <= 10 * tol)}
        if ref_ke is not None:
            ke = P.kinetic_energy(st.u)
            out[key]["ke_rel_err"] = abs(ke - ref_ke) / abs(ref_ke)
        del st, setup
    import resource

    out["host_peak_rss_gb"] = resource.getrusage(resource.RUSAGE_SELF).ru_maxrss / 1e6
    print(json.dumps(out))


if __name__ == "__main__":
    main()
