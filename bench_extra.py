"""Secondary measurements for the other BASELINE.json configs (not the
driver's bench line): prints one JSON object per case.

  python bench_extra.py [--cases step512,step512f32,step840f32,vjp512,channel]

* stepN / stepNf32 : RK4 step, periodic N^3 (isotropic IC), fp64 / fp32
* vjpN             : unrolled RK4 gradient of the kinetic energy over one
                     step (forward tape + backward), fp64
* channel          : RK4 step of the Re_tau=180 channel (512x256x256,
                     tanh y, FFT(x,z) x tridiagonal(y) pressure)
Device time by CUDA events, median of the timed repetitions.
"""

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)


def _time(fn, reps, warm):
    import torch

    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    ts.sort()
    return ts[len(ts) // 2]


def case_step(n, dtype):
    import numpy as np

    import paper_2604_18536_b200 as P
    from paper_2604_18536_b200 import cases

    g = cases.periodic_box(n, dtype=np.float64 if dtype == "f64" else np.float32)
    setup = P.Setup(g, P.BoundarySpec.all_periodic(3), nu=1 / 1600, solver="spectral", method="rk4")
    st = setup.new_state(u0=cases.isotropic(g, setup.solver, seed=0))
    ms = _time(lambda: P.rk_step(st, 1e-3, P.RK4, setup.solver, setup), 5, 2)
    return {"case": f"rk4 step {n}^3 {dtype}", "ms": ms, "cell_updates_per_s": n**3 / (ms * 1e-3)}


def case_vjp(n):
    import paper_2604_18536_b200 as P
    from paper_2604_18536_b200 import cases

    g = cases.periodic_box(n)
    setup = P.Setup(g, P.BoundarySpec.all_periodic(3), nu=1 / 1600, solver="spectral", method="rk4")
    u0 = cases.isotropic(g, setup.solver, seed=0)
    loss = P.KineticEnergyLoss()
    ms = _time(lambda: P.unrolled_gradient(loss, u0, 1, 1e-3, setup), 3, 1)
    return {"case": f"unrolled RK4 gradient (1 step, tape + backward) {n}^3 f64", "ms": ms,
            "cell_updates_per_s": n**3 / (ms * 1e-3)}


def case_channel(nx=512, ny=256, nz=256):
    import paper_2604_18536_b200 as P
    from paper_2604_18536_b200 import cases

    setup = cases.channel_setup(nx, ny, nz, gamma=2.0, solver="direct", method="rk4")
    st = setup.new_state()
    P.project_into(st.u, setup.solver, setup.bcs)
    ms = _time(lambda: P.rk_step(st, 1e-3, P.RK4, setup.solver, setup), 5, 2)
    return {"case": f"channel Re_tau=180 {nx}x{ny}x{nz} f64 rk4 step (fft-tridiag)", "ms": ms,
            "cell_updates_per_s": nx * ny * nz / (ms * 1e-3)}


def case_solve(n, dtype):
    """Spectral Poisson solve alone (5 FFT passes, in place on the solver's
    contiguous buffer; no copies)."""
    import ctypes

    import numpy as np
    import torch

    import paper_2604_18536_b200 as P
    from paper_2604_18536_b200 import _native as N
    from paper_2604_18536_b200 import cases

    g = cases.periodic_box(n, dtype=np.float64 if dtype == "f64" else np.float32)
    s = P.make_solver("spectral", g, P.BoundarySpec.all_periodic(3))
    buf = torch.randn(g.shape, dtype=torch.float64 if dtype == "f64" else torch.float32, device="cuda")
    st = torch.cuda.current_stream().cuda_stream

    def run():
        N.call("sfb_solver_solve", s.handle, buf.data_ptr(), buf.data_ptr(), ctypes.c_void_p(st))

    ms = _time(run, 10, 3)
    esz = 8 if dtype == "f64" else 4
    half = n * n * (n // 2 + 1) * 2 * esz
    gbytes = (2 * (n**3 * esz + half) + 6 * half) / 1e9  # R2C + C2R + 3 strided passes (r+w)
    return {"case": f"spectral solve {n}^3 {dtype}", "ms": ms, "gb_moved_min": gbytes, "gbs": gbytes / (ms * 1e-3)}


def case_cg(n=256):
    """Matrix-free CG projection + SSP33 step on a tanh-stretched channel-like
    grid (periodic x, walls y, symmetric/wall z): grids the FFT paths do not
    cover."""
    import numpy as np

    import paper_2604_18536_b200 as P
    from paper_2604_18536_b200.grid import tanh_grid, uniform_grid

    g = P.Grid((uniform_grid(0.0, 2.0, n), tanh_grid(0.0, 1.0, n // 2, 1.6), tanh_grid(0.0, 0.7, n // 2, 1.2)),
               (True, False, False))
    bcs = P.BoundarySpec([(P.Periodic(), P.Periodic()), (P.Dirichlet(0.0), P.Dirichlet(0.0)),
                          (P.Symmetric(), P.Dirichlet(0.0))])
    solver = P.make_solver("cg", g, bcs, tol=1e-8, max_iter=20000)
    setup = P.Setup(g, bcs, nu=1e-3, force=(1.0, 0.0, 0.0), solver=solver, method="ssp33")
    rng = np.random.default_rng(0)
    u0 = P.VelocityField(g)
    for a in range(3):
        u0.u[a].copy_(P.VelocityField(g, [rng.standard_normal(g.ext_shape) * 0.1 for _ in range(3)]).u[a])
    P.project_into(u0, solver, bcs)
    st = setup.new_state(u0=u0)
    ms = _time(lambda: P.rk_step(st, 1e-4, P.SSP33, setup.solver, setup), 3, 1)
    cells = int(np.prod(g.shape))
    return {"case": f"SSP33 step, CG pressure (tol 1e-8), stretched {g.shape} periodic/wall/symmetric f64",
            "ms": ms, "cg_iterations_last_solve": solver.iterations, "cell_updates_per_s": cells / (ms * 1e-3)}


def case_les(nx=512, ny=256, nz=256, kind="smagorinsky"):
    """Channel Re_tau=180 RK4 step with an LES closure (les.py): nu_t kernel +
    eddy-stress divergence per stage on top of the RHS (generic k-register
    path), FFT(x,z) x tridiagonal(y) pressure."""
    import paper_2604_18536_b200 as P
    from paper_2604_18536_b200 import cases

    setup = cases.channel_setup(nx, ny, nz, gamma=2.0, solver="direct", method="rk4")
    setup.closure = P.ClosureModel(kind)
    st = setup.new_state()
    P.project_into(st.u, setup.solver, setup.bcs)
    ms = _time(lambda: P.rk_step(st, 1e-3, P.RK4, setup.solver, setup), 5, 2)
    return {"case": f"channel {nx}x{ny}x{nz} f64 rk4 step with {kind} closure", "ms": ms,
            "cell_updates_per_s": nx * ny * nz / (ms * 1e-3)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cases", default="step512,step512f32,step840f32,vjp512,channel")
    args = ap.parse_args()
    for c in args.cases.split(","):
        if c.startswith("step"):
            f32 = c.endswith("f32")
            n = int(c[4:-3] if f32 else c[4:])
            r = case_step(n, "f32" if f32 else "f64")
        elif c.startswith("vjp"):
            r = case_vjp(int(c[3:]))
        elif c.startswith("solve"):
            f32 = c.endswith("f32")
            n = int(c[5:-3] if f32 else c[5:])
            r = case_solve(n, "f32" if f32 else "f64")
        elif c.startswith("les"):
            r = case_les(kind=c[4:] if len(c) > 4 else "smagorinsky")
        elif c.startswith("cg"):
            r = case_cg(int(c[2:]) if len(c) > 2 else 256)
        elif c == "channel":
            r = case_channel()
        else:
            continue
        print(json.dumps(r), flush=True)


if __name__ == "__main__":
    main()
