"""compute-sanitizer target (memcheck / racecheck / initcheck): small runs of
every native path -- RK4 steps through rk_step and run_steps (fused stage
kernels, on-the-fly and deferred projections, register FFT with the tiled
spectrum), the VJP (tape + backward), the channel (FFT x tridiagonal) and CG
solvers, an LES closure, HostEnsemble's copy streams and the rhs pullback's
TMA ring on a ragged grid.
    compute-sanitizer --tool memcheck python scripts/sanitize.py"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_18536_b200 as P  # noqa: E402
from paper_2604_18536_b200 import cases  # noqa: E402

# periodic RK4 (24^3 lengths use the register FFT engine: 24 = 4 x 6, half 12 -> Stockham)
for n, dt in ((24, np.float64), (32, np.float32)):
    g = cases.periodic_box(n, dtype=dt)
    setup = P.Setup(g, P.BoundarySpec.all_periodic(3), nu=1 / 1600, force=(0.1, 0.0, 0.0), solver="spectral",
                    method="rk4")
    st = setup.new_state(u0=cases.isotropic(g, setup.solver, seed=1))
    P.rk_step(st, 1e-3, P.RK4, setup.solver, setup)
    P.run_steps(setup, 2, dt=1e-3, state=st, project_initial=False)
    gr = P.unrolled_gradient(P.KineticEnergyLoss(), st.u, 1, 1e-3, setup)
    torch.cuda.synchronize()
# channel (FFT x tridiagonal), with and without a closure; CG on a small stretched box
for closure in (None, P.ClosureModel("smagorinsky")):
    setup = cases.channel_setup(16, 24, 8, closure=closure, method="rk4")
    st = setup.new_state()
    P.rk_step(st, 1e-3, P.RK4, setup.solver, setup)
g = cases.channel_grid(8, 12, 8)
setup = P.Setup(g, P.BoundarySpec.channel(dim=3, wall_axis=1), nu=1 / 180, force=(1.0, 0.0, 0.0), solver="cg",
                method="ssp33", solver_max_iter=5000)
st = setup.new_state(u0=cases.channel_ic(g, 1 / 180))
P.rk_step(st, 1e-3, P.SSP33, setup.solver, setup)
torch.cuda.synchronize()
# HostEnsemble: two pinned-host members, copies on their own streams
g = cases.periodic_box(16)
setup = P.Setup(g, P.BoundarySpec.all_periodic(3), nu=1 / 1600, solver="spectral", method="rk4")
host = []
for seed in (1, 2):
    u = cases.isotropic(g, setup.solver, seed=seed)
    host.append([c.cpu().pin_memory() for c in u.u])
ens = P.HostEnsemble(setup, host, chunks=4)
ens.run(2, 1e-3)
ens.synchronize()
# rhs pullback on a ragged stretched grid (TMA ring with out-of-bounds boxes)
g = P.Grid(tuple(P.tanh_grid(0.0, 1.0 + 0.2 * a, n, 1.3) for a, n in enumerate((9, 13, 37))), (True,) * 3)
rng = np.random.default_rng(0)
vb = P.VelocityField(g, [rng.standard_normal(g.ext_shape) for _ in range(3)])
uu = P.VelocityField(g, [rng.standard_normal(g.ext_shape) for _ in range(3)])
P.rhs_pullback(vb, uu, 0.01, P.BoundarySpec.all_periodic(3))
torch.cuda.synchronize()
print("sanitize target ok")
