"""Target for an ncu launch list of one RK4 unrolled-gradient step at n^3
(argv[1], default 512): tape forward + reverse sweep, after one warm-up."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_18536_b200 as P  # noqa: E402
from paper_2604_18536_b200 import cases  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 512
g = cases.periodic_box(n)
setup = P.Setup(g, P.BoundarySpec.all_periodic(3), nu=1 / 1600, solver="spectral", method="rk4")
u0 = cases.isotropic(g, setup.solver, seed=0)
for _ in range(2):
    P.unrolled_gradient(P.KineticEnergyLoss(), u0, 1, 1e-3, setup)
torch.cuda.synchronize()
print("ok")
