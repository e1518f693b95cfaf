"""Target for ncu --set full of the spectral-solve passes: two projections of
an n^3 random field (argv[1], default 840) through project_into; profile the
second one's kernels (ncu -k regex:k_rfft -s 5 -c 5)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_18536_b200 as P  # noqa: E402
from paper_2604_18536_b200 import cases  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 840
dtype = sys.argv[2] if len(sys.argv) > 2 else "f64"
import numpy as np  # noqa: E402

grid = cases.periodic_box(n, dtype=np.float64 if dtype == "f64" else np.float32)
bcs = P.BoundarySpec.all_periodic(3)
solver = P.make_solver("spectral", grid, bcs)
u = P.VelocityField(grid)
for c in u.u:
    c.normal_()
for _ in range(2):
    P.project_into(u, solver, bcs)
torch.cuda.synchronize()
print("ok")
