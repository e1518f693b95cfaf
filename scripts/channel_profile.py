"""Target for an ncu launch list of channel RK4 steps (512x256x256, the
Re_tau=180 case of BASELINE config 4): two warm-up steps, then two steps."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_18536_b200 as P  # noqa: E402
from paper_2604_18536_b200 import cases  # noqa: E402

closure = sys.argv[1] if len(sys.argv) > 1 else None
setup = cases.channel_setup(512, 256, 256, gamma=2.0, solver="direct", method="rk4",
                            closure=P.ClosureModel(closure) if closure else None)
st = setup.new_state()
P.project_into(st.u, setup.solver, setup.bcs)
for _ in range(4):
    P.rk_step(st, 1e-3, P.RK4, setup.solver, setup)
torch.cuda.synchronize()
print("ok")
