import ctypes, sys, os
sys.path.insert(0, '.')
import numpy as np, torch
import paper_2604_18536_b200 as P
from paper_2604_18536_b200 import _native as N
for shape in [(1680, 128, 64), (64, 1680, 64)]:
    b = [P.uniform_grid(0.0, 1.0, n) for n in shape]
    g = P.Grid(b, (True,) * 3)
    s = P.make_solver("spectral", g, P.BoundarySpec.all_periodic(3))
    buf = torch.randn(shape, dtype=torch.float64, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    f = lambda: N.call("sfb_solver_solve", s.handle, buf.data_ptr(), buf.data_ptr(), ctypes.c_void_p(st))
    for _ in range(3): f()
    torch.cuda.synchronize()
    a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(10): f()
    e.record(); torch.cuda.synchronize()
    print(shape, os.environ.get("SFB_FFT_STOCKHAM", "reg"), a.elapsed_time(e) / 10, "ms")
