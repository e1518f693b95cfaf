"""HostEnsemble end-to-end throughput at 840^3 fp64 for a few chunk / member
counts (the e2e leg of bench.py): one JSON line per variant.
    python scripts/e2e_probe.py [n]"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_18536_b200 as P  # noqa: E402
from paper_2604_18536_b200 import cases  # noqa: E402


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 840
    g = cases.periodic_box(n)
    setup = P.Setup(g, P.BoundarySpec.all_periodic(3), nu=1 / 1600, solver="spectral", method="rk4")
    state = setup.new_state(u0=cases.isotropic(g, setup.solver, seed=0))
    ext = state.u.u[0].shape
    hosts = []
    for m in range(3):
        h = [torch.empty(ext, dtype=torch.float64, pin_memory=True) for _ in range(3)]
        for a in range(3):
            h[a].copy_(state.u.u[a])
            if m:
                h[a][1:-1].copy_(torch.roll(h[a][1:-1], m * n // 3, dims=0))
        hosts.append(h)
    torch.cuda.synchronize()
    for members, chunks, rounds in ((2, 8, 10), (2, 4, 10), (2, 16, 10), (3, 8, 7), (2, 8, 20)):
        ens = P.HostEnsemble(setup, hosts[:members], chunks=chunks, state=state)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        ens.run(rounds, 1e-3)
        ens.join()
        e1.record()
        torch.cuda.synchronize()
        steps = members * rounds
        ms = e0.elapsed_time(e1) / steps
        print(json.dumps({"members": members, "chunks_per_component": chunks, "member_steps": steps,
                          "ms_per_member_step": ms, "cell_updates_per_s": n ** 3 / (ms * 1e-3)}), flush=True)
        del ens
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
