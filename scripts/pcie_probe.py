"""PCIe copy rates on the box: pinned host <-> HBM, one direction alone and
both directions at once, for a few chunk sizes (the e2e leg of bench.py is
bounded by these).  Prints one JSON line per case."""
import json

import torch


def rate(fn, nbytes, reps=3):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    fn()
    torch.cuda.synchronize()
    best = 0.0
    for _ in range(reps):
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        best = max(best, nbytes / (e0.elapsed_time(e1) * 1e-3) / 1e9)
    return best


def main():
    nb = 4 << 30
    n = nb // 8
    h_in = torch.empty(n, dtype=torch.float64, pin_memory=True)
    h_out = torch.empty(n, dtype=torch.float64, pin_memory=True)
    d_a = torch.empty(n, dtype=torch.float64, device="cuda")
    d_b = torch.empty(n, dtype=torch.float64, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    main_s = torch.cuda.current_stream()
    for chunk_mb in (64, 256, 1024, 4096):
        c = (chunk_mb << 20) // 8
        sl = [slice(i, min(i + c, n)) for i in range(0, n, c)]

        def h2d():
            for s in sl:
                d_a[s].copy_(h_in[s], non_blocking=True)

        def d2h():
            for s in sl:
                h_out[s].copy_(d_b[s], non_blocking=True)

        def both():
            s1.wait_stream(main_s)
            s2.wait_stream(main_s)
            with torch.cuda.stream(s1):
                h2d()
            with torch.cuda.stream(s2):
                d2h()
            main_s.wait_stream(s1)
            main_s.wait_stream(s2)

        print(json.dumps({"chunk_mb": chunk_mb, "h2d_GBs": rate(h2d, nb), "d2h_GBs": rate(d2h, nb),
                          "duplex_each_GBs": rate(both, nb)}), flush=True)


if __name__ == "__main__":
    main()
