"""Compact table of profiles/ncu_digest.py outputs: python profiles/digest_table.py digest.txt [...]"""
import sys

KEYS = ["time_ms", "dram_rd_GB", "dram_wr_GB", "dram_pct", "regs", "warps_active_pct", "ipc", "inst", "fp64_pct",
        "st_long_sb", "st_barrier", "st_wait", "st_mio", "st_short_sb", "smem_bank_conf", "lsu_smem_wavefronts"]
for path in sys.argv[1:]:
    print("==", path)
    print("kernel".ljust(34) + "".join(k[:9].rjust(10) for k in KEYS))
    for blk in open(path).read().split("---")[1:]:
        lines = blk.strip().split("\n")
        d = {}
        for ln in lines[1:]:
            p = ln.split()
            if len(p) >= 2:
                d[p[0]] = p[1]
        def fmt(v):
            try:
                return f"{float(v):.4g}"
            except ValueError:
                return v
        print(lines[0].strip()[-32:].ljust(34) + "".join(fmt(d.get(k, "-")).rjust(10) for k in KEYS))
