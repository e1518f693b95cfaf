"""Summarise an ncu --csv launch list (gpu__time_duration.sum [+ dram bytes])
into per-kernel totals.  Usage: python profiles/parse_launches.py file.csv [first_id]"""
import collections
import csv
import io
import sys


def load(path):
    lines = [l for l in open(path) if not l.startswith("==")]
    rows = list(csv.DictReader(io.StringIO("".join(lines))))
    k = collections.OrderedDict()
    for r in rows:
        key = (int(r["ID"]), r["Kernel Name"])
        v = r["Metric Value"].replace(",", "")
        unit = r.get("Metric Unit", "")
        val = float(v)
        if unit in ("usecond",):
            val *= 1e3
        elif unit in ("msecond",):
            val *= 1e6
        elif unit == "Kbyte":
            val *= 1e3
        elif unit == "Mbyte":
            val *= 1e6
        elif unit == "Gbyte":
            val *= 1e9
        k.setdefault(key, {})[r["Metric Name"]] = val
    return k


def main():
    k = load(sys.argv[1])
    first = int(sys.argv[2]) if len(sys.argv) > 2 else 0
    last = int(sys.argv[3]) if len(sys.argv) > 3 else 10**9
    agg = collections.OrderedDict()
    for (i, name), m in k.items():
        if i < first or i > last:
            continue
        short = name.split("(")[0][:70]
        a = agg.setdefault(short, [0, 0.0, 0.0])
        a[0] += 1
        a[1] += m.get("gpu__time_duration.sum", 0.0)
        a[2] += m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
    tot = sum(a[1] for a in agg.values())
    print(f"{'kernel':72s} {'n':>4s} {'ms':>9s} {'share':>6s} {'GB':>8s} {'GB/s':>7s}")
    for name, (n, ns, b) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{name:72s} {n:4d} {ns / 1e6:9.3f} {ns / tot:6.1%} {b / 1e9:8.2f} {b / max(ns, 1):7.0f}")
    print(f"total {tot / 1e6:.3f} ms")


if __name__ == "__main__":
    main()
