"""Instruction mix of the kernels in an `ncu --page source --csv --print-source sass`
export: share of executed warp-instructions and of stall samples per opcode.
    python profiles/sass_mix.py export.csv [kernel-substring] [top]"""
import collections
import csv
import sys


def load(path):
    kern, hdr, data = None, None, collections.defaultdict(list)
    for line in open(path):
        if line.startswith('"Kernel Name"'):
            kern, hdr = line.split('","')[1], None
            continue
        if line.startswith('"Address"'):
            hdr = next(csv.reader([line]))
            continue
        r = next(csv.reader([line]))
        if hdr and len(r) == len(hdr):
            data[kern].append(dict(zip(hdr, r)))
    return data


def main():
    data = load(sys.argv[1])
    want = sys.argv[2] if len(sys.argv) > 2 else ""
    top = int(sys.argv[3]) if len(sys.argv) > 3 else 20
    for k, rows in data.items():
        if want not in k:
            continue
        tot = sum(float(r["Instructions Executed"] or 0) for r in rows)
        cls, st = collections.Counter(), collections.Counter()
        for r in rows:
            op = r["Source"].strip().split()
            o = (op[1] if op and op[0].startswith("@") else (op[0] if op else "?")).split(".")[0]
            cls[o] += float(r["Instructions Executed"] or 0)
            st[o] += float(r["Warp Stall Sampling (All Samples)"] or 0)
        tots = sum(st.values()) or 1.0
        print(f"{k[:100]}\n  executed warp-instructions {tot:.3e}")
        for o, c in cls.most_common(top):
            print(f"   {o:10s} {100 * c / tot:6.1f}%  stall {100 * st[o] / tots:5.1f}%")


if __name__ == "__main__":
    main()
