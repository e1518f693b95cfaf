"""profiles/ncu_summary.json from an ncu launch list of `bench.py --steps 2
--warmup 1` (gpu__time_duration + dram bytes): DRAM traffic per launch of the
stage kernels of one run_steps RK4 step (the step scripts/step_summary.py
picks), the figure bench.py reports as roofline.traffic.
    python scripts/make_ncu_summary.py launch_list.csv source-description"""
import json
import sys

sys.path.insert(0, "profiles")
import parse_launches as PL  # noqa: E402

CELLS = 840 ** 3
# fp64 bytes/cell per stage variant; history form: 120
# (stage 0), 56 (stages 1-2), 178 (stage 3)
ALG = {126: 104, 58: 128, 50: 80, 46: 72, 120: 80, 56: 80, 178: 128, 40: 48}
k = PL.load(sys.argv[1])
ids = [i for (i, n) in k]
start = [i for (i, n) in k if "k_stage_march" in n and int(n.split("k_stage_march<")[1].split(",")[4]) & 64][0]
stages = []
for (i, n), m in k.items():
    if i >= start and "k_stage_march" in n:
        fl = int(n.split("k_stage_march<")[1].split(",")[4])
        if stages and (fl & 64 or not fl & 16):
            break
        stages.append((fl, m.get("dram__bytes_read.sum", 0) + m.get("dram__bytes_write.sum", 0),
                       m.get("gpu__time_duration.sum", 0)))
names = ["stage0", "stage1", "stage2", "stage3"]
out = {
    "source": sys.argv[2] if len(sys.argv) > 2 else sys.argv[1],
    "stage_kernel": {
        "kernel": "k_stage_march<double,TJ,32,CPT,FL,MINB> of one run_steps RK4 step (history form: FL 120 = stage 0 "
                  "applying the deferred projection, 56 = stages 1-2, 178 = stage 3; running-sum form: 126 / 58 / 50)",
        "per_launch_bytes": {f"{nm} (FL{fl})": b for nm, (fl, b, _) in zip(names, stages)},
        "per_launch_ns": {f"{nm} (FL{fl})": t for nm, (fl, _, t) in zip(names, stages)},
        "algorithmic_per_launch_bytes": {f"{nm} (FL{fl})": ALG[fl] * CELLS for nm, (fl, _, _) in zip(names, stages)},
        "dram_bytes_per_launch": sum(b for _, b, _ in stages) / len(stages),
    },
}
json.dump(out, open("profiles/ncu_summary.json", "w"), indent=1)
print(json.dumps(out, indent=1))
