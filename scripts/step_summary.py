"""Per-kernel summary of ONE RK4 step from an ncu launch list of
`bench.py --steps 2 --warmup 1`: the step that starts at the second stage-0
launch (k_stage_march with FL 46) and ends before the next one."""
import subprocess
import sys

sys.path.insert(0, "profiles")
import parse_launches as PL  # noqa: E402

k = PL.load(sys.argv[1])
starts = [i for (i, name) in k if "k_stage_march" in name and ", 46," in name]
first, last = starts[1], starts[2] - 1
print(f"# one RK4 step (launch IDs {first}-{last} of {sys.argv[1]}); ncu --metrics "
      "gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none "
      "(serialised, cold-cache: compare shares)")
sys.stdout.flush()
subprocess.run([sys.executable, "profiles/parse_launches.py", sys.argv[1], str(first), str(last)], check=True)
