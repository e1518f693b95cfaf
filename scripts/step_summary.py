"""Per-kernel summary of ONE RK4 step from an ncu launch list of
`bench.py --steps 2 --warmup 1` (run_steps): the second timed step, which
starts at the stage-0 launch that applies the previous step's deferred
projection (k_stage_march with FL 126: PER|S|SU0|NEXT|PROJ|U0P) and ends
before the final gradient subtract of run_steps (or the next stage 0)."""
import subprocess
import sys

sys.path.insert(0, "profiles")
import parse_launches as PL  # noqa: E402

k = PL.load(sys.argv[1])
ids = [i for (i, name) in k]
starts = [i for (i, name) in k if "k_stage_march" in name and ", 126," in name]
first = starts[0]
after = [i for (i, name) in k if i > first and ("k_grad_sub" in name or ("k_stage_march" in name and
                                                                          (", 46," in name or ", 126," in name)))]
last = max(i for i in ids if i < after[0])
print(f"# one RK4 step (launch IDs {first}-{last} of {sys.argv[1]}); ncu --metrics "
      "gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none "
      "(serialised, cold-cache: compare shares)")
sys.stdout.flush()
subprocess.run([sys.executable, "profiles/parse_launches.py", sys.argv[1], str(first), str(last)], check=True)
