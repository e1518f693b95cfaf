"""Per-kernel summary of ONE RK4 step from an ncu launch list of
`bench.py --steps 2 --warmup 1` (run_steps): the second timed step, which
starts at the stage-0 launch that applies the previous step's deferred
projection (k_stage_march with FL_U0P, FL 120 / 126) and ends
before the final gradient subtract of run_steps (or the next stage 0)."""
import subprocess
import sys

sys.path.insert(0, "profiles")
import parse_launches as PL  # noqa: E402

k = PL.load(sys.argv[1])
ids = [i for (i, name) in k]


def fl(name):
    return int(name.split("k_stage_march<")[1].split(",")[4]) if "k_stage_march<" in name else -1


# stage 0 of a step: applies the deferred projection (FL_U0P = 64) or runs on
# a projected state (no FL_PROJ = 16)
starts = [i for (i, name) in k if fl(name) >= 0 and fl(name) & 64]
first = starts[0]
after = [i for (i, name) in k if i > first and ("k_grad_sub" in name or (fl(name) >= 0 and (fl(name) & 64 or
                                                                                             not fl(name) & 16)))]
last = max(i for i in ids if i < after[0])
print(f"# one RK4 step (launch IDs {first}-{last} of {sys.argv[1]}); ncu --metrics "
      "gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none "
      "(serialised, cold-cache: compare shares)")
sys.stdout.flush()
subprocess.run([sys.executable, "profiles/parse_launches.py", sys.argv[1], str(first), str(last)], check=True)
