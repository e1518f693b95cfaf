# End-of-round evidence on one B200: GPU tests, smoke, bench (with the CPU
# baseline), the reference arm, extra cases, a one-step ncu launch list and
# ncu --set full digests of the stage kernels and of the spectral-solve
# passes.  Output under gpurun_out/$1 (summaries copied to profiles/ by hand;
# the .ncu-rep files are deleted because gpurun merges at most 64 MiB back).
set -x
O=gpurun_out/${1:-rnew}
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,power.limit --format=csv > $O/gpu.txt 2>&1
if [ -z "$SKIP_TESTS" ]; then
  timeout 1200 python -m pytest tests -m gpu -q > $O/pytest_gpu.txt 2>&1
  python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.txt 2>&1
fi
timeout 600 python bench.py > $O/bench_840_f64.json 2> $O/bench_840_f64.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_reference.json 2> $O/bench_reference.err
timeout 600 python bench.py --slab --no-cpu-baseline > $O/bench_840_f64_slab_n1.json 2>/dev/null
timeout 1200 python bench_extra.py --cases step512,step512f32,step840f32,vjp512,channel,les_smagorinsky,cg128,solve840 > $O/bench_extra.jsonl 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file $O/launch_list.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 1 > /dev/null 2>&1
python scripts/step_summary.py $O/launch_list.csv > $O/launch_list_step_summary.txt
if [ -z "$SKIP_NCU_FULL" ]; then
  F="ncu --set full --clock-control none --import-source on"
  # the four stage kernels of the second timed run_steps step (FL 126, 58, 58, 50)
  timeout 1500 $F -k regex:"k_stage_march" -s 5 -c 4 -o $O/stage python bench.py --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 1 > /dev/null 2>&1
  python profiles/ncu_digest.py $O/stage.ncu-rep > $O/ncu_stage_digest.txt 2>&1
  timeout 900 $F -k regex:k_rfft -s 5 -c 5 -o $O/solve python scripts/ncu_solve.py 840 > /dev/null 2>&1
  python profiles/ncu_digest.py $O/solve.ncu-rep > $O/ncu_solve_digest.txt 2>&1
  rm -f $O/*.ncu-rep
fi
