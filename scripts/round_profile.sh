# End-of-round evidence on one B200: GPU tests, smoke, bench (with the CPU
# baseline), the reference arm, extra cases, a one-step ncu launch list and
# ncu --set full digests of each distinct kernel of the step.  Output under
# gpurun_out/$1 (copied to profiles/ by hand; the .ncu-rep files are deleted
# because gpurun merges at most 64 MiB back).
set -x
O=gpurun_out/${1:-rnew}
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,power.limit --format=csv > $O/gpu.txt 2>&1
if [ -z "$SKIP_TESTS" ]; then
  python -m pytest tests -m gpu -q > $O/pytest_gpu.txt 2>&1
  python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.txt 2>&1
fi
python bench.py > $O/bench_840_f64.json 2> $O/bench_840_f64.err
python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_reference.json 2> $O/bench_reference.err
python bench.py --slab --no-cpu-baseline > $O/bench_840_f64_slab_n1.json 2>/dev/null
python bench_extra.py --cases step512,step512f32,step840f32,vjp512,channel,les_smagorinsky,cg128,solve840 > $O/bench_extra.jsonl 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file $O/launch_list.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 1 > /dev/null 2>&1
python scripts/step_summary.py $O/launch_list.csv > $O/launch_list_step_summary.txt
# the timed step of `--steps 1 --warmup 1` starts after 29 stage/FFT launches
# (initial projection + warm-up step); its 4th stage is the 8th stage launch,
# its gradient subtract the 3rd
F="ncu --set full --clock-control none --import-source on"
B="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 1"
$F -k regex:"k_stage_march|k_rfft" -s 29 -c 7 -o $O/full_a $B > /dev/null 2>&1
$F -k regex:"k_stage_march" -s 7 -c 1 -o $O/full_b $B > /dev/null 2>&1
$F -k regex:"k_grad_sub" -s 2 -c 1 -o $O/full_c $B > /dev/null 2>&1
for r in a b c; do python profiles/ncu_digest.py $O/full_$r.ncu-rep; done > $O/ncu_full_digest.txt 2>&1
rm -f $O/*.ncu-rep
