# ncu --set full (with source) of the stage kernels of one 840^3 RK4 step
# (both run_steps variants: stage 0 applying the deferred projection, stages
# 1-3) and of the spectral-solve passes; digests into $O.
O=gpurun_out/${1:-ncu_stage}
mkdir -p $O
F="ncu --set full --clock-control none --import-source on"
B="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 1"
$F -k regex:"k_stage_march" -s 4 -c 8 -o $O/stage $B > $O/stage.log 2>&1
python profiles/ncu_digest.py $O/stage.ncu-rep > $O/stage_digest.txt 2>&1
ncu -i $O/stage.ncu-rep --page source --csv --print-source sass > $O/stage_source.csv 2>/dev/null
