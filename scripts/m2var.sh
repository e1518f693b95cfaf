# axis-0 fused pass occupancy variants (prebuilt in varlibs/)
L=paper_2604_18536_b200/libstagflow_b200.so
for v in varlibs/lib_m2_*.so; do
  cp $v $L
  for a in "840 f64" "512 f64"; do set -- $a
    echo "$v n=$1 $2 $(python bench.py --n $1 --dtype $2 --steps 8 --warmup 3 --no-cpu-baseline --e2e-steps 1 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.readlines()[-1]); print('ms', d['ms_per_step'])")"
    ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_rfft_strided" -c 12 --csv --log-file gpurun_out/mv.csv python bench.py --n $1 --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 1 > /dev/null 2>&1
    python profiles/parse_launches.py gpurun_out/mv.csv | head -5
  done
done
