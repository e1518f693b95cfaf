# try row-pass CTA geometries (prebuilt variants in varlibs/) on the 840^3 step
set -x
L=paper_2604_18536_b200/libstagflow_b200.so
mkdir -p gpurun_out
for v in varlibs/lib_*.so; do
  cp $v $L
  echo "== $v"
  python bench.py --steps 6 --warmup 3 --no-cpu-baseline --e2e-steps 1 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.readlines()[-1]); print('ms', d['ms_per_step'])"
  ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_rfft_r2c|k_rfft_c2r" -c 8 --csv --log-file gpurun_out/rv.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 1 > /dev/null 2>&1
  python profiles/parse_launches.py gpurun_out/rv.csv | head -4
done
