# fp32 strided-pass geometry variants (prebuilt in varlibs/)
L=paper_2604_18536_b200/libstagflow_b200.so
for v in varlibs/lib_*.so; do
  cp $v $L
  for n in 840 512; do
    echo "$v n=$n $(python bench.py --n $n --dtype f32 --steps 8 --warmup 3 --no-cpu-baseline --e2e-steps 1 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.readlines()[-1]); print('ms', d['ms_per_step'])")"
  done
  ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_rfft_strided" -c 12 --csv --log-file gpurun_out/fv.csv python bench.py --n 840 --dtype f32 --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 1 > /dev/null 2>&1
  python profiles/parse_launches.py gpurun_out/fv.csv | head -5
done
