L=paper_2604_18536_b200/libstagflow_b200.so
for v in varlibs/lib_pb_*.so; do
  cp $v $L
  echo "$v $(python bench_extra.py --cases vjp512 2>/dev/null)"
  ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_rhs_pb" -c 8 --csv --log-file gpurun_out/pb.csv python bench_extra.py --cases vjp512 > /dev/null 2>&1
  python profiles/parse_launches.py gpurun_out/pb.csv 2>/dev/null | head -4
done
