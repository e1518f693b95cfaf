timeout 600 python -m pytest tests -m gpu -x -q -k "step or rk or smoke or golden" 2>&1 | tail -2
ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum --clock-control none -k regex:"k_stage" -s 8 -c 8 --csv --log-file gpurun_out/nc.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > /dev/null 2>&1; python profiles/parse_launches.py gpurun_out/nc.csv | head -6
