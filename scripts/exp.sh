timeout 600 python -m pytest tests -m gpu -q -x 2>&1 | tail -1
st() { ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum --clock-control none -k regex:"k_stage" -s 8 -c 8 --csv --log-file gpurun_out/nc.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > /dev/null 2>&1; python profiles/parse_launches.py gpurun_out/nc.csv | head -6; }
st
timeout 300 python bench.py --no-cpu-baseline | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('step', d['ms_per_step'])"
