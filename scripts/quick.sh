# quick GPU iteration: selected tests, bench (no CPU baseline), one-step launch list summary
# usage: bash scripts/quick.sh <tag> [pytest -k expr]
O=gpurun_out/${1:-quick}
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/gpu.txt 2>&1
if [ -n "$2" ]; then timeout 900 python -m pytest tests -m gpu -q -x -k "$2" > $O/pytest.txt 2>&1; tail -3 $O/pytest.txt; fi
timeout 300 python bench.py --no-cpu-baseline > $O/bench.json 2> $O/bench.err; cat $O/bench.json | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('ms/step', d['ms_per_step'], 'value', d['value'], 'frac', d['roofline']['frac'], 'clk', d['clocks'])"
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $O/launch_list.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 1 > /dev/null 2>&1
python scripts/step_summary.py $O/launch_list.csv > $O/step_summary.txt 2>&1; cat $O/step_summary.txt
