timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 300 python bench.py --no-cpu-baseline | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['roofline'])"
SFB_NO_PROJFUSE=1 timeout 300 python bench.py --no-cpu-baseline | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('noproj', d['ms_per_step'])"
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"k_stage|k_rfft|k_grad|k_planes|k_div" -s 60 -c 40 --csv --log-file gpurun_out/nc.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > /dev/null 2>&1; python profiles/parse_launches.py gpurun_out/nc.csv | head -20
