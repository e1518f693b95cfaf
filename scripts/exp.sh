timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 300 python bench.py --no-cpu-baseline | cut -c1-400
SFB_NO_DIVFUSE=1 timeout 300 python bench.py --no-cpu-baseline | cut -c1-300
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -s 150 -c 60 --csv --log-file gpurun_out/nc.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline > /dev/null 2>&1; python profiles/parse_launches.py gpurun_out/nc.csv | head -14
