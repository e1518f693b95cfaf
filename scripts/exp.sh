mkdir -p gpurun_out/p2
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -2 > gpurun_out/p2/pytest_gpu.txt
python -c "
import sys;sys.path.insert(0,'.')
import __graft_entry__ as g; g.smoke()" > gpurun_out/p2/smoke.txt 2>&1
timeout 600 python bench.py > gpurun_out/p2/bench.json 2> gpurun_out/p2/bench.err
timeout 600 python bench.py --slab --no-cpu-baseline > gpurun_out/p2/bench_slab.json 2>/dev/null
timeout 900 python bench_extra.py --cases step512,step512f32,step840f32,vjp512,channel,solve840,solve512,cg128,les_smagorinsky > gpurun_out/p2/bench_extra.jsonl 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/p2/launch_list.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 1 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_stage_march|k_rfft|k_grad_sub" -s 6 -c 7 -o gpurun_out/p2/ncu_full python bench.py --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 1 > gpurun_out/p2/ncu_full.log 2>&1
tail -1 gpurun_out/p2/ncu_full.log; cat gpurun_out/p2/pytest_gpu.txt gpurun_out/p2/smoke.txt
