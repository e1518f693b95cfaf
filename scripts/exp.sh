timeout 600 python -m pytest tests/test_distributed_gpu.py -q 2>&1 | tail -2
SFB_SLAB_CHUNKS=1 timeout 600 python -m pytest tests/test_distributed_gpu.py -q 2>&1 | tail -1
SFB_SLAB_CHUNKS=3 timeout 600 python -m pytest tests/test_distributed_gpu.py -q 2>&1 | tail -1
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -1
timeout 300 python bench.py --slab --no-cpu-baseline | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('slab', d['ms_per_step'], d['gpu_launches'])"
