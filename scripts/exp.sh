timeout 600 python -m pytest tests -m gpu -q 2>&1 | tail -2
timeout 300 python bench.py --slab --no-cpu-baseline | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('slab', d['ms_per_step'], d['gpu_launches'])"
timeout 300 python bench.py --no-cpu-baseline | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('std', d['ms_per_step'], d['gpu_launches'])"
