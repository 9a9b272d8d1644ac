set -u
timeout 300 python -m pytest tests/test_gpu_dense.py tests/test_gpu_golden.py tests/test_gpu_vectors.py -x -q 2>&1 | tail -3
timeout 120 python bench.py --workload c3 --steps 20 --warmup 5 --no-cpu-baseline --stages 2>&1 >/tmp/b.json | head -9
python -c "import json;d=json.loads(open('/tmp/b.json').read().strip().splitlines()[-1]);print('c3 ms',d['ms_per_step'])"
