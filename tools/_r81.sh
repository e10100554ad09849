timeout 900 python -m pytest tests/test_gpu_graph.py -q -m gpu -x -k "pipeline" 2>&1 | tail -2
timeout 300 python bench.py --no-cpu-baseline 2> /dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'], d['e2e'])"
