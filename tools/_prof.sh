timeout -s KILL 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/t77.log 2>&1; tail -3 gpurun_out/t77.log
timeout -s KILL 600 python bench.py --config cfg3 --steps 2 --warmup 1 > gpurun_out/b77.log 2>&1; tail -1 gpurun_out/b77.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['kernel_ms_per_launch'])"
