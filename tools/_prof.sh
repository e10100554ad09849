timeout -s KILL 400 python -m pytest tests/test_gpu_numeric.py tests/test_gpu_graph.py -m gpu -q -x -p no:cacheprovider > gpurun_out/t38.log 2>&1; tail -3 gpurun_out/t38.log
timeout -s KILL 300 python tools/bench_stages.py > gpurun_out/stages38.log 2>&1; grep fista gpurun_out/stages38.log | cut -c1-250
CPCAG_FISTA_LIN=0 timeout -s KILL 300 python tools/bench_stages.py > gpurun_out/stages38b.log 2>&1; grep fista gpurun_out/stages38b.log | cut -c1-250
timeout -s KILL 400 python bench.py --steps 5 --warmup 3 > gpurun_out/bench38.log 2>&1; tail -1 gpurun_out/bench38.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['e2e']['value'], d['stage_ms'])"
