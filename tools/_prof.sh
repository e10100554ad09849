timeout -s KILL 400 python -m pytest tests/test_gpu_graph.py tests/test_gpu_approx.py -m gpu -q -x -p no:cacheprovider > gpurun_out/t43.log 2>&1; tail -2 gpurun_out/t43.log
timeout -s KILL 300 python tools/bench_stages.py > gpurun_out/stages43.log 2>&1; grep -E "kron" gpurun_out/stages43.log | cut -c1-200
