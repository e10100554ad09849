timeout -s KILL 400 python -m pytest tests/test_gpu_numeric.py tests/test_gpu_graph.py -m gpu -q -x -p no:cacheprovider > gpurun_out/t67.log 2>&1; tail -3 gpurun_out/t67.log
timeout -s KILL 300 python tools/bench_stages.py 2>&1 | grep fista | cut -c1-200
CPCAG_FISTA_TC=0 timeout -s KILL 300 python tools/bench_stages.py 2>&1 | grep fista | cut -c1-200
CPCAG_TRACE=1 JIT_N=60 timeout -s KILL 300 python tools/jitter.py > gpurun_out/jit67.log 2>&1
grep "kron ms" gpurun_out/jit67.log | head -1
grep "cpcag trace" gpurun_out/jit67.log | awk '{print $(NF-1), $0}' | sort -rn | head -10
