timeout -s KILL 400 python -m pytest tests/test_gpu_numeric.py -m gpu -q -x -p no:cacheprovider -k "alternate_decode" > gpurun_out/t41.log 2>&1; tail -3 gpurun_out/t41.log
CPCAG_TRACE=1 timeout -s KILL 300 python tools/bench_stages.py > gpurun_out/stages41.log 2>&1; grep -E "decode|kron|fista" gpurun_out/stages41.log | cut -c1-220 | tail -10
