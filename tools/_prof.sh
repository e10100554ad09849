timeout -s KILL 600 python -m pytest tests/test_gpu_numeric.py tests/test_gpu_band_apply.py tests/test_sharded.py -m gpu -q -x -p no:cacheprovider > gpurun_out/t76.log 2>&1; tail -2 gpurun_out/t76.log
timeout -s KILL 300 python tools/bench_stages.py 2>&1 | grep -E "decode" | cut -c1-200
