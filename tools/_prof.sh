timeout -s KILL 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/t75.log 2>&1; tail -4 gpurun_out/t75.log
timeout -s KILL 300 python tools/bench_stages.py 2>&1 | grep -E "decode|fista" | cut -c1-200
