timeout -s KILL 600 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/t36.log 2>&1; tail -30 gpurun_out/t36.log | grep -v "^$" | tail -25
timeout -s KILL 400 python bench.py --config cfg3 --steps 2 --warmup 1 > gpurun_out/bench36_cfg3.log 2>&1; tail -1 gpurun_out/bench36_cfg3.log | cut -c 600-
