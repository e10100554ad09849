timeout -s KILL 300 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/t24.log 2>&1; tail -2 gpurun_out/t24.log
timeout -s KILL 200 python tools/bench_stages.py > gpurun_out/stages24.log 2>&1; cat gpurun_out/stages24.log | cut -c1-200
timeout -s KILL 300 python bench.py --config cfg2 --steps 2 --warmup 1 > gpurun_out/bench24_cfg2.log 2>&1; tail -1 gpurun_out/bench24_cfg2.log
timeout -s KILL 400 python bench.py --config cfg3 --steps 2 --warmup 1 > gpurun_out/bench24_cfg3.log 2>&1; tail -1 gpurun_out/bench24_cfg3.log
