timeout -s KILL 300 python tools/bench_stages.py > gpurun_out/stages37.log 2>&1; cat gpurun_out/stages37.log | cut -c1-250 | tail -8
