timeout -s KILL 300 python tools/bench_stages.py > gpurun_out/stages40.log 2>&1; cat gpurun_out/stages40.log | cut -c1-200 | tail -8
