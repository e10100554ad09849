CPCAG_TRACE=1 timeout -s KILL 300 python bench.py --config cfg2 --steps 1 --warmup 1 > gpurun_out/b56.log 2>&1; grep -E "trace|\[knn\]" gpurun_out/b56.log | tail -14; tail -1 gpurun_out/b56.log | cut -c1-150
timeout -s KILL 300 python -m pytest tests/test_gpu_graph.py -m gpu -q -x -p no:cacheprovider > gpurun_out/t56.log 2>&1; tail -2 gpurun_out/t56.log
