timeout -s KILL 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b48a.log 2>&1; grep "\[bench\]" gpurun_out/b48a.log
timeout -s KILL 600 python -m pytest tests/test_gpu_graph.py -m gpu -q -x -p no:cacheprovider -k "knn or tc or gram" > gpurun_out/t48.log 2>&1; tail -3 gpurun_out/t48.log
timeout -s KILL 600 python bench.py --config cfg2 --steps 2 --warmup 1 > gpurun_out/b48c.log 2>&1; tail -1 gpurun_out/b48c.log | cut -c 500-900
CPCAG_KNN_FILTER=v1 timeout -s KILL 600 python bench.py --config cfg2 --steps 2 --warmup 1 > gpurun_out/b48d.log 2>&1; tail -1 gpurun_out/b48d.log | cut -c 500-900
