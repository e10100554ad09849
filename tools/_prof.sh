timeout -s KILL 300 python -m pytest tests/test_gpu_graph.py -m gpu -q -x -p no:cacheprovider -k "knn or tc or gram" > gpurun_out/t57.log 2>&1; tail -2 gpurun_out/t57.log
CPCAG_KNN_NT=128 CPCAG_TRACE=1 timeout -s KILL 300 python bench.py --config cfg2 --steps 1 --warmup 1 2>&1 | grep -E "filter|\[knn\]" | tail -2
CPCAG_KNN_NT=256 CPCAG_TRACE=1 timeout -s KILL 300 python bench.py --config cfg2 --steps 1 --warmup 1 2>&1 | grep -E "filter|\[knn\]" | tail -2
CPCAG_KNN_NT=256 CPCAG_KNN=tc timeout -s KILL 300 python -m pytest tests/test_gpu_graph.py -m gpu -q -x -p no:cacheprovider -k "knn or tc" > gpurun_out/t57b.log 2>&1; tail -2 gpurun_out/t57b.log
