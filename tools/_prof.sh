timeout -s KILL 150 python -m pytest tests/test_gpu_numeric.py tests/test_sharded.py -m gpu -v -x -p no:cacheprovider > gpurun_out/t_numeric.log 2>&1
timeout -s KILL 60 python -m pytest tests/test_gpu_graph.py -m gpu -v -x -k "gram" -p no:cacheprovider > gpurun_out/t_gram.log 2>&1
timeout -s KILL 120 python -m pytest tests/test_gpu_graph.py -m gpu -v -x -k "not gram" -p no:cacheprovider > gpurun_out/t_graph.log 2>&1
echo done
