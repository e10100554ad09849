timeout -s KILL 100 python -m pytest tests/test_gpu_numeric.py -m gpu -v -x -p no:cacheprovider > gpurun_out/t_numeric.log 2>&1
timeout -s KILL 60 python -m pytest tests/test_gpu_graph.py -m gpu -v -x -k "gram" > gpurun_out/t_gram.log 2>&1
echo done
