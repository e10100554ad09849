timeout -s KILL 300 python -m pytest tests/test_gpu_band_apply.py -m gpu -q -x -p no:cacheprovider > gpurun_out/t28.log 2>&1; tail -2 gpurun_out/t28.log
timeout -s KILL 500 python tools/band_sweep.py 1,1024,32,1 1,1024,32,0 4,1024,32,1 5,1024,32,1 2,1024,32,1 3,1024,32,1 1,512,32,1 1,1024,16,1 1,512,16,1 > gpurun_out/sweep28.log 2>&1; cat gpurun_out/sweep28.log | tail -10
