timeout -s KILL 400 python tools/band_sweep.py 1,1024,32 2,1024,32 3,1024,32 1,512,32 1,512,16 1,1024,16 3,512,16 > gpurun_out/sweep27.log 2>&1; cat gpurun_out/sweep27.log | tail -9
timeout -s KILL 300 python -m pytest tests/test_gpu_band_apply.py -m gpu -q -x -p no:cacheprovider > gpurun_out/t27.log 2>&1; tail -2 gpurun_out/t27.log
