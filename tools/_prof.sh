timeout -s KILL 300 python -m pytest tests/test_gpu_band_apply.py -m gpu -q -x -p no:cacheprovider > gpurun_out/t30.log 2>&1; tail -2 gpurun_out/t30.log
timeout -s KILL 500 python tools/band_sweep.py 1,1024,32,1 1,512,32,1 1,1024,16,1 1,512,16,1 > gpurun_out/sweep30.log 2>&1; cat gpurun_out/sweep30.log | tail -5
CPCAG_BAND_SPLIT=32 timeout -s KILL 500 python tools/band_sweep.py 1,1024,32,1 1,512,16,1 > gpurun_out/sweep30b.log 2>&1; cat gpurun_out/sweep30b.log | tail -2
