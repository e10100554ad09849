timeout -s KILL 300 python -m pytest tests/test_gpu_band_apply.py -m gpu -q -x -p no:cacheprovider > gpurun_out/t32.log 2>&1; tail -2 gpurun_out/t32.log
for cfg in 1,1024,32,1 1,512,16,1; do CPCAG_BAND_PROF=1 SWEEP_ITERS=5 timeout -s KILL 300 python tools/band_sweep.py $cfg 2>&1 | grep -E "band prof|V=" | tail -2; done
CPCAG_BAND_SPLIT=40 CPCAG_BAND_PROF=1 SWEEP_ITERS=5 timeout -s KILL 300 python tools/band_sweep.py 1,1024,32,1 2>&1 | grep -E "band prof|V=" | tail -2
CPCAG_BAND_SPLIT=32 CPCAG_BAND_PROF=1 SWEEP_ITERS=5 timeout -s KILL 300 python tools/band_sweep.py 1,1024,32,1 2>&1 | grep -E "band prof|V=" | tail -2
