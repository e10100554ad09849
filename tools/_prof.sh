timeout -s KILL 400 python -m pytest tests/test_gpu_approx.py tests/test_gpu_band_apply.py -m gpu -q -x -p no:cacheprovider > gpurun_out/t34.log 2>&1; tail -25 gpurun_out/t34.log
for r in 4 8; do CPCAG_BAND_RPL=$r SWEEP_ITERS=5 timeout -s KILL 300 python tools/band_sweep.py 1,1024,32,1 5,1024,32,1 2>&1 | grep -E "V=" | sed "s/^/RPL=$r /"; done
