timeout -s KILL 300 python -m pytest tests/test_gpu_band_apply.py tests/test_sharded.py tests/test_gpu_numeric.py -m gpu -q -x -p no:cacheprovider > gpurun_out/t25.log 2>&1; tail -3 gpurun_out/t25.log
timeout -s KILL 400 python bench.py --config cfg3 --steps 2 --warmup 1 > gpurun_out/bench25_cfg3.log 2>&1; tail -1 gpurun_out/bench25_cfg3.log
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:"cg_apply_(band|col)_k" -c 2 -o gpurun_out/band_r1 -f python bench.py --config cfg3 --steps 1 --warmup 1 > gpurun_out/ncu25.log 2>&1; tail -3 gpurun_out/ncu25.log
