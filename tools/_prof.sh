timeout -s KILL 300 python -m pytest tests/test_gpu_band_apply.py tests/test_sharded.py tests/test_gpu_numeric.py -m gpu -q -x -p no:cacheprovider > gpurun_out/t26.log 2>&1; tail -3 gpurun_out/t26.log
timeout -s KILL 400 python bench.py --config cfg3 --steps 2 --warmup 1 > gpurun_out/bench26_cfg3.log 2>&1; tail -1 gpurun_out/bench26_cfg3.log | cut -c 700-
CPCAG_BAND_RB=16 timeout -s KILL 400 python bench.py --config cfg3 --steps 2 --warmup 1 > gpurun_out/bench26_cfg3_rb16.log 2>&1; tail -1 gpurun_out/bench26_cfg3_rb16.log | cut -c 700-
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:"cg_apply_(band|col)_k" -c 2 -o gpurun_out/band_r1b -f python bench.py --config cfg3 --steps 1 --warmup 1 > gpurun_out/ncu26.log 2>&1; tail -2 gpurun_out/ncu26.log
