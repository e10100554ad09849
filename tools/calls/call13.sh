set -x
python tools/decode_small.py cfg3 fp64 2 > gpurun_out/ds3.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"lc_k|lr_reg" -c 2 -o gpurun_out/prof_cfg3c python tools/decode_small.py cfg3 fp64 2 > gpurun_out/ncu3.log 2>&1
