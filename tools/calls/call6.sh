set -x
python tools/decode_small.py cfg1 fp32 3 > gpurun_out/ds1.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"lc_smem|lr_reg" -c 2 -o gpurun_out/prof_v5 python tools/decode_small.py cfg1 fp32 3 > gpurun_out/ncu1.log 2>&1
timeout 600 python tools/decode_timing.py cfg3 > gpurun_out/decode_timing3.log 2>&1
