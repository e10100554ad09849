set -x
python tools/decode_small.py cfg1 fp32 3 > gpurun_out/ds1.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"lc_k" -c 1 -o gpurun_out/prof_lc32 python tools/decode_small.py cfg1 fp32 3 > gpurun_out/ncu1.log 2>&1
python tools/decode_small.py cfg1 fp64 3 > gpurun_out/ds1.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"lc_k" -c 1 -o gpurun_out/prof_lc64 python tools/decode_small.py cfg1 fp64 3 > gpurun_out/ncu1b.log 2>&1
