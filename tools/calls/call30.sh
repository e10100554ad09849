O=gpurun_out/c30
mkdir -p $O
timeout -s KILL 900 python tools/decode_timing.py cfg3 > $O/plain.log 2>&1 && \
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:"^lr_col_k" -s 4 -c 1 -o $O/lrcol -f python tools/decode_timing.py cfg3 > $O/ncu.log 2>&1; echo "ncu rc=$?"
