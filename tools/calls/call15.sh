set -x
timeout 600 python tools/decode_timing.py cfg3 > gpurun_out/decode_timing3.log 2>&1; head -1 gpurun_out/decode_timing3.log | cut -c1-300
