set -x
timeout 1500 python -m pytest tests -q -m gpu --timeout 900 > gpurun_out/t_all.log 2>&1; tail -5 gpurun_out/t_all.log
timeout 600 python tools/decode_timing.py cfg3 > gpurun_out/decode_timing3.log 2>&1; head -3 gpurun_out/decode_timing3.log
