set -x
timeout 900 python -m pytest tests/test_gpu_numeric.py tests/test_sharded.py -x -q -m gpu > gpurun_out/t_dec.log 2>&1; tail -2 gpurun_out/t_dec.log
timeout 600 python tools/decode_timing.py cfg3 > gpurun_out/decode_timing3.log 2>&1; head -3 gpurun_out/decode_timing3.log | cut -c1-300
