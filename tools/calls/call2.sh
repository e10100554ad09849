set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_numeric.py tests/test_sharded.py -x -q -m gpu > gpurun_out/t_dec.log 2>&1
tail -5 gpurun_out/t_dec.log
timeout 900 python tools/decode_timing.py > gpurun_out/decode_timing.log 2>&1
tail -12 gpurun_out/decode_timing.log
