O=gpurun_out/c29
mkdir -p $O
timeout -s KILL 900 python -m pytest tests/test_gpu_numeric.py tests/test_sharded.py -q -x --timeout 600 -k "decode or decoder or shard" > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest.log
timeout -s KILL 900 python tools/decode_timing.py cfg3 > $O/decode_cfg3.log 2>&1; echo "cfg3 rc=$?"; cat $O/decode_cfg3.log
