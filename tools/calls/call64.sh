# Pipelined dense tile: FISTA tests (one-GPU dense path and sharded), world-1 bench block.
O=gpurun_out/shf2
rm -rf $O; mkdir -p $O
timeout -s KILL 900 python -m pytest tests/test_sharded_fista.py tests/test_gpu_numeric.py tests/test_golden_pipeline.py -m gpu -x -q > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest.log
timeout -s KILL 600 python tools/shf_bench_world1.py > $O/bench_world1.log 2>&1; echo "bench rc=$?"; tail -1 $O/bench_world1.log
