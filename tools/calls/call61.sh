# Sharded FISTA with the dense block kernels: tests, timing, world-1 bench block.
O=gpurun_out/shf
mkdir -p $O
timeout -s KILL 600 python -m pytest tests/test_sharded_fista.py -m gpu -x -q > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -6 $O/pytest.log
timeout -s KILL 600 python tools/shf_timing.py > $O/timing.log 2>&1; echo "timing rc=$?"; tail -6 $O/timing.log
timeout -s KILL 600 python tools/shf_bench_world1.py > $O/bench_world1.log 2>&1; echo "bench rc=$?"; tail -1 $O/bench_world1.log
