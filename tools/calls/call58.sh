# Sharded FISTA: GPU tests + a timing of the emulated / one-rank solve at the config-1 compressed size.
O=gpurun_out/shf
rm -rf $O; mkdir -p $O
timeout -s KILL 600 python -m pytest tests/test_sharded_fista.py -m gpu -x -q > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -15 $O/pytest.log
timeout -s KILL 600 python tools/shf_timing.py > $O/timing.log 2>&1; echo "timing rc=$?"; tail -12 $O/timing.log
