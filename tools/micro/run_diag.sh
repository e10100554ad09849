timeout -s KILL 900 python -m pytest tests/test_gpu_fista_persist.py tests/test_gpu_numeric.py -m gpu -x -q 2>&1 | tail -2
CG=3 timeout -s KILL 900 python tools/cfg1_parity.py 2>&1 | grep FISTA
timeout -s KILL 900 python -m pytest tests/test_gpu_fullsize.py -x -q -k full_iterations 2>&1 | tail -2
