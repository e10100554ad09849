timeout 900 python -m pytest tests/test_gpu_fullsize.py -q -m gpu -x -k second 2>&1 | tail -2
