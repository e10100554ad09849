set -x

timeout 900 python tools/cfg3_precision.py > gpurun_out/cfg3_precision.log 2>&1

