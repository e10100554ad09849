set -x
timeout 900 python -m pytest tests/test_gpu_fullsize.py tests/test_sharded.py -q -m gpu -x 2>&1 | tail -5
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --config cfg3 --sharded --steps 3 --warmup 1 > gpurun_out/sh.log 2>&1; grep -v "^\[bench\]" gpurun_out/sh.log | grep "metric\|Error" | tail -3
