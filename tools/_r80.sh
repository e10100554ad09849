set -x
timeout 1500 python -m pytest tests -q -m gpu -x 2>&1 | tail -4
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --config cfg3 --sharded --steps 3 --warmup 1 > gpurun_out/sh.log 2>&1; grep -v "^\[bench\]" gpurun_out/sh.log | grep "metric\|Error" | tail -3
timeout 600 python bench.py 2> gpurun_out/b1.err | tail -1
grep "step ms\|graphs=" gpurun_out/b1.err
