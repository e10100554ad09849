set -x
mkdir -p gpurun_out/r02
python bench.py --config cfg3 --steps 2 --warmup 1 > gpurun_out/r02/cfg3.out 2> gpurun_out/r02/cfg3.err; tail -c 400 gpurun_out/r02/cfg3.out
python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29555 bench.py --config cfg3 --sharded --steps 2 --warmup 1 > gpurun_out/r02/cfg3_sharded_n1.out 2> gpurun_out/r02/cfg3_sharded_n1.err; tail -c 800 gpurun_out/r02/cfg3_sharded_n1.out; tail -5 gpurun_out/r02/cfg3_sharded_n1.err
