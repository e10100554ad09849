# sharded decoder at one rank vs the single-GPU decoder (cfg3)
O=gpurun_out/c53
rm -rf $O; mkdir -p $O
timeout -s KILL 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 1 --config cfg3 --sharded --steps 2 --warmup 1 --json-out $O/bench_cfg3_sharded_n1.json > $O/sharded.log 2>&1; echo "sharded rc=$?"; tail -c 900 $O/bench_cfg3_sharded_n1.json
