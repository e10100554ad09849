# the driver's launches: plain default bench, torchrun N = 1 (adds the sharded_cfg3 block), reference arm
O=gpurun_out/c56
rm -rf $O; mkdir -p $O
timeout -s KILL 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29513 bench.py --gpus 1 --steps 5 --warmup 3 > $O/torchrun_n1.log 2>&1; echo "torchrun rc=$?"; tail -1 $O/torchrun_n1.log | python -c "
import json,sys; d=json.loads(sys.stdin.readline()); print(d['value'], d['e2e']['value'], d.get('sharded_cfg3'))"
timeout -s KILL 900 python bench.py > $O/default.log 2>&1; echo "default rc=$?"; tail -1 $O/default.log | python -c "
import json,sys; d=json.loads(sys.stdin.readline()); print(d['value'], d['e2e'], d['roofline']['frac'], d['cpu_baseline']['value'], d['gpu_launches'], d['clocks'])"
