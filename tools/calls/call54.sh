# sharded decoder in the sorted row order: tests + N = 1 against the single-GPU decoder (cfg3)
O=gpurun_out/c54
rm -rf $O; mkdir -p $O
timeout -s KILL 1500 python -m pytest tests -m gpu -x -q > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest.log
timeout -s KILL 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 1 --config cfg3 --sharded --steps 2 --warmup 1 --json-out $O/bench_cfg3_sharded_n1.json > $O/sharded.log 2>&1; echo "sharded rc=$?"; python -c "
import json; d=json.load(open('$O/bench_cfg3_sharded_n1.json')); print('sharded n1', d['value'])"
timeout -s KILL 900 python bench.py --config cfg3 --steps 2 --warmup 1 --json-out $O/bench_cfg3.json > $O/bench_cfg3.log 2>&1; echo "cfg3 rc=$?"; python -c "
import json; d=json.load(open('$O/bench_cfg3.json')); print('single', d['value'])"
