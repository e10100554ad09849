# K = 3 power iteration at 768 threads: bench + the power tests
O=gpurun_out/c52
rm -rf $O; mkdir -p $O
timeout -s KILL 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --json-out $O/bench_cfg1.json > $O/bench_cfg1.log 2>&1; echo "cfg1 rc=$?"; grep "\[bench\] step" $O/bench_cfg1.log | cut -c1-200
python -c "
import json; d=json.load(open('$O/bench_cfg1.json')); print(d['value'], d['e2e']['value'], d['stage_ms'])"
timeout -s KILL 900 python -m pytest tests/test_gpu_numeric.py -m gpu -x -q > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest.log
