set -x
O=gpurun_out/c18
mkdir -p $O
timeout -s KILL 900 python -m pytest tests/test_gpu_numeric.py -q -x --timeout 600 -k "decoder or decode" > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -15 $O/pytest.log
timeout -s KILL 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --json-out $O/bench_cfg1.json > $O/bench_cfg1.log 2>&1; echo "cfg1 rc=$?"; grep "\[bench\]" $O/bench_cfg1.log | head -3
python -c "
import json; d=json.load(open('$O/bench_cfg1.json')); print(d['value'], d['e2e']['value'], d['roofline']); print(d['stage_ms'], d['kernel_share'])"
