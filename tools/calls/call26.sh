O=gpurun_out/c26
mkdir -p $O
timeout -s KILL 900 python -m pytest tests/test_gpu_fista_persist.py tests/test_gpu_numeric.py -q -x --timeout 600 -k "fista" > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -15 $O/pytest.log
CPCAG_TRACE=1 timeout -s KILL 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --json-out $O/bench_cfg1.json > $O/bench_cfg1.log 2>&1; echo "cfg1 rc=$?"; grep "\[bench\]\|fista_persist\]" $O/bench_cfg1.log | head -4
python -c "
import json; d=json.load(open('$O/bench_cfg1.json')); r=d['roofline']; print(d['value'], r['kernel'], r['avg_launch_ms'], r['frac']); print(d['stage_ms'], d['kernel_share'])"
