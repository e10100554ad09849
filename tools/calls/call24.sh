O=gpurun_out/c24
mkdir -p $O
timeout -s KILL 1200 python -m pytest tests/test_gpu_numeric.py tests/test_gpu_graph.py tests/test_golden_pipeline.py -q -x --timeout 900 > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest.log
timeout -s KILL 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --json-out $O/bench_cfg1.json > $O/bench_cfg1.log 2>&1; echo "cfg1 rc=$?"; grep "\[bench\]" $O/bench_cfg1.log | head -3
python -c "
import json; d=json.load(open('$O/bench_cfg1.json')); r=d['roofline']; print(d['value'], r['kernel'], r['avg_launch_ms'], r['frac']); print(d['stage_ms'], d['kernel_share'])"
