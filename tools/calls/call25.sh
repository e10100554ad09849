O=gpurun_out/c25
mkdir -p $O
timeout -s KILL 1500 python -m pytest tests -m gpu -q --timeout 900 > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -5 $O/pytest_gpu.log
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 $O/smoke.log
timeout -s KILL 900 python bench.py --steps 5 --warmup 3 --json-out $O/bench_cfg1.json > $O/bench_cfg1.log 2>&1; echo "cfg1 rc=$?"; grep "\[bench\]" $O/bench_cfg1.log | head -2
python -c "
import json; d=json.load(open('$O/bench_cfg1.json')); r=d['roofline']; print(d['value'], d['e2e']['value'], r['kernel'], r['avg_launch_ms'], r['frac']); print(d['config']); print(d['stage_ms'], d['cpu_baseline']['value'])"
timeout -s KILL 900 python bench.py --impl reference --steps 1 --warmup 1 --json-out $O/bench_ref.json > $O/bench_ref.log 2>&1; echo "ref rc=$?"; tail -c 600 $O/bench_ref.json
