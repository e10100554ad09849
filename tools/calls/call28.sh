O=gpurun_out/c28
mkdir -p $O
timeout -s KILL 900 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --json-out $O/bench_cfg1.json > $O/bench_cfg1.log 2>&1; echo "cfg1 rc=$?"; grep "\[bench\] step" $O/bench_cfg1.log | head -2
python -c "
import json; d=json.load(open('$O/bench_cfg1.json')); r=d['roofline']; print(d['value'], d['e2e']['value'], r['kernel'], r['avg_launch_ms'], r['frac']); print(d['stage_ms'])"
