O=gpurun_out/b2; rm -rf $O; mkdir -p $O
for r in 1 2; do timeout -s KILL 600 python bench.py --steps 5 --warmup 3 --json-out $O/bench_cfg1_$r.json > $O/cfg1_$r.log 2>&1; echo "cfg1 rc=$? $(grep 'step ms' $O/cfg1_$r.log)"; done
timeout -s KILL 600 python bench.py --config cfg2 --steps 3 --warmup 3 --json-out $O/bench_cfg2.json > $O/cfg2.log 2>&1; echo "cfg2 rc=$? $(grep 'step ms' $O/cfg2.log)"
timeout -s KILL 900 python bench.py --config cfg3 --steps 3 --warmup 3 --json-out $O/bench_cfg3.json > $O/cfg3.log 2>&1; echo "cfg3 rc=$? $(grep 'step ms' $O/cfg3.log)"
python -c "
import json
for f in ['bench_cfg1_1','bench_cfg1_2','bench_cfg2','bench_cfg3']:
    d=json.load(open('$O/'+f+'.json')); print(f, d['value'], d.get('clocks'), d.get('e2e',{}).get('value') if isinstance(d.get('e2e'),dict) else None)"
