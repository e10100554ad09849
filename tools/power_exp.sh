# Power-iteration experiment at cfg1: phase times and the single-CTA threshold.
O=gpurun_out/power; rm -rf $O; mkdir -p $O
for v in "" "CPCAG_POWER_SMALL_NNZ=20000" "CPCAG_POWER_SMALL_NNZ=20000 CPCAG_POWER_NB=74"; do
  env CPCAG_POWER_PROF=1 $v timeout -s KILL 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --json-out $O/b.json > $O/log.txt 2>&1
  echo "== $v rc=$?"; grep "power_iter" $O/log.txt | sort | uniq -c | head -4
  env $v timeout -s KILL 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --json-out $O/b.json > $O/log2.txt 2>&1
  python -c "
import json;d=json.load(open('$O/b.json'));print(d['value'], d.get('stage_ms'))"
done
