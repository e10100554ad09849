CPCAG_TRACE=1 timeout -s KILL 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b49.log 2>&1; grep "\[bench\]" gpurun_out/b49.log | head -3
python - <<'PY'
import re
lines=open('gpurun_out/b49.log').read().splitlines()
# print kron trace blocks whose 'solves+schur' or others exceed 30 ms
for i,l in enumerate(lines):
    m=re.match(r'\[cpcag trace\] (.+?)\s+([0-9.]+) ms', l)
    if m and float(m.group(2))>15: print(i, l)
PY
