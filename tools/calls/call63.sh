# Launch list (gpu__time_duration) of the sharded FISTA kernels at NCCL world size 1, after a clean run.
O=gpurun_out/shf
mkdir -p $O
timeout -s KILL 600 python tools/shf_bench_world1.py > $O/bench_world1.log 2>&1 || { echo "plain run failed"; tail -5 $O/bench_world1.log; exit 1; }
tail -1 $O/bench_world1.log
timeout -s KILL 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:shf_ -c 1600 --csv \
  --log-file $O/launches_shf.csv python tools/shf_bench_world1.py > $O/ncu.log 2>&1; echo "ncu rc=$?"
python - <<'PY'
import csv, collections
rows = [r for r in csv.reader(open("gpurun_out/shf/launches_shf.csv")) if len(r) > 5]
hdr = rows[0]
ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
ui = hdr.index("Metric Unit")
acc = collections.defaultdict(list)
for r in rows[1:]:
    try:
        v = float(r[vi].replace(",", ""))
    except ValueError:
        continue
    if r[ui] == "ns":
        v /= 1e3
    elif r[ui] == "ms":
        v *= 1e3
    acc[r[ki].split("(")[0]].append(v)
with open("gpurun_out/shf/launches_shf_summary.txt", "w") as f:
    for k, v in sorted(acc.items(), key=lambda kv: -sum(kv[1])):
        line = f"{k:40s} launches {len(v):5d}  avg {sum(v)/len(v):8.2f} us  total {sum(v)/1e3:8.3f} ms"
        print(line); f.write(line + "\n")
PY
