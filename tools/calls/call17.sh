set -x
O=gpurun_out/r02s
mkdir -p $O
timeout -s KILL 1500 python -m pytest tests -m gpu -q -x --timeout 900 > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest_gpu.log
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 $O/smoke.log
timeout -s KILL 600 python bench.py --steps 5 --warmup 3 --json-out $O/bench_cfg1.json > $O/bench_cfg1.log 2>&1; echo "cfg1 rc=$?"; grep "\[bench\]" $O/bench_cfg1.log | head -3
timeout -s KILL 600 python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > $O/plain1.log 2>&1 && \
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file $O/launches_cfg1.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > $O/ncu_launch.log 2>&1; echo "launch list rc=$?"
python tools/launch_summary.py $O/launches_cfg1.csv > $O/launches_cfg1_summary.txt; head -14 $O/launches_cfg1_summary.txt
