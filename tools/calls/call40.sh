# monotonic-counter grid barrier (power iteration, persistent FISTA): parity + bench + launch list
O=gpurun_out/c40
mkdir -p $O
timeout -s KILL 900 python -m pytest tests -m gpu -q -x -k "power or fista or persist or pipeline" > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -1 $O/pytest.log
timeout -s KILL 600 python bench.py --steps 10 --warmup 4 --no-cpu-baseline --json-out $O/bench.json > $O/bench.log 2>&1; echo "bench rc=$?"; grep "step ms" $O/bench.log | cut -c1-200
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
  --log-file $O/launches_cfg1.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > $O/ncu_launch.log 2>&1
echo "launch list rc=$?"; python tools/launch_summary.py $O/launches_cfg1.csv 10
