# symmetric kNN tiles kKc 32: knn parity + cfg1 launch list
O=gpurun_out/c37
mkdir -p $O
timeout -s KILL 900 python -m pytest tests -m gpu -q -x -k "knn or graph or golden" > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -1 $O/pytest.log
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
  --log-file $O/launches_cfg1.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > $O/ncu_launch.log 2>&1
echo "launch list rc=$?"; python tools/launch_summary.py $O/launches_cfg1.csv 30 | grep -i "knn\|total"
