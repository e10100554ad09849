O=gpurun_out/c33
mkdir -p $O
timeout -s KILL 600 python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > $O/plain1.log 2>&1 && \
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
  --log-file $O/launches_cfg1.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > $O/ncu_launch.log 2>&1
echo "launch list rc=$?"; python tools/launch_summary.py $O/launches_cfg1.csv 30
