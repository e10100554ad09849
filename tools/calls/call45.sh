# launch list of one cfg1 step at the current HEAD
O=gpurun_out/c45
rm -rf $O; mkdir -p $O
timeout -s KILL 600 python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > $O/plain1.log 2>&1 && \
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
  --log-file $O/launches_cfg1.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > $O/ncu_launch.log 2>&1
echo "launch list rc=$?"; python tools/launch_summary.py $O/launches_cfg1.csv > $O/launches_cfg1_summary.txt; head -30 $O/launches_cfg1_summary.txt
