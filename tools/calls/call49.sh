# cfg4 bench line at the current HEAD
O=gpurun_out/c49
rm -rf $O; mkdir -p $O
timeout -s KILL 1500 python bench.py --config cfg4 --steps 1 --warmup 1 --json-out $O/bench_cfg4.json > $O/bench_cfg4.log 2>&1; echo "cfg4 rc=$?"; tail -c 1500 $O/bench_cfg4.json
