# Session check: GPU tests + bench lines for cfg1/cfg2/cfg3 (no profiler).
O=gpurun_out/chk
rm -rf $O; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/smi.txt 2>&1
timeout -s KILL 1500 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest_gpu.log
timeout -s KILL 600 python bench.py --steps 5 --warmup 3 --json-out $O/bench_cfg1.json > $O/bench_cfg1.log 2>&1; echo "cfg1 rc=$?"; tail -c 600 $O/bench_cfg1.json
timeout -s KILL 600 python bench.py --config cfg2 --steps 3 --warmup 3 --json-out $O/bench_cfg2.json > $O/bench_cfg2.log 2>&1; echo "cfg2 rc=$?"; tail -c 400 $O/bench_cfg2.json
timeout -s KILL 900 python bench.py --config cfg3 --steps 3 --warmup 3 --json-out $O/bench_cfg3.json > $O/bench_cfg3.log 2>&1; echo "cfg3 rc=$?"; tail -c 600 $O/bench_cfg3.json
