# decoder planning overlapped with the power iterations: pipeline/decoder parity, bench, stage trace
O=gpurun_out/c39
mkdir -p $O
timeout -s KILL 900 python -m pytest tests -m gpu -q -x -k "pipeline or golden or decode or fullsize" > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -1 $O/pytest.log
timeout -s KILL 600 python bench.py --steps 10 --warmup 4 --no-cpu-baseline --json-out $O/bench.json > $O/bench.log 2>&1; echo "bench rc=$?"; grep "\[bench\]" $O/bench.log | cut -c1-220
CPCAG_TRACE=1 timeout -s KILL 600 python bench.py --steps 1 --warmup 2 --no-e2e --no-cpu-baseline > $O/trace_bench.log 2> $O/trace.log; echo "trace rc=$?"
tail -32 $O/trace.log
