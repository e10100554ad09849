# stage trace of the cfg1 step (synchronising marks)
O=gpurun_out/c38
mkdir -p $O
CPCAG_TRACE=1 timeout -s KILL 600 python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > $O/trace_bench.log 2> $O/trace.log; echo "rc=$?"
grep "\[bench\] step" $O/trace_bench.log | cut -c1-150
