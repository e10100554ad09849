CPCAG_TRACE=1 JIT_N=40 timeout -s KILL 300 python tools/jitter.py > gpurun_out/jit68.log 2>&1
grep -E "pipeline flush" gpurun_out/jit68.log
grep "cpcag trace" gpurun_out/jit68.log | grep -v "enter" | awk '{print $(NF-1), $0}' | sort -rn | head -14
