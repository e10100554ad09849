CPCAG_TRACE=1 JIT_N=60 timeout -s KILL 300 python tools/jitter.py > gpurun_out/jit66.log 2>&1
grep "kron ms" gpurun_out/jit66.log | head -1
grep "cpcag trace" gpurun_out/jit66.log | awk '{print $(NF-1), $0}' | sort -rn | head -12
