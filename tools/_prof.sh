nproc; uptime; ps -eo pcpu,comm --sort=-pcpu | head -8
JIT_ONE=1 JIT_N=40 timeout -s KILL 300 python tools/jitter.py 2>&1 | grep -E "pipeline flush" | sed 's/^/default /'
JIT_ONE=1 JIT_NOGC=1 JIT_N=40 timeout -s KILL 300 python tools/jitter.py 2>&1 | grep -E "pipeline flush" | sed 's/^/nogc /'
JIT_ONE=1 CUDA_MODULE_LOADING=EAGER JIT_N=40 timeout -s KILL 300 python tools/jitter.py 2>&1 | grep -E "pipeline flush" | sed 's/^/eager /'
uptime
