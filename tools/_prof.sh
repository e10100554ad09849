JIT_ONE=1 JIT_N=40 timeout -s KILL 300 python tools/jitter.py 2>&1 | grep -E "pipeline flush" | sed 's/^/default /'
JIT_ONE=1 JIT_RESERVE=8 JIT_N=40 timeout -s KILL 300 python tools/jitter.py 2>&1 | grep -E "pipeline flush" | sed 's/^/reserve8 /'
