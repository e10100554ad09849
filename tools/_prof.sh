timeout -s KILL 300 python tools/bench_stages.py 2>&1 | grep -E "decode|fista|kron" | cut -c1-220
for nb in 1 8 40 148; do CPCAG_POWER_NB=$nb timeout -s KILL 300 python tools/bench_stages.py 2>&1 | grep fista | cut -c1-120 | sed "s/^/NB=$nb /"; done
