for k in 16 8 6 4; do CPCAG_FAST2_CTAS=$k timeout -s KILL 300 python tools/bench_stages.py 2>&1 | grep "decode" | cut -c1-140 | sed "s/^/ctas=$k /"; done
