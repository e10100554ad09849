for v in 4096 16384 65536; do CPCAG_POWER_SMALL_NNZ=$v timeout -s KILL 300 python tools/bench_stages.py 2>&1 | grep fista | cut -c1-150 | sed "s/^/small_nnz=$v /"; done
for sp in 2 4 8 17; do CPCAG_FISTA_SPLITS=$sp timeout -s KILL 300 python tools/bench_stages.py 2>&1 | grep fista | cut -c1-150 | sed "s/^/splits=$sp /"; done
