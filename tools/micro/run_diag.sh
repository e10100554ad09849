CPCAG_FISTA_PERSIST_PROF=1 python tools/fista_diag.py 2>&1 | grep -v "^shape" | tail -3
./tools/micro/barrier_bench | head -3
