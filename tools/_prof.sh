timeout -s KILL 300 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/t_all.log 2>&1
tail -3 gpurun_out/t_all.log
timeout -s KILL 300 python bench.py --steps 3 --warmup 2 --json-out gpurun_out/bench17.json > gpurun_out/bench17.log 2>&1
tail -1 gpurun_out/bench17.log | cut -c1-2500
timeout -s KILL 120 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
