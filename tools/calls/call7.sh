set -x
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; tail -2 gpurun_out/smoke.log
timeout 1500 python -m pytest tests -q -m gpu -x --timeout 900 > gpurun_out/t_all.log 2>&1; tail -5 gpurun_out/t_all.log
