set -x
timeout 1500 python -m pytest tests -q -m gpu --timeout 900 > gpurun_out/t_all.log 2>&1; tail -4 gpurun_out/t_all.log
python tools/sanitize_case.py > gpurun_out/san_plain.log 2>&1 && \
timeout 1200 compute-sanitizer --tool memcheck --print-limit 20 python tools/sanitize_case.py > gpurun_out/san_memcheck.log 2>&1; tail -4 gpurun_out/san_memcheck.log
