set -x
python tools/sanitize_case.py > gpurun_out/san_plain.log 2>&1 && \
timeout 1200 compute-sanitizer --tool memcheck --print-limit 20 python tools/sanitize_case.py > gpurun_out/san_memcheck.log 2>&1; tail -4 gpurun_out/san_memcheck.log
timeout 900 python tools/cfg4_probe.py > gpurun_out/cfg4_probe.log 2>&1; cat gpurun_out/cfg4_probe.log | cut -c1-400
