# lc one band per wave (cfg3) + hardwired streaming hints (cfg1)
O=gpurun_out/c43
rm -rf $O; mkdir -p $O
VARIANTS=f32/krylov64 timeout -s KILL 900 python tools/decode_timing.py cfg3 > $O/decode_cfg3.log 2>&1; echo "cfg3 rc=$?"; cat $O/decode_cfg3.log | cut -c1-400
timeout -s KILL 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --json-out $O/bench_cfg1.json > $O/bench_cfg1.log 2>&1; echo "cfg1 rc=$?"; grep "\[bench\] step" $O/bench_cfg1.log | cut -c1-200
python -c "
import json; d=json.load(open('$O/bench_cfg1.json')); print(d['value'], d['stage_ms'], d['kernel_roofline'])"
timeout -s KILL 900 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_numeric.py -m gpu -x -q > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest.log
