# power two-step + decoder row permutation + lc L2 policy experiment
O=gpurun_out/c41
rm -rf $O; mkdir -p $O
timeout -s KILL 900 python -m pytest tests/test_gpu_numeric.py tests/test_gpu_fullsize.py -m gpu -x -q > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -5 $O/pytest.log
timeout -s KILL 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --json-out $O/bench_cfg1.json > $O/bench_cfg1.log 2>&1; echo "cfg1 rc=$?"; grep "\[bench\] step" $O/bench_cfg1.log | cut -c1-200
python -c "
import json; d=json.load(open('$O/bench_cfg1.json')); print(d['value'], d['stage_ms'], d['kernel_share'])"
for pol in 0 1 2 3; do
  CPCAG_LC_POLICY=$pol VARIANTS=f32/krylov64 timeout -s KILL 600 python tools/decode_timing.py cfg3 > $O/decode_cfg3_pol$pol.log 2>&1; echo "pol $pol rc=$?"; cat $O/decode_cfg3_pol$pol.log | cut -c1-400
done
