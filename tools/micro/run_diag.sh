timeout -s KILL 900 python -m pytest tests/test_gpu_numeric.py tests/test_gpu_band_apply.py -m gpu -x -q 2>&1 | tail -2
for v in 1 0; do CPCAG_CG_VEC=$v timeout -s KILL 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --json-out gpurun_out/b_vec$v.json > /dev/null 2>&1; echo "vec=$v rc=$?"; python -c "
import json;d=json.load(open('gpurun_out/b_vec$v.json'));print(d['value'], d['stage_ms']['decode'], {k: round(v*d['value']*1e3,2) for k,v in d['kernel_share'].items()})"; done
