# decoder tests + cfg1 bench + one ncu capture of the slab apply
O=gpurun_out/c20
mkdir -p $O
timeout -s KILL 900 python -m pytest tests/test_gpu_numeric.py -q -x --timeout 600 -k "decoder or decode" > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest.log
timeout -s KILL 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --json-out $O/bench_cfg1.json > $O/bench_cfg1.log 2>&1; echo "cfg1 rc=$?"; grep "\[bench\]" $O/bench_cfg1.log | head -2
python -c "
import json; d=json.load(open('$O/bench_cfg1.json')); r=d['roofline']; print(d['value'], r['kernel'], r['avg_launch_ms'], r['frac']); print(d['stage_ms'], d['kernel_roofline'])"
if [ "$1" = "ncu" ]; then
python tools/profile_step.py > $O/plain.log 2>&1 && \
timeout -s KILL 600 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:"^slab_k" -c 1 -o $O/slab -f python tools/profile_step.py > $O/ncu.log 2>&1; echo "ncu rc=$?"
fi
