# Quick GPU iteration: selected tests + a cfg1 bench line.
O=gpurun_out/quick
rm -rf $O; mkdir -p $O
timeout -s KILL 900 python -m pytest ${TESTS:-tests} -m gpu -x -q > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -15 $O/pytest.log
if [ -z "$NOBENCH" ]; then
timeout -s KILL 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --json-out $O/bench_cfg1.json > $O/bench_cfg1.log 2>&1; echo "cfg1 rc=$?"
python -c "
import json;d=json.load(open('$O/bench_cfg1.json'));print({k:d.get(k) for k in ['value','e2e','stage_ms','kernel_share']})"
fi
