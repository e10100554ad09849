timeout 900 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_graph.py -q -m gpu -x 2>&1 | tail -2
for v in "X=0" "CPCAG_KNN_DBG=1"; do
  env $v timeout 300 python bench.py --config cfg2 --steps 3 --warmup 2 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', d['value'], d.get('kernel_ms'))"
done
