for v in "CPCAG_FAST2_MINB=4" "CPCAG_FAST2_MINB=5" "CPCAG_FAST2_MINB=6" "CPCAG_FAST2_MINB=5 CPCAG_FAST2_CTAS=10" "CPCAG_FAST2_MINB=6 CPCAG_FAST2_CTAS=12"; do
  env $v timeout 300 python bench.py --no-cpu-baseline --no-e2e 2> /dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v', d['value'], d['stage_ms']['decode'], d['roofline']['avg_launch_ms'])"
done
