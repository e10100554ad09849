for v in "X=1" "CPCAG_KRON_SLICE=172" "CPCAG_KRON_SLICE=258" "CPCAG_KRON_SLICE=344" "CPCAG_KRON_SLICE=516" ; do
  env $v timeout 300 python bench.py --no-cpu-baseline --no-e2e 2> gpurun_out/b_$v.err | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v', d['value'], d['stage_ms'])"
done
