# lr bank-aware entry order (cfg3) + CG vector-kernel cache modes (cfg1)
O=gpurun_out/c42
rm -rf $O; mkdir -p $O
VARIANTS=f32/krylov64,f64 timeout -s KILL 900 python tools/decode_timing.py cfg3 > $O/decode_cfg3.log 2>&1; echo "cfg3 rc=$?"; cat $O/decode_cfg3.log | cut -c1-400
for m in 0 1 2 3 4 5 6 7; do
  CPCAG_CG_MODE=$m timeout -s KILL 300 python tools/decode_timing.py cfg1 > $O/decode_cfg1_m$m.log 2>&1; echo "mode $m rc=$?"; grep "krylov fp32" $O/decode_cfg1_m$m.log | cut -c1-400
done
timeout -s KILL 1500 python -m pytest tests -m gpu -x -q > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -5 $O/pytest.log
