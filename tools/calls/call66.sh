# ncu --set full of the sharded FISTA's two dense tile kernels (one launch each, world size 1), after a clean run.
O=gpurun_out/shf3
rm -rf $O; mkdir -p $O
timeout -s KILL 600 python tools/shf_bench_world1.py > $O/bench_world1.log 2>&1 || { echo "plain run failed"; exit 1; }
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:"shf_dense_(grad_prox|block_sums)_k" -s 20 -c 2 \
  -o $O/full_shf -f python tools/shf_bench_world1.py > $O/ncu_full.log 2>&1; echo "ncu rc=$?"
python tools/ncu_summary.py $O/full_shf.ncu-rep > $O/full_shf.md 2> $O/summary.err; echo "summary rc=$?"; cat $O/full_shf.md | head -20
