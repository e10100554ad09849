# Round evidence for profiles/: GPU tests, smoke, bench lines (cfg1 default +
# reference arm, cfg0, cfg2, cfg3), timed-region launch lists, and one ncu
# --set full capture per top kernel (each after its command ran clean).
# usage: bash tools/prof_round.sh [outdir]
O=${1:-gpurun_out/prof}
rm -rf $O; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/smi.txt 2>&1
timeout -s KILL 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 $O/pytest_gpu.log
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 $O/smoke.log
timeout -s KILL 600 python bench.py --steps 5 --warmup 3 --json-out $O/bench_cfg1.json > $O/bench_cfg1.log 2>&1; echo "cfg1 rc=$?"; grep "\[bench\] step" $O/bench_cfg1.log
timeout -s KILL 600 python bench.py --impl reference --steps 2 --warmup 1 --json-out $O/bench_ref.json > $O/bench_ref.log 2>&1; echo "ref rc=$?"
timeout -s KILL 600 python bench.py --config cfg0 --steps 5 --warmup 3 --json-out $O/bench_cfg0.json > $O/bench_cfg0.log 2>&1; echo "cfg0 rc=$?"
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file $O/launches_cfg1.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > $O/ncu_launch.log 2>&1; echo "launch list rc=$?"
for k in cg_apply_fast2 pcg_persistent fista_persist power_iter_coop cg_update cg_residual; do
  timeout -s KILL 600 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:$k -c 1 -o $O/full_cfg1_$k -f python tools/profile_step.py > $O/ncu_full_cfg1_$k.log 2>&1; echo "ncu $k rc=$?"
done
timeout -s KILL 900 python bench.py --config cfg3 --steps 3 --warmup 3 --json-out $O/bench_cfg3.json > $O/bench_cfg3.log 2>&1; echo "cfg3 rc=$?"
timeout -s KILL 900 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file $O/launches_cfg3.csv python bench.py --config cfg3 --steps 1 --warmup 1 > $O/ncu_launch3.log 2>&1; echo "launch list cfg3 rc=$?"
SWEEP_ITERS=3 timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:"cg_apply_(band|col)_k|cg_update|cg_residual" -s 4 -c 4 -o $O/full_cfg3 -f python tools/band_sweep.py 1,1024,32,1 > $O/ncu_full_cfg3.log 2>&1; echo "ncu cfg3 rc=$?"
timeout -s KILL 600 python bench.py --config cfg2 --steps 3 --warmup 3 --json-out $O/bench_cfg2.json > $O/bench_cfg2.log 2>&1; echo "cfg2 rc=$?"
timeout -s KILL 900 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file $O/launches_cfg2.csv python bench.py --config cfg2 --steps 1 --warmup 1 > $O/ncu_launch2.log 2>&1; echo "launch list cfg2 rc=$?"
timeout -s KILL 900 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:knn_tc_filter2 -c 1 -o $O/full_cfg2_tc -f python bench.py --config cfg2 --steps 1 --warmup 1 > $O/ncu_full_cfg2.log 2>&1; echo "ncu cfg2 rc=$?"
# summarise the full captures here and drop the reports (gpurun copies back <= 64 MiB)
for r in $O/*.ncu-rep; do python tools/ncu_summary.py $r > ${r%.ncu-rep}.md 2>/dev/null; done
python tools/ncu_hot.py $O/full_cfg1_cg_apply_fast2.ncu-rep cg_apply_fast2 20 > $O/hot_cfg1_apply.txt 2>/dev/null
python tools/ncu_hot.py $O/full_cfg1_fista_persist.ncu-rep fista_persist 20 > $O/hot_cfg1_fista.txt 2>/dev/null
rm -f $O/*.ncu-rep
ls $O | wc -l; du -sh $O
