# Round evidence for profiles/: GPU tests, smoke, bench lines (cfg1 default +
# reference arm, cfg0, cfg2, cfg3), the timed-region launch list of cfg1, and
# ncu --set full captures of the top kernels (each after its command ran clean).
# usage: bash tools/prof_round.sh [outdir]
O=${1:-gpurun_out/prof}
rm -rf $O; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/smi.txt 2>&1
timeout -s KILL 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 $O/pytest_gpu.log
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 $O/smoke.log
timeout -s KILL 900 python bench.py --steps 20 --warmup 5 --json-out $O/bench_cfg1.json > $O/bench_cfg1.log 2>&1; echo "cfg1 rc=$?"; grep "\[bench\] step" $O/bench_cfg1.log
timeout -s KILL 900 python bench.py --impl reference --steps 3 --warmup 1 --json-out $O/bench_ref.json > $O/bench_ref.log 2>&1; echo "ref rc=$?"
timeout -s KILL 600 python bench.py --config cfg0 --steps 20 --warmup 5 --json-out $O/bench_cfg0.json > $O/bench_cfg0.log 2>&1; echo "cfg0 rc=$?"
timeout -s KILL 600 python bench.py --config cfg2 --steps 3 --warmup 3 --json-out $O/bench_cfg2.json > $O/bench_cfg2.log 2>&1; echo "cfg2 rc=$?"
timeout -s KILL 900 python bench.py --config cfg3 --steps 2 --warmup 1 --json-out $O/bench_cfg3.json > $O/bench_cfg3.log 2>&1; echo "cfg3 rc=$?"
# launch list of one timed cfg1 step
timeout -s KILL 600 python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > $O/plain1.log 2>&1 && \
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
  --log-file $O/launches_cfg1.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > $O/ncu_launch.log 2>&1
echo "launch list rc=$?"; python tools/launch_summary.py $O/launches_cfg1.csv > $O/launches_cfg1_summary.txt
# full captures of the cfg1 step's top kernels
python tools/profile_step.py > $O/plain_step.log 2>&1 && \
for k in slab_k pcg_smem_k fista_persist_k power_iter_coopk_k cg_update_k cg_residual_k; do
  timeout -s KILL 600 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:"^$k" -c 1 \
    -o $O/full_cfg1_$k -f python tools/profile_step.py > $O/ncu_full_cfg1_$k.log 2>&1; echo "ncu $k rc=$?"
done
# cfg3 decoder kernels (one fixed-iteration decode)
timeout -s KILL 900 python tools/decode_timing.py cfg3 > $O/decode_cfg3.log 2>&1 && \
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:"^(lc_k|lr_reg_k|cg_update_k|cg_residual_k)" -s 8 -c 4 \
  -o $O/full_cfg3 -f python tools/decode_timing.py cfg3 > $O/ncu_full_cfg3.log 2>&1; echo "ncu cfg3 rc=$?"
for r in $O/*.ncu-rep; do python tools/ncu_summary.py $r > ${r%.ncu-rep}.md 2>/dev/null; python tools/ncu_metrics.py $r > ${r%.ncu-rep}_metrics.txt 2>/dev/null; done
python tools/ncu_summary.py $O/full_cfg1_slab_k.ncu-rep $O/ncu_traffic_slab.json > /dev/null 2>&1
python tools/ncu_hot.py $O/full_cfg1_slab_k.ncu-rep slab_k 25 > $O/hot_cfg1_slab.txt 2>/dev/null
python tools/ncu_hot.py $O/full_cfg1_fista_persist_k.ncu-rep fista_persist 25 > $O/hot_cfg1_fista.txt 2>/dev/null
rm -f $O/*.ncu-rep
ls $O | wc -l; du -sh $O
