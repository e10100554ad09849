# launch list of a few sharded CG iterations at cfg3 (one rank)
O=gpurun_out/c55
rm -rf $O; mkdir -p $O
MASTER_ADDR=127.0.0.1 MASTER_PORT=29512 RANK=0 LOCAL_RANK=0 WORLD_SIZE=1 timeout -s KILL 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"lc_k|lr_reg_k|lr_k|cg_|pack_|nccl|ncclDev" --launch-skip 12 --launch-count 36 --csv --log-file $O/launches.csv python bench.py --gpus 1 --config cfg3 --sharded --steps 1 --warmup 0 > $O/ncu.log 2>&1; echo "rc=$?"
python tools/launch_summary.py $O/launches.csv | head -20
tail -3 $O/ncu.log | cut -c1-300
