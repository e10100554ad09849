set -x
O=gpurun_out/c19
mkdir -p $O
python tools/profile_step.py > $O/plain.log 2>&1 && \
timeout -s KILL 600 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:"^slab_k" -c 2 -o $O/slab -f python tools/profile_step.py > $O/ncu.log 2>&1; echo "ncu rc=$?"; tail -3 $O/ncu.log
