O=gpurun_out/c27
mkdir -p $O
python tools/profile_step.py > $O/plain.log 2>&1 && \
timeout -s KILL 600 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:"fista_persist_k" -c 1 -o $O/fista -f python tools/profile_step.py > $O/ncu.log 2>&1; echo "ncu rc=$?"
