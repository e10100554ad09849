O=gpurun_out/r82; mkdir -p $O
CPCAG_APPLY=fast5 timeout 300 python tools/profile_step.py > /dev/null 2>&1; echo "plain rc=$?"
for v in fast2 fast5; do
CPCAG_APPLY=$v timeout -s KILL 600 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:cg_apply_$v -c 1 -o $O/$v -f python tools/profile_step.py > $O/$v.log 2>&1; echo "ncu $v rc=$?"
done
