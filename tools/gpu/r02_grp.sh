mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
T=${TAG:-r02grp}
for v in "" "--opt level0_group_span=4" "--opt level0_group_span=8"; do
for cfg in C4 C2; do
  echo "== $cfg $v" >> gpurun_out/${T}.log
  KNNJ_JOIN_STATS=1 timeout 600 python tools/probe_steps.py --config $cfg --steps 3 $v 2>&1 | grep -E "mixed tc part|pass: tc|step 2" | tail -4 | cut -c1-280 >> gpurun_out/${T}.log
done
done
echo done
