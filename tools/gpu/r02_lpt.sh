mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
T=${TAG:-r02lpt}
for v in "" "--opt lpt=0"; do
for cfg in C5 C2; do
  echo "== $cfg $v" >> gpurun_out/${T}.log
  KNNJ_JOIN_STATS=1 timeout 600 python tools/probe_steps.py --config $cfg --steps 3 $v 2>&1 | grep -E "join stats|step 2" | tail -2 | cut -c1-300 >> gpurun_out/${T}.log
done
done
echo done
