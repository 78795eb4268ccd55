mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
T=${TAG:-r02t}
for v in "--opt tc_slack=40" "--opt tc_slack=64"; do
  echo "== C4 $v" >> gpurun_out/${T}.log
  KNNJ_JOIN_STATS=1 timeout 600 python tools/probe_steps.py --config C4 --steps 3 $v 2>&1 | grep -E "mixed tc|step 2" | tail -2 | cut -c1-330 >> gpurun_out/${T}.log
done
for v in "--opt tc_slack=32" "--opt tc_slack=16"; do
  echo "== C5 $v" >> gpurun_out/${T}.log
  KNNJ_JOIN_STATS=1 timeout 600 python tools/probe_steps.py --config C5 --steps 3 $v 2>&1 | grep -E "join stats|step 2" | tail -3 | cut -c1-330 >> gpurun_out/${T}.log
done
for v in "" "--opt tc_slack=32"; do
  echo "== NS $v" >> gpurun_out/${T}.log
  KNNJ_JOIN_STATS=1 timeout 600 python tools/probe_steps.py --config NS --steps 3 $v 2>&1 | grep -E "join stats|step 2" | tail -2 | cut -c1-330 >> gpurun_out/${T}.log
done
echo done
