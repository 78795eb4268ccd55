mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
T=${TAG:-r02s}
for v in "" "--opt sweep_order=0" "--opt box_filter=0" "--opt kth_bound=0"; do
  echo "== C5 $v" >> gpurun_out/${T}.log
  KNNJ_JOIN_STATS=1 timeout 600 python tools/probe_steps.py --config C5 --steps 3 $v 2>&1 | grep -E "join stats|step 2" | tail -3 | cut -c1-300 >> gpurun_out/${T}.log
done
for v in "" "--opt sweep_order=0"; do
  echo "== C4 $v" >> gpurun_out/${T}.log
  KNNJ_JOIN_STATS=1 timeout 600 python tools/probe_steps.py --config C4 --steps 2 $v 2>&1 | grep -E "mixed tc|step 1" | tail -3 | cut -c1-300 >> gpurun_out/${T}.log
done
echo done
