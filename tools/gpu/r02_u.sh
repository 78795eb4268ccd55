mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
T=${TAG:-r02u}
for v in "" "--opt item_tc_min_q=16" "--opt item_tc_min_q=8"; do
  echo "== C4 $v" >> gpurun_out/${T}.log
  KNNJ_JOIN_STATS=1 timeout 600 python tools/probe_steps.py --config C4 --steps 3 $v 2>&1 | grep -E "mixed tc|step 2" | tail -2 | cut -c1-330 >> gpurun_out/${T}.log
done
for cfg in C5 C2; do
  echo "== shards $cfg" >> gpurun_out/${T}.log
  timeout 900 python tools/shard_timing.py --config $cfg --shards 8 --steps 2 2>&1 | tail -10 | cut -c1-300 >> gpurun_out/${T}.log
done
echo done
