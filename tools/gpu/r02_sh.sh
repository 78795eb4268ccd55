mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
T=${TAG:-r02sh}
KNNJ_TRACE=1 timeout 600 python tools/probe_steps.py --config C5 --steps 3 > gpurun_out/${T}_C5_trace.log 2>&1
for cfg in C5 C2; do
  echo "== shards $cfg" >> gpurun_out/${T}.log
  timeout 900 python tools/shard_timing.py --config $cfg --shards 8 --steps 2 2>&1 | tail -9 | cut -c1-300 >> gpurun_out/${T}.log
done
lscpu | head -20 > gpurun_out/${T}_lscpu.txt
echo done
