mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
T=${TAG:-r02v}
timeout 900 python -m pytest tests/test_gpu_shard_hist.py tests/test_gpu_multiprocess.py tests/test_gpu_fullsize.py -q -x -k "sharded or torchrun or knobs or grid or C5 or C4" > gpurun_out/${T}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_pytest.log
for cfg in C5 C2; do
  echo "== shards $cfg" >> gpurun_out/${T}.log
  timeout 900 python tools/shard_timing.py --config $cfg --shards 8 --steps 2 2>&1 | tail -9 | cut -c1-300 >> gpurun_out/${T}.log
done
KNNJ_JOIN_STATS=1 timeout 600 python tools/probe_steps.py --config C4 --steps 3 > gpurun_out/${T}_C4.log 2>&1
echo done
