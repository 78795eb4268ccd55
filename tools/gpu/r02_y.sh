mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
T=${TAG:-r02y}
timeout 1200 python -m pytest tests/test_gpu_stream.py tests/test_gpu_parity.py tests/test_gpu_shard_hist.py tests/test_gpu_mixed.py -q -x > gpurun_out/${T}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_pytest.log
for v in "" "--opt bound_grid=0" "--opt bound_group_span=4" "--opt bound_group_span=16"; do
  echo "== C5 $v" >> gpurun_out/${T}.log
  KNNJ_JOIN_STATS=1 timeout 600 python tools/probe_steps.py --config C5 --steps 3 $v 2>&1 | grep -E "pass:|step 2" | tail -4 | cut -c1-330 >> gpurun_out/${T}.log
done
for cfg in C2 NS C4; do
  echo "== $cfg" >> gpurun_out/${T}.log
  KNNJ_JOIN_STATS=1 timeout 600 python tools/probe_steps.py --config $cfg --steps 3 2>&1 | grep -E "pass:|step 2" | tail -4 | cut -c1-330 >> gpurun_out/${T}.log
done
echo done
