mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
T=${TAG:-r02fin}
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_stream.py tests/test_gpu_shard_hist.py -q -x > gpurun_out/${T}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_pytest.log
for cfg in C5 C2; do
  echo "== $cfg" >> gpurun_out/${T}.log
  KNNJ_TRACE=1 timeout 600 python tools/probe_steps.py --config $cfg --steps 3 2>&1 | grep -E "pass: (join kernel|finalize)|step 2" | tail -5 | cut -c1-300 >> gpurun_out/${T}.log
done
echo done
