mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
T=${TAG:-r02fb}
timeout 1500 python -m pytest tests/test_gpu_mixed.py tests/test_gpu_parity.py tests/test_gpu_shard_hist.py tests/test_gpu_screen.py tests/test_gpu_adapter.py -q -x > gpurun_out/${T}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_pytest.log
for v in "" "--opt fallback_group_span=0"; do
for cfg in C4 C3 C1; do
  echo "== $cfg $v" >> gpurun_out/${T}.log
  timeout 600 python tools/probe_steps.py --config $cfg --steps 3 $v 2>&1 | grep -E "step 2" | tail -1 | cut -c1-300 >> gpurun_out/${T}.log
done
done
echo done
