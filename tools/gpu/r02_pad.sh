mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
T=${TAG:-r02pad}
timeout 2400 python -m pytest tests -m gpu -q -x --durations=5 > gpurun_out/${T}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_pytest.log
for cfg in C5 C2; do
  echo "== $cfg" >> gpurun_out/${T}.log
  timeout 600 python tools/probe_steps.py --config $cfg --steps 3 2>&1 | grep -E "step 2" | tail -1 | cut -c1-250 >> gpurun_out/${T}.log
done
echo done
