mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
T=${TAG:-r02r}
timeout 300 python tools/small_run.py clusters:16:0.05 40000 18 32 join_chunks=1 > gpurun_out/${T}_plain.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_plain.log
timeout 2400 python -m pytest tests -m gpu -q -x --durations=10 > gpurun_out/${T}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_pytest.log
for cfg in C5 C4 C2 NS; do KNNJ_JOIN_STATS=1 timeout 900 python tools/probe_steps.py --config $cfg --steps 3 > gpurun_out/${T}_$cfg.log 2>&1; done
echo done
