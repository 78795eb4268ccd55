mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
T=${TAG:-r02l}
timeout 2400 python -m pytest tests -m gpu -q -x --durations=15 > gpurun_out/${T}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_pytest.log
KNNJ_JOIN_STATS=1 timeout 900 python tools/probe_steps.py --config C4 --steps 2 > gpurun_out/${T}_C4.log 2>&1
for cfg in C2 NS C3 C1; do timeout 900 python tools/probe_steps.py --config $cfg --steps 3 > gpurun_out/${T}_$cfg.log 2>&1; done
echo done
