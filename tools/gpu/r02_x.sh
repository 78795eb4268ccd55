mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
T=${TAG:-r02x}
timeout 2400 python -m pytest tests -m gpu -q -x --durations=5 > gpurun_out/${T}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_pytest.log
for cfg in C5 C2 NS C4 C3 C1; do KNNJ_JOIN_STATS=1 timeout 900 python tools/probe_steps.py --config $cfg --steps 3 > gpurun_out/${T}_$cfg.log 2>&1; done
KNNJ_TRACE=1 timeout 600 python tools/probe_steps.py --config C5 --steps 3 --pinned > gpurun_out/${T}_C5_pinned.log 2>&1
timeout 900 python bench.py > gpurun_out/${T}_bench.log 2>&1
timeout 900 python bench.py --impl reference > gpurun_out/${T}_ref.log 2>&1
echo done
