mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
T=${TAG:-r02fin2}
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/${T}_pytest.log 2>&1
for c in C5 C2 NS C4; do KNNJ_TRACE=1 timeout 900 python tools/probe_steps.py --config $c --steps 3 > gpurun_out/${T}_$c.log 2>&1; done
echo done
