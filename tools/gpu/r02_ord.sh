mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
T=${TAG:-r02ord}
timeout 900 python tools/probe_steps.py --config C5 --steps 3 --opt box_filter=0 > gpurun_out/${T}_C5_nofilter.log 2>&1
timeout 900 python tools/probe_steps.py --config C5 --steps 3 > gpurun_out/${T}_C5.log 2>&1
timeout 900 python tools/probe_steps.py --config C4 --steps 2 > gpurun_out/${T}_C4.log 2>&1
timeout 900 python tools/probe_steps.py --config C2 --steps 3 > gpurun_out/${T}_C2.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/${T}_pytest.log 2>&1
echo done
