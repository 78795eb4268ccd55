mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
T=${TAG:-r02sw}
timeout 900 python tools/probe_steps.py --config C5 --steps 3 --opt sweep_order=0 > gpurun_out/${T}_C5_nosweep.log 2>&1
timeout 900 python tools/probe_steps.py --config C5 --steps 3 --opt box_filter=0 > gpurun_out/${T}_C5_nofilter.log 2>&1
echo done
