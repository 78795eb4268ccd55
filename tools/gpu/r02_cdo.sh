mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
T=${TAG:-r02cdo}
for o in 0 1; do timeout 900 python tools/probe_steps.py --config C5 --steps 3 --opt chunk_device_out=$o > gpurun_out/${T}_C5_$o.log 2>&1; done
timeout 900 python tools/probe_steps.py --config C5 --steps 3 --opt chunk_device_out=1 --opt fin_blocks=148 > gpurun_out/${T}_C5_1_fb148.log 2>&1
timeout 900 python tools/probe_steps.py --config C2 --steps 3 --opt chunk_device_out=1 > gpurun_out/${T}_C2_1.log 2>&1
timeout 900 python tools/probe_steps.py --config C2 --steps 3 > gpurun_out/${T}_C2_0.log 2>&1
echo done
