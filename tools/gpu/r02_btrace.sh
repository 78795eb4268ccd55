mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
T=${TAG:-r02bt}
for o in 0 1; do
KNNJ_TRACE=1 timeout 600 python tools/probe_steps.py --config C5 --steps 2 --opt tc_small_cta=$o > gpurun_out/${T}_C5_$o.log 2>&1
done
echo done
