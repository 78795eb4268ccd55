mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
T=${TAG:-r02small}
for c in C5 C2 C4; do
 for o in 0 1; do
  timeout 900 python tools/probe_steps.py --config $c --steps 3 --opt tc_small_cta=$o > gpurun_out/${T}_${c}_$o.log 2>&1
 done
done
echo done
