mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
T=${TAG:-r02f}
timeout 900 python -m pytest tests/test_gpu_stream.py -q -x > gpurun_out/${T}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_pytest.log
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/${T}_bench.log 2>&1
for q in 995 999; do
  KNNJ_JOIN_STATS=1 timeout 600 python tools/probe_steps.py --config C5 --steps 3 --opt kth_bound_q=$q > gpurun_out/${T}_C5_q$q.log 2>&1
done
for fb in 0 148; do
  timeout 600 python tools/probe_steps.py --config C5 --steps 3 --opt fin_blocks=$fb > gpurun_out/${T}_C5_fb$fb.log 2>&1
done
echo done
