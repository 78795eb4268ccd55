mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
T=${TAG:-r02k}
timeout 900 python -m pytest tests/test_gpu_mixed.py tests/test_gpu_stream.py -q -x > gpurun_out/${T}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_pytest.log
for q in 64 32; do
KNNJ_JOIN_STATS=1 timeout 900 python tools/probe_steps.py --config C4 --steps 2 --opt item_tc_min_q=$q > gpurun_out/${T}_C4_q$q.log 2>&1
done
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/${T}_bench.log 2>&1
echo done
