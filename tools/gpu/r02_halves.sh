mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
T=${TAG:-r02hv}
timeout 900 python -m pytest tests/test_gpu_shard_hist.py -q -x -k "halves or knobs" > gpurun_out/${T}_pytest.log 2>&1
for c in C5 C2 NS; do timeout 900 python tools/probe_steps.py --config $c --steps 3 > gpurun_out/${T}_$c.log 2>&1; done
KNNJ_TRACE=1 timeout 600 python tools/probe_steps.py --config C5 --steps 1 > gpurun_out/${T}_C5_trace.log 2>&1
echo done
