mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
T=${TAG:-r02h}
timeout 900 python -m pytest tests/test_gpu_mixed.py tests/test_gpu_stream.py -q -x > gpurun_out/${T}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_pytest.log
for jc in 8 16; do
  KNNJ_TRACE=1 timeout 600 python tools/probe_steps.py --config C5 --steps 3 --pinned --opt join_chunks=$jc > gpurun_out/${T}_C5_pinned_jc$jc.log 2>&1
done
KNNJ_TRACE=1 timeout 600 python tools/probe_steps.py --config C5 --steps 3 --pinned --opt join_chunks=16 --opt copy_blocks=0 > gpurun_out/${T}_C5_pinned_cb0.log 2>&1
KNNJ_JOIN_STATS=1 timeout 900 python tools/probe_steps.py --config C4 --steps 2 > gpurun_out/${T}_C4.log 2>&1
echo done
