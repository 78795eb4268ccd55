mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
T=${TAG:-r02g}
timeout 900 python -m pytest tests/test_gpu_mixed.py tests/test_gpu_stream.py -q -x > gpurun_out/${T}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_pytest.log
KNNJ_TRACE=1 timeout 600 python tools/probe_steps.py --config C5 --steps 3 --pinned > gpurun_out/${T}_C5_pinned.log 2>&1
KNNJ_TRACE=1 timeout 600 python tools/probe_steps.py --config C5 --steps 3 --pinned --opt fin_blocks=0 > gpurun_out/${T}_C5_pinned_fb0.log 2>&1
KNNJ_JOIN_STATS=1 timeout 900 python tools/probe_steps.py --config C4 --steps 2 > gpurun_out/${T}_C4.log 2>&1
KNNJ_JOIN_STATS=1 timeout 900 python tools/probe_steps.py --config C4 --steps 2 --opt item_tc_min_q=32 > gpurun_out/${T}_C4_q32.log 2>&1
echo done
