mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
T=${TAG:-r02n}
timeout 900 python -m pytest tests/test_gpu_stream.py tests/test_gpu_parity.py tests/test_gpu_mixed.py -q -x > gpurun_out/${T}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_pytest.log
for cfg in C5 C4; do KNNJ_TRACE=1 KNNJ_JOIN_STATS=1 timeout 900 python tools/probe_steps.py --config $cfg --steps 3 > gpurun_out/${T}_$cfg.log 2>&1; done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_join -c 2 \
   -o gpurun_out/${T}_c4_simt -f python tools/probe_steps.py --config C4 --steps 1 > gpurun_out/${T}_c4_ncu_simt.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_tc -s 1 -c 1 \
   -o gpurun_out/${T}_c4_tc -f python tools/probe_steps.py --config C4 --steps 1 > gpurun_out/${T}_c4_ncu_tc.log 2>&1
echo done
