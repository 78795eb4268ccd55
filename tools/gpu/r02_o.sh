mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
T=${TAG:-r02o}
for cfg in C5 C2 NS; do
  KNNJ_JOIN_STATS=1 timeout 600 python tools/probe_steps.py --config $cfg --steps 3 > gpurun_out/${T}_${cfg}_base.log 2>&1
  KNNJ_JOIN_STATS=1 KNNJ_LIB_PATH=paper_1810_04758_b200/ab/libknnj_lane.so timeout 600 python tools/probe_steps.py --config $cfg --steps 3 > gpurun_out/${T}_${cfg}_lane.log 2>&1
done
KNNJ_LIB_PATH=paper_1810_04758_b200/ab/libknnj_lane.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_screen.py -q -x > gpurun_out/${T}_lane_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_lane_pytest.log
echo done
for cfg in C5 C2 NS; do
  KNNJ_JOIN_STATS=1 timeout 600 python tools/probe_steps.py --config $cfg --steps 3 --opt tc_small_cta=1 > gpurun_out/${T}_${cfg}_small.log 2>&1
done
timeout 900 python -m pytest tests/test_gpu_shard_hist.py -q -x -k "knobs" > gpurun_out/${T}_small_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_small_pytest.log
echo done2
