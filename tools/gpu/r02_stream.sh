# streamed results + radius bound: parity tests, then timings (A/B) on C5, C2, NS, C4
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
T=${TAG:-r02d}
timeout 1500 python -m pytest tests/test_gpu_stream.py tests/test_gpu_parity.py tests/test_gpu_shard_hist.py tests/test_gpu_screen.py -q -x > gpurun_out/${T}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_pytest.log
for cfg in C5 C2; do
  KNNJ_JOIN_STATS=1 KNNJ_LIB_PATH=paper_1810_04758_b200/ab/libknnj_nobatch.so timeout 600 python tools/probe_steps.py --config $cfg --steps 3 > gpurun_out/${T}_${cfg}_nobatch.log 2>&1
  KNNJ_JOIN_STATS=1 timeout 600 python tools/probe_steps.py --config $cfg --steps 3 --opt kth_bound=0 > gpurun_out/${T}_${cfg}_batch.log 2>&1
  KNNJ_JOIN_STATS=1 timeout 600 python tools/probe_steps.py --config $cfg --steps 3 > gpurun_out/${T}_${cfg}_bound.log 2>&1
done
for cfg in NS C4 C3 C1; do
  KNNJ_JOIN_STATS=1 timeout 600 python tools/probe_steps.py --config $cfg --steps 3 > gpurun_out/${T}_${cfg}_bound.log 2>&1
done
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/${T}_bench.log 2>&1
echo done
