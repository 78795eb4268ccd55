mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
T=${TAG:-r02ld2}
for cfg in C5 C2 NS C4; do
  echo "== $cfg base" >> gpurun_out/${T}.log
  timeout 600 python tools/probe_steps.py --config $cfg --steps 3 2>&1 | grep -E "step 2" | tail -1 | cut -c1-250 >> gpurun_out/${T}.log
  echo "== $cfg ld2" >> gpurun_out/${T}.log
  KNNJ_LIB_PATH=paper_1810_04758_b200/ab/libknnj_ld2.so timeout 600 python tools/probe_steps.py --config $cfg --steps 3 2>&1 | grep -E "step 2" | tail -1 | cut -c1-250 >> gpurun_out/${T}.log
done
KNNJ_LIB_PATH=paper_1810_04758_b200/ab/libknnj_ld2.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_screen.py -q -x > gpurun_out/${T}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_pytest.log
echo done
