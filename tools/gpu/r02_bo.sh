mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
T=${TAG:-r02bo}
for cfg in C5 C2 NS C4; do
for lib in "" paper_1810_04758_b200/ab/libknnj_bo.so paper_1810_04758_b200/ab/libknnj_bo2.so; do
  echo "== $cfg lib=$lib" >> gpurun_out/${T}.log
  KNNJ_LIB_PATH=$lib timeout 600 python tools/probe_steps.py --config $cfg --steps 3 2>&1 | grep -E "step 2" | tail -1 | cut -c1-250 >> gpurun_out/${T}.log
done
done
KNNJ_LIB_PATH=paper_1810_04758_b200/ab/libknnj_bo.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_screen.py -q -x > gpurun_out/${T}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_pytest.log
echo done
