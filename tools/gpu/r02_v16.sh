mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
T=${TAG:-r02v16}
for lib in "" "paper_1810_04758_b200/ab/libknnj_v16.so"; do
for v in "" "--opt copy_blocks=148"; do
  echo "== C5 pinned lib=$lib $v" >> gpurun_out/${T}.log
  KNNJ_LIB_PATH=$lib KNNJ_TRACE=1 timeout 600 python tools/probe_steps.py --config C5 --steps 3 --pinned $v 2>&1 | grep -E "knnj\] pass: (join kernel|finalize)|step 2" | tail -3 | cut -c1-230 >> gpurun_out/${T}.log
done
done
KNNJ_LIB_PATH=paper_1810_04758_b200/ab/libknnj_v16.so timeout 600 python -m pytest tests/test_gpu_stream.py -q -x > gpurun_out/${T}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_pytest.log
echo done
