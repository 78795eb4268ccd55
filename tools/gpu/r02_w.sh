mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
T=${TAG:-r02w}
timeout 900 python -m pytest tests/test_gpu_stream.py -q -x > gpurun_out/${T}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_pytest.log
for v in "" "--opt rows_bulk=0" "--opt copy_blocks=148" "--opt copy_blocks=37"; do
  echo "== C5 pinned $v" >> gpurun_out/${T}.log
  KNNJ_TRACE=1 timeout 600 python tools/probe_steps.py --config C5 --steps 3 --pinned $v 2>&1 | grep -E "knnj\] pass: (join kernel|finalize)|step 2" | tail -4 | cut -c1-230 >> gpurun_out/${T}.log
done
echo done
