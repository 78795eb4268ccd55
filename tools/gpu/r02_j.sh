mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
T=${TAG:-r02j}
timeout 900 python -m pytest tests/test_gpu_mixed.py -q -x > gpurun_out/${T}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_pytest.log
for v in "--opt copy_blocks=37" "--opt copy_blocks=74" "--opt copy_blocks=148" "--opt copy_blocks=148 --opt fin_blocks=148" "--opt copy_blocks=74 --opt join_chunks=16"; do
  echo "== $v" >> gpurun_out/${T}_C5.log
  KNNJ_TRACE=1 timeout 600 python tools/probe_steps.py --config C5 --steps 3 --pinned $v 2>&1 | grep -E "knnj\] pass: (join kernel|finalize)|step" | tail -4 | cut -c1-230 >> gpurun_out/${T}_C5.log
done
KNNJ_JOIN_STATS=1 timeout 900 python tools/probe_steps.py --config C4 --steps 2 > gpurun_out/${T}_C4.log 2>&1
echo done
