# GPU tests (args: pytest selection) + C5/C2 probe timings; everything into gpurun_out/
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout ${TEST_TIMEOUT:-1500} python -m pytest ${PYTEST_ARGS:-tests -m gpu -x -q} > gpurun_out/${TAG:-chk}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG:-chk}_pytest.log
for c in ${PROBE_CONFIGS:-C5}; do
  KNNJ_JOIN_STATS=1 timeout 300 python tools/probe_steps.py --config $c --steps 3 > gpurun_out/${TAG:-chk}_probe_$c.log 2>&1
done
echo done
