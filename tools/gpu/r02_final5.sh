mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
T=${TAG:-r02f5}
timeout 1800 python -m pytest tests -m gpu -q -x --durations=8 > gpurun_out/${T}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_pytest.log
timeout 900 python bench.py > gpurun_out/${T}_bench.log 2>&1
for cfg in C4 NS C2 C3 C1; do timeout 900 python bench.py --config $cfg --no-cpu-baseline > gpurun_out/${T}_bench_$cfg.log 2>&1; done
timeout 900 python bench.py --impl reference > gpurun_out/${T}_ref.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/${T}_smoke.log
echo done
