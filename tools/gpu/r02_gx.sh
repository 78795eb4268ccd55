mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
T=${TAG:-r02gx}
timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/${T}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_pytest.log
for c in C5 C4 C2 NS; do timeout 900 python tools/probe_steps.py --config $c --steps 3 > gpurun_out/${T}_$c.log 2>&1; done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_c5_launches.csv \
   python tools/probe_steps.py --config C5 --steps 1 > gpurun_out/${T}_c5_ncu_launch.log 2>&1
echo done
