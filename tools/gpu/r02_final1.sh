mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
T=${TAG:-r02f1}
timeout 2400 python -m pytest tests -m gpu -q -x --durations=8 > gpurun_out/${T}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_pytest.log
timeout 900 python bench.py > gpurun_out/${T}_bench.log 2>&1
for cfg in NS C2 C4; do timeout 900 python bench.py --config $cfg --no-cpu-baseline > gpurun_out/${T}_bench_$cfg.log 2>&1; done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_c5_launches.csv \
   python tools/probe_steps.py --config C5 --steps 1 > gpurun_out/${T}_c5_ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_tc -s 1 -c 1 \
   -o gpurun_out/${T}_c5_join -f python tools/probe_steps.py --config C5 --steps 1 > gpurun_out/${T}_c5_ncu_join.log 2>&1
echo done
