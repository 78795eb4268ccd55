mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
T=${TAG:-r02f6}
timeout 900 python bench.py > gpurun_out/${T}_bench.log 2>&1
for cfg in C4 NS C2 C3 C1; do timeout 900 python bench.py --config $cfg --no-cpu-baseline > gpurun_out/${T}_bench_$cfg.log 2>&1; done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_c5_launches.csv \
   python tools/probe_steps.py --config C5 --steps 1 > gpurun_out/${T}_c5_ncu_launch.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/${T}_smoke.log
echo done
