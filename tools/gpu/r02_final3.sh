mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
T=${TAG:-r02f3}
timeout 900 python bench.py > gpurun_out/${T}_bench.log 2>&1
for cfg in C4 NS C2 C3 C1; do timeout 900 python bench.py --config $cfg --no-cpu-baseline > gpurun_out/${T}_bench_$cfg.log 2>&1; done
timeout 900 python bench.py --impl reference > gpurun_out/${T}_ref.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_c5_launches.csv \
   python tools/probe_steps.py --config C5 --steps 1 > gpurun_out/${T}_c5_ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_tc -s 1 -c 1 \
   -o gpurun_out/${T}_c5_join -f python tools/probe_steps.py --config C5 --steps 1 > gpurun_out/${T}_c5_ncu_join.log 2>&1
for cfg in C5 C2; do
  echo "== shards $cfg" >> gpurun_out/${T}_shards.log
  timeout 900 python tools/shard_timing.py --config $cfg --shards 8 --steps 2 2>&1 | tail -9 | cut -c1-300 >> gpurun_out/${T}_shards.log
done
echo done
