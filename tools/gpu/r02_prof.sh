# C5 phase timings after the sampler change, ncu full captures of the C5 and C4 level-0
# joins, compute-sanitizer over every kernel family, the NS bench line
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
T=${TAG:-r02c}
KNNJ_TRACE=1 timeout 300 python tools/probe_steps.py --config C5 --steps 3 > gpurun_out/${T}_c5_trace.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_tc -c 1 \
   -o gpurun_out/${T}_c5_join -f python tools/probe_steps.py --config C5 --steps 1 > gpurun_out/${T}_c5_ncu_join.log 2>&1
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:k_join -c 1 \
   -o gpurun_out/${T}_c4_join -f python tools/probe_steps.py --config C4 --steps 1 > gpurun_out/${T}_c4_ncu_join.log 2>&1
for tool in memcheck racecheck synccheck; do
  timeout 1200 compute-sanitizer --tool $tool --print-limit 50 python tools/sanitize_run.py > gpurun_out/${T}_sanitize_$tool.log 2>&1
  echo "rc=$?" >> gpurun_out/${T}_sanitize_$tool.log
done
timeout 900 python bench.py --config NS > gpurun_out/${T}_ns_bench.log 2>&1
echo done
