# C5 diagnostics: join stats, join timing decomposition, ncu launch list + join/hist captures
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
KNNJ_JOIN_STATS=1 timeout 300 python tools/probe_steps.py --config C5 --steps 2 > gpurun_out/c5_stats.log 2>&1
for m in 1 2 3; do KNNJ_JOIN_DBG=$m timeout 300 python tools/probe_steps.py --config C5 --steps 2 > gpurun_out/c5_dbg$m.log 2>&1; done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c5_launches.csv \
   python tools/probe_steps.py --config C5 --steps 1 > gpurun_out/c5_ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
   -k "regex:k_tc<.int.1, .int.2, .int.4, .bool.0" -c 1 \
   -o gpurun_out/c5_join -f python tools/probe_steps.py --config C5 --steps 1 > gpurun_out/c5_ncu_join.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
   -k "regex:k_tc<.int.1, .int.2, .int.4, .bool.1" -c 2 \
   -o gpurun_out/c5_hist -f python tools/probe_steps.py --config C5 --steps 1 > gpurun_out/c5_ncu_hist.log 2>&1
echo done
