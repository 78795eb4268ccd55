# C5 + C4 diagnostics: join stats, ncu launch lists, full captures of the dominant kernels
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
T=${TAG:-r02b}
KNNJ_JOIN_STATS=1 timeout 300 python tools/probe_steps.py --config C5 --steps 2 > gpurun_out/${T}_c5_stats.log 2>&1
KNNJ_JOIN_STATS=1 timeout 300 python tools/probe_steps.py --config C4 --steps 2 > gpurun_out/${T}_c4_stats.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_c5_launches.csv \
   python tools/probe_steps.py --config C5 --steps 1 > gpurun_out/${T}_c5_ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
   -k "regex:k_tc<1, 2, 4, false" -c 1 \
   -o gpurun_out/${T}_c5_join -f python tools/probe_steps.py --config C5 --steps 1 > gpurun_out/${T}_c5_ncu_join.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
   -k "regex:k_hist_grid" -c 2 \
   -o gpurun_out/${T}_c5_hist -f python tools/probe_steps.py --config C5 --steps 1 > gpurun_out/${T}_c5_ncu_hist.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_c4_launches.csv \
   python tools/probe_steps.py --config C4 --steps 1 > gpurun_out/${T}_c4_ncu_launch.log 2>&1
timeout 1500 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
   -k "regex:k_join<6" -c 1 \
   -o gpurun_out/${T}_c4_join -f python tools/probe_steps.py --config C4 --steps 1 > gpurun_out/${T}_c4_ncu_join.log 2>&1
echo done
