# full ncu capture of the C4 level-0 SIMT join (k_join<6, 128, 32>) and the C2 tcgen05 join
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 1500 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
   -k "regex:k_join<6, 128, 32>" -c 1 \
   -o gpurun_out/c4_join -f python tools/probe_steps.py --config C4 --steps 1 > gpurun_out/c4_ncu_join.log 2>&1
echo "c4 rc=$?" >> gpurun_out/c4_ncu_join.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c4_launches.csv \
   python tools/probe_steps.py --config C4 --steps 1 > gpurun_out/c4_ncu_launch.log 2>&1
echo done
