mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
T=${TAG:-r02fin}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_finalize -s 2 -c 1 \
   -o gpurun_out/${T}_c5_fin -f python tools/probe_steps.py --config C5 --steps 1 > gpurun_out/${T}_c5_ncu_fin.log 2>&1
echo done
