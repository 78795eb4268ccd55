mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
T=${TAG:-r02e}
./tools/micro/pcie_write > gpurun_out/${T}_pcie.log 2>&1
for jc in 1 8; do
  KNNJ_JOIN_STATS=1 timeout 600 python tools/probe_steps.py --config C5 --steps 3 --opt join_chunks=$jc > gpurun_out/${T}_C5_jc$jc.log 2>&1
done
KNNJ_JOIN_STATS=1 timeout 600 python tools/probe_steps.py --config C5 --steps 3 --opt join_chunks=1 --opt kth_bound=0 > gpurun_out/${T}_C5_nobound.log 2>&1
for cfg in C2 NS; do
  KNNJ_JOIN_STATS=1 timeout 600 python tools/probe_steps.py --config $cfg --steps 3 --opt join_chunks=1 --opt kth_bound=0 > gpurun_out/${T}_${cfg}.log 2>&1
done
echo done
