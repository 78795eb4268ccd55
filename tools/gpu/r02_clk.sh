mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
T=${TAG:-r02clk}
KNNJ_JOIN_STATS=1 KNNJ_LIB_PATH=paper_1810_04758_b200/ab/clk/libknnj_b200.so timeout 600 python tools/probe_steps.py --config C5 --steps 2 > gpurun_out/${T}_C5.log 2>&1
KNNJ_JOIN_STATS=1 timeout 600 python tools/probe_steps.py --config C5 --steps 2 > gpurun_out/${T}_C5_plain.log 2>&1
KNNJ_JOIN_STATS=1 KNNJ_LIB_PATH=paper_1810_04758_b200/ab/clk/libknnj_b200.so timeout 600 python tools/probe_steps.py --config C2 --steps 2 > gpurun_out/${T}_C2.log 2>&1
timeout 600 python tools/probe_steps.py --config C5 --steps 2 --opt tc_small_cta=1 > gpurun_out/${T}_C5_small.log 2>&1
echo done
