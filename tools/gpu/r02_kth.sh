mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
T=${TAG:-r02kth}
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/${T}_pytest.log 2>&1
KNNJ_JOIN_STATS=1 KNNJ_LIB_PATH=paper_1810_04758_b200/ab/clk/libknnj_b200.so timeout 600 python tools/probe_steps.py --config C5 --steps 2 > gpurun_out/${T}_C5_clk.log 2>&1
for c in C5 C2 NS C4; do timeout 900 python tools/probe_steps.py --config $c --steps 3 > gpurun_out/${T}_$c.log 2>&1; done
echo done
