mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
T=${TAG:-r02cp}
for cb in 74 148 296; do
timeout 900 python tools/probe_steps.py --config C5 --steps 3 --pinned --opt copy_blocks=$cb > gpurun_out/${T}_C5_cb$cb.log 2>&1
done
timeout 900 python tools/probe_steps.py --config C5 --steps 3 --pinned --opt copy_blocks=148 --opt join_chunks=32 > gpurun_out/${T}_C5_cb148_ch32.log 2>&1
timeout 900 python tools/probe_steps.py --config C5 --steps 3 --pinned --opt copy_blocks=148 --opt fin_blocks=148 > gpurun_out/${T}_C5_cb148_fb148.log 2>&1
echo done
