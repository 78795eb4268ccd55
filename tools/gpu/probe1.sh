set -x
nproc; free -g; nvidia-smi --query-gpu=name,memory.total --format=csv; df -h /tmp | tail -1
timeout 600 python bench.py --config C5 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/p1_c5.log 2>&1; echo rc=$?
tail -c 3000 gpurun_out/p1_c5.log
