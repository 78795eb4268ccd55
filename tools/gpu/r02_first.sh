# round-2 first GPU pass: gpu tests, default bench, launch list of the bench
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r02a_smi.txt
timeout 2400 python -m pytest tests -m gpu -q -x --durations=25 > gpurun_out/r02a_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r02a_pytest.log
timeout 900 python bench.py > gpurun_out/r02a_bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/r02a_bench.log
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r02a_ref.log 2>&1; echo "ref rc=$?" >> gpurun_out/r02a_ref.log
echo done
