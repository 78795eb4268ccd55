#!/bin/bash
# One gpurun pass: GPU parity tests, smoke, the default bench line, the ncu launch list
# and one full ncu capture of the join kernel. Everything lands in gpurun_out/.
#   env: PYTEST_ARGS (default "tests -m gpu -x -q"), BENCH_ARGS, SKIP_NCU, NCU_KERNEL (regex on
#        the demangled name, default the tcgen05 join), NCU_BENCH_ARGS
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt 2>&1
nproc > gpurun_out/nproc.txt; lscpu > gpurun_out/lscpu.txt 2>&1
if [ -z "$SKIP_TESTS" ]; then
timeout 1200 python -m pytest ${PYTEST_ARGS:-tests -m gpu -x -q} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
fi
if [ -z "$SKIP_BENCH" ]; then
timeout 900 python bench.py ${BENCH_ARGS:-} > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
fi
if [ -z "$SKIP_NCU" ]; then
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
   python bench.py --steps 1 --warmup 0 --no-cpu-baseline ${NCU_BENCH_ARGS:-} > gpurun_out/ncu_launch_run.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
   -k "regex:${NCU_KERNEL:-k_tc<.int.1, .int.2, .int.4, .bool.0}" -c 1 \
   -o gpurun_out/prof -f python bench.py --steps 1 --warmup 0 --no-cpu-baseline ${NCU_BENCH_ARGS:-} > gpurun_out/ncu_full.log 2>&1
fi
echo done
