mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
T=${TAG:-r02q}
timeout 300 python tools/small_run.py clusters:16:0.05 40000 18 32 join_chunks=1 > gpurun_out/${T}_plain.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_plain.log
timeout 600 /usr/local/cuda/bin/cuda-gdb -batch -ex "set pagination off" -ex run -ex bt -ex "info threads" --args python tools/small_run.py clusters:16:0.05 40000 18 32 join_chunks=1 > gpurun_out/${T}_gdb.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_gdb.log
timeout 300 python tools/small_run.py uniform 60000 4 32 > gpurun_out/${T}_u4.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_u4.log
echo done
