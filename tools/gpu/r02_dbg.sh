mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
T=${TAG:-r02p}
timeout 600 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_stream.py -q -x -k "identical and clusters" > gpurun_out/${T}_memcheck_stream.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_memcheck_stream.log
timeout 600 compute-sanitizer --tool memcheck --print-limit 20 python tools/sanitize_run.py > gpurun_out/${T}_memcheck_sanitize.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_memcheck_sanitize.log
echo done
