mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
T=${TAG:-r02i}
for v in "" "--opt fin_blocks=592 --opt copy_blocks=1184" "--opt fin_blocks=148 --opt copy_blocks=296" "--opt out_priority=0"; do
  echo "== $v" >> gpurun_out/${T}_C5.log
  KNNJ_TRACE=1 timeout 600 python tools/probe_steps.py --config C5 --steps 3 --pinned $v 2>&1 | grep -E "knnj\] pass: (join kernel|finalize)|step" | tail -4 | cut -c1-260 >> gpurun_out/${T}_C5.log
  timeout 600 python tools/probe_steps.py --config C5 --steps 2 $v 2>&1 | tail -1 | cut -c1-200 >> gpurun_out/${T}_C5.log
done
echo done
