# A/B timings of engine options: AB_CASES="C5:lane_rare=0 C5:lane_rare=1 ..." (config:opt=v,opt=v)
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
for c in $AB_CASES; do
  cfg=${c%%:*}; opts=${c#*:}; args=""
  if [ "$opts" != "$c" ] && [ -n "$opts" ]; then for o in ${opts//,/ }; do args="$args --opt $o"; done; fi
  echo "== $c" >> gpurun_out/${TAG:-ab}.log
  KNNJ_JOIN_STATS=1 timeout 300 python tools/probe_steps.py --config $cfg --steps ${AB_STEPS:-3} $args 2>&1 | grep -E "join stats|hist grid|step" | tail -${AB_TAIL:-3} >> gpurun_out/${TAG:-ab}.log
done
echo done
