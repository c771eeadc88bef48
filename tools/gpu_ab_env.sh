# A/B of an environment knob: VAR=name VALUES="a b c" bash tools/gpu_ab_env.sh
for v in $VALUES; do
  export $VAR=$v
  timeout 300 python tools/profile_step.py c3 4 >/dev/null 2>&1
  MORLAX_HOST_TIMING=1 timeout 300 python tools/profile_step.py c3 6 2>&1 | grep "host enqueue" | tail -4 | awk -v v=$v '{print v, $NF}'
done
