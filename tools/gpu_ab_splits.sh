for sp in ${SPLITS:-148 74}; do
  echo "splits $sp"; MORLAX_DF_SPLITS=$sp timeout 300 python tools/profile_step.py c3 4 >/dev/null 2>&1
  MORLAX_DF_SPLITS=$sp MORLAX_HOST_TIMING=1 timeout 300 python tools/profile_step.py c3 6 2>&1 | grep "host enqueue" | tail -3
done
