# rollout A/B variants (MB_ROLL_PROF phase clock), built on the box's copy only
for v in "$@"; do
  NVCC="nvcc -DMB_ROLL_PROF $v" bash paper_2603_09237_b200/build.sh > /dev/null 2>&1 || { echo "build failed $v"; continue; }
  echo "== $v"; timeout 300 python tools/profile_step.py c3 2 2>&1 | grep -E "rollout CTA0" | tail -2
done
