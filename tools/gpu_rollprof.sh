# rollout phase timing (CTA 0's clock) from an MB_ROLL_PROF build, on the box's copy only
NVCC="nvcc -DMB_ROLL_PROF $*" bash paper_2603_09237_b200/build.sh > /dev/null 2>&1 || { echo build failed; exit 1; }
timeout 300 python tools/profile_step.py c3 2 2>&1 | grep -E "rollout CTA0" | tail -4
