# A/B: the worktree _ab_old (round-1 rollout) vs this tree, both MB_ROLL_PROF builds
echo "== old"; (cd _ab_old && timeout 300 python tools/profile_step.py c3 2 2>&1 | grep -E "rollout CTA0" | tail -1)
NVCC="nvcc -DMB_ROLL_PROF" bash paper_2603_09237_b200/build.sh > /dev/null 2>&1
echo "== new"; timeout 300 python tools/profile_step.py c3 2 2>&1 | grep -E "rollout CTA0" | tail -2
