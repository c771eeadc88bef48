# ncu --set full of one config-3 rollout launch (after a clean run without ncu)
TAG=${1:-roll}
timeout 300 python tools/profile_step.py c3 1 > /dev/null 2>&1; echo "profile_step rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:k_rollout_tc -c 1 -o gpurun_out/${TAG} python tools/profile_step.py c3 1 > gpurun_out/${TAG}_ncu.log 2>&1; echo "ncu rc=$?"
