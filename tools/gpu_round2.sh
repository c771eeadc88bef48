# Round-2 profile pass (one GPU call): bench line, the per-launch list of one
# config-3 iteration, ncu --set full captures of the dominant kernels (each
# after its command ran clean without ncu). Outputs under gpurun_out/$TAG*.
TAG=${1:-r2}
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 900 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; echo "bench rc=$?"
timeout 600 python tools/profile_step.py c3 1 > /dev/null 2>&1; echo "profile_step rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/${TAG}_launches.csv python tools/profile_step.py c3 1 > gpurun_out/${TAG}_ncu_launch.log 2>&1; echo "ncu launches rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on --profile-from-start off --kernel-name-base demangled -k "regex:k_dm_adam|k_rollout_tc|k_head" -c 5 -o gpurun_out/${TAG}_prof_misc python tools/profile_step.py c3 1 > gpurun_out/${TAG}_ncu_misc.log 2>&1; echo "ncu misc rc=$?"
