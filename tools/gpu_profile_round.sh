# Round profile: bench line, per-launch list of one config-3 iteration, and
# ncu --set full captures of the top kernels (each after its command ran
# clean without ncu). Outputs under gpurun_out/.
set -x
timeout 900 python bench.py > gpurun_out/bench_round.json 2> gpurun_out/bench_round.err; echo "bench rc=$?"
timeout 600 python tools/profile_step.py c3 1 > /dev/null 2>&1; echo "profile_step rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/launches_round.csv python tools/profile_step.py c3 1 > gpurun_out/ncu_launch_round.log 2>&1; echo "ncu launches rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on --profile-from-start off --kernel-name-base demangled -k "regex:k_dm_adam|k_head|k_rollout_tc|k_gather_minibatch|k_pack_weights|k_gtheta_prep" -c 10 -o gpurun_out/prof_round_misc python tools/profile_step.py c3 1 > gpurun_out/ncu_round_misc.log 2>&1; echo "ncu misc rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on --profile-from-start off --kernel-name-base demangled -k "regex:k_img_gemm" -s 2 -c 12 -o gpurun_out/prof_round_gemm python tools/profile_step.py c3 1 > gpurun_out/ncu_round_gemm.log 2>&1; echo "ncu gemm rc=$?"
