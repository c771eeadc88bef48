set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
cat gpurun_out/bench.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/launches.csv python tools/profile_step.py c3 1 > gpurun_out/ncu_launch.log 2>&1; echo "ncu1 rc=$?"
python tools/launchsum.py gpurun_out/launches.csv
timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:"k_img_gemm|k_rollout_tc" -c 6 -o gpurun_out/prof_full python tools/profile_step.py c3 1 > gpurun_out/ncu_full.log 2>&1; echo "ncu2 rc=$?"
