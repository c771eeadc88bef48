timeout -s KILL 900 python -m pytest -q -x -m gpu tests/test_gpu_parity.py tests/test_gpu_benchshape.py tests/test_gpu_multirank.py > gpurun_out/pytest_side.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_side.log
bash tools/gpu_ab_env.sh none
