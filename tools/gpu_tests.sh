# selected GPU tests with their printed diagnostics: bash tools/gpu_tests.sh <pytest args>
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 1500 python -m pytest -s -q -m gpu "$@" > gpurun_out/pytest_sel.log 2>&1; echo "pytest rc=$?"
grep -E "errors|passed|failed|Error|assert|FAILED" gpurun_out/pytest_sel.log | tail -40
