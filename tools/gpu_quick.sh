# parity tests + bench (one GPU call)
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"; tail -5 gpurun_out/bench.err
python -c "
import json; d=json.load(open('gpurun_out/bench.json')); print('ms/iter', d['ms_per_step'], 'value', d['value'], 'e2e', d['e2e']['value'], 'launches', d['gpu_launches']); print(d['roofline']); print(d['cpu_baseline']); print(json.dumps(d['other_configs'], indent=1)); print(d['pareto'])
"
