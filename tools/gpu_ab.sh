timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench.json 2>/dev/null; python -c "
import json; d=json.load(open('gpurun_out/bench.json')); print('ms/iter', round(d['ms_per_step'],2), 'e2e', d['e2e']['value'], 'launches', d['gpu_launches'], 'c2 us', round(d['other_configs']['config2']['value'],1), 'c4 ms', round(d['other_configs']['config4']['ms_per_step'],2)); print({k:v['ms'] for k,v in d['breakdown_ms_per_iter'].items()})"
