timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for v in 1; do MORLAX_FUSED_ADAM=$v timeout 600 python bench.py --no-cpu-baseline --no-legs > gpurun_out/bench.json 2>/dev/null; python -c "
import json; d=json.load(open('gpurun_out/bench.json')); print('fused=$v ms/iter', round(d['ms_per_step'],2), 'launches', d['gpu_launches']); print({k:v['ms'] for k,v in d['breakdown_ms_per_iter'].items()})"; done
bash tools/gpu_ncu_one.sh "k_head" 2 head 2
