timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for i in 1 2; do timeout 600 python bench.py --no-cpu-baseline --no-legs > gpurun_out/bench.json 2>/dev/null; python -c "
import json; d=json.load(open('gpurun_out/bench.json')); print('ms/iter', round(d['ms_per_step'],2), 'launches', d['gpu_launches']); print({k:v['ms'] for k,v in d['breakdown_ms_per_iter'].items()})"; done
timeout 300 python - <<'PY'
import bench, paper_2603_09237_b200 as mb
for _ in range(2):
    print('c2 us', round(bench.leg_c2(mb, 1500.0)["value"], 1))
PY
