timeout 600 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -2
for g in 148 112 74; do MORLAX_GEMM_GRID=$g timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_g$g.json 2>/dev/null; python -c "
import json; d=json.load(open('gpurun_out/bench_g$g.json')); print('grid=$g ms/iter', round(d['ms_per_step'],2)); print({k:v['ms'] for k,v in d['breakdown_ms_per_iter'].items()})"; done
