# A/B: fused dM+Adam epilogue vs separate Adam
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -2
for f in 1 0; do MORLAX_FUSED_ADAM=$f timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_f$f.json 2>/dev/null; python -c "
import json; d=json.load(open('gpurun_out/bench_f$f.json')); print('fused=$f ms/iter', round(d['ms_per_step'],2)); print({k:v['ms'] for k,v in d['breakdown_ms_per_iter'].items()})"; done
