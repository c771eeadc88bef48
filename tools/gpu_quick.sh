# parity tests + bench + GEMM microbenchmarks (one GPU call)
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
python -c "
import json; d=json.load(open('gpurun_out/bench.json')); print('ms/iter', d['ms_per_step'], 'value', d['value'], 'e2e', d['e2e']['value']); print(d['roofline'])
for k,v in d['breakdown_ms_per_iter'].items(): print(k, v)
"
timeout 300 python tools/gemm_bench.py; timeout 300 python tools/gemm_variants.py
