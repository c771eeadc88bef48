# GEMM + rollout parity subset, then two bench runs (kill timeouts: a hang must not hold the box)
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout -s KILL 600 python -m pytest -q -x -m gpu tests/test_gpu_tcgemm.py tests/test_gpu_benchshape.py > gpurun_out/pytest_qc.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/pytest_qc.log
for rep in 1 2; do
timeout -s KILL 240 python bench.py --no-legs --no-cpu-baseline --steps 10 > gpurun_out/qc.json 2>gpurun_out/qc.err; echo "bench rc=$?"
python -c "
import json; d=json.load(open('gpurun_out/qc.json')); b=d['breakdown_ms_per_iter']
print('iter_ms %.3f' % d['ms_per_step'], ' '.join('%s %.3f' % (k, v['ms']) for k, v in sorted(b.items(), key=lambda x: -x[1]['ms'])[:12]))" || tail -5 gpurun_out/qc.err
done
