# parity tests + bench (one GPU call); serialised-chain breakdown too
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/pytest_gpu.log
for f in 0 1; do MORLAX_ONE_STREAM=$f timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_s$f.json 2> gpurun_out/bench.err; echo "bench rc=$?"; tail -3 gpurun_out/bench.err
python -c "
import json; d=json.load(open('gpurun_out/bench_s$f.json')); print('one_stream=$f ms/iter', round(d['ms_per_step'],2), 'launches', d['gpu_launches']); print({k:(v['ms'],v['launches']) for k,v in d['breakdown_ms_per_iter'].items()})"; done
