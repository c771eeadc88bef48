# rollout change: env / rollout parity tests, bench, phase profile
timeout -s KILL 600 python -m pytest -q -m gpu tests/test_gpu_benchshape.py tests/test_gpu_parity.py -k "teacher or env or rollout or evaluate" > gpurun_out/pytest_rc.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_rc.log
grep -E "humanoid6 teacher" gpurun_out/pytest_rc.log | head -2
timeout -s KILL 240 python bench.py --no-legs --no-cpu-baseline --steps 10 > gpurun_out/rb.json 2>gpurun_out/rb.err; echo "bench rc=$?"
python -c "
import json; d=json.load(open('gpurun_out/rb.json')); b=d['breakdown_ms_per_iter']
print('iter_ms %.3f' % d['ms_per_step'], 'rollout %.3f' % b['rollout/rollout']['ms'])" || tail -5 gpurun_out/rb.err
bash tools/gpu_rollprof.sh
