# new rollout: teacher-forced parity first (short kill timeout: a hang must not hold the box), then timing
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout -s KILL 240 python -m pytest -s -q -m gpu tests/test_gpu_benchshape.py -k teacher > gpurun_out/pytest_tf.log 2>&1; echo "teacher rc=$?"
grep -E "errors|passed|failed|Error|assert|FAILED|normwise" gpurun_out/pytest_tf.log | tail -20
timeout -s KILL 240 python bench.py --no-legs --no-cpu-baseline --steps 5 > gpurun_out/rb.json 2>gpurun_out/rb.err; echo "bench rc=$?"
python -c "
import json; d=json.load(open('gpurun_out/rb.json')); b=d['breakdown_ms_per_iter']
print('iter_ms %.3f' % d['ms_per_step'], 'rollout %.3f' % b['rollout/rollout']['ms'])" || tail -5 gpurun_out/rb.err
