# rollout in-situ time (bench breakdown, CUDA events) for build variants: $@ = NVCC define sets
for v in "$@"; do
  NVCC="nvcc $v" bash paper_2603_09237_b200/build.sh > /dev/null 2>&1 || { echo "build failed $v"; continue; }
  timeout 300 python bench.py --no-legs --no-cpu-baseline --steps 5 > gpurun_out/rb.json 2>/dev/null
  python -c "
import json,sys; d=json.load(open('gpurun_out/rb.json')); b=d['breakdown_ms_per_iter']
print('== $v', 'iter_ms %.3f' % d['ms_per_step'], 'rollout %.3f' % b['rollout/rollout']['ms'], 'noise', b.get('rollout/noise',{}).get('ms'))"
done
