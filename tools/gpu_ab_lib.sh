# A/B of prebuilt library variants (tools/_ab/lib_<tag>.so) on the bench, alternating: $@ = tags
for rep in ${REPS:-1 2}; do
  for v in "$@"; do
    cp tools/_ab/lib_$v.so paper_2603_09237_b200/libmorlax_b200.so
    timeout 300 python bench.py --no-legs --no-cpu-baseline --steps 10 > gpurun_out/ab.json 2>/dev/null
    python -c "
import json; d=json.load(open('gpurun_out/ab.json')); b=d['breakdown_ms_per_iter']
print('== $v', 'iter_ms %.3f' % d['ms_per_step'], ' '.join('%s %.3f' % (k.split('/')[1], b[k]['ms']) for k in b if k.startswith('update/')))"
  done
done
