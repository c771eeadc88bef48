# A/B of env settings on the bench (in-situ): each argument is an env assignment list ("X=1 Y=2" or "none")
for v in "$@"; do
  if [ "$v" = none ]; then vv=""; else vv="$v"; fi
  for rep in 1 2; do
    env $vv timeout 300 python bench.py --no-legs --no-cpu-baseline --steps 10 > gpurun_out/ab.json 2>/dev/null
    python -c "
import json; d=json.load(open('gpurun_out/ab.json')); print('== $v', 'iter_ms %.3f' % d['ms_per_step'], d.get('clocks'))"
  done
done
