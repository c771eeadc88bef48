for i in 1 2; do timeout 900 python bench.py > gpurun_out/bench_full.json 2>/dev/null; python -c "
import json; d=json.load(open('gpurun_out/bench_full.json')); print('ms/iter', round(d['ms_per_step'],2), 'value', round(d['value']/1e6,2), 'e2e', round(d['e2e']['value']/1e6,2))"; done
for i in 1 2; do timeout 900 python bench.py --no-cpu-baseline --no-legs > gpurun_out/bench.json 2>/dev/null; python -c "
import json; d=json.load(open('gpurun_out/bench.json')); print('nolegs ms/iter', round(d['ms_per_step'],2), 'value', round(d['value']/1e6,2), 'e2e', round(d['e2e']['value']/1e6,2))"; done
