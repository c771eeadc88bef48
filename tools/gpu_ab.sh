timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for v in 1 1; do timeout 600 python bench.py --no-cpu-baseline --no-legs > gpurun_out/bench.json 2>/dev/null; python -c "
import json; d=json.load(open('gpurun_out/bench.json')); print('ms/iter', round(d['ms_per_step'],2))"; done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/launches_ab.csv python tools/profile_step.py c3 1 > /dev/null 2>&1; echo "ncu rc=$?"
