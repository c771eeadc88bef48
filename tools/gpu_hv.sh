timeout 900 python -m pytest tests -m gpu -x -q -k "hypervolume or pareto" 2>&1 | tail -5
timeout 300 python tools/hv_bench.py
