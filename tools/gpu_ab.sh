ls oracle/_ref/ | head -3
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "checkpoint or single_rank" 2>&1 | tail -5
