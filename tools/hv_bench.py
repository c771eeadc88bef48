"""Exact (device WFG) and Monte-Carlo hypervolume timings on the config-5 front."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_09237_b200 as mb  # noqa: E402

rng = np.random.default_rng(4)
w = rng.dirichlet(np.ones(6), size=1024)
pts = w / np.linalg.norm(w, axis=1, keepdims=True) + rng.normal(0, 0.02, (1024, 6))
ref = -np.ones(6)
mb.hypervolume_exact(pts[:64], ref)
for n in (256, 512, 1024):
    t0 = time.perf_counter()
    v, _ = mb.hypervolume_exact(pts[:n], ref)
    print(f"exact n={n}: {v!r} {1e3 * (time.perf_counter() - t0):.1f} ms")
t0 = time.perf_counter()
print("mc:", mb.hypervolume_detailed(pts, ref), f"{1e3 * (time.perf_counter() - t0):.1f} ms")
