"""evaluate_params on the device at the reference's default EvalConfig
(grid_resolution 10, 8 episodes) for the config-3 actor (mo-humanoid6, 6
objectives: 3003 grid points)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_09237_b200 as mb  # noqa: E402

spec = mb.HypernetSpec(6, 256, [256], [45, 256, 256, 12], True, True)
flat = mb.init_hypernet(spec, 2)
mb.evaluate_params(spec, flat, "mo-humanoid6", 2, 8, 1)
t0 = time.perf_counter()
W, R = mb.evaluate_params(spec, flat, "mo-humanoid6", 10, 8, 1)
print(f"evaluate_params: {len(W)} points x 8 episodes in {1e3 * (time.perf_counter() - t0):.1f} ms; "
      f"mean return[0] {R[0]}")
