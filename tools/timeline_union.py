"""Fraction of one config-3 iteration in which no launch of ours is in flight
(per-launch CUDA events, all streams): the ceiling of what CUDA graphs could
recover from launch gaps."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2603_09237_b200 as mb  # noqa: E402

t = mb.Trainer(mb.TrainConfig(**bench.BASE["c3"]))
for i in range(3):
    t.iteration(i)
mb.LIB.morlax_trainer_profile_enable(t._h, 1)
t.iteration(3)
n = mb.LIB.morlax_trainer_profile_timeline_count(t._h)
spans = []
for i in range(n):
    name = C.create_string_buffer(64)
    st, a, b = C.c_int(), C.c_double(), C.c_double()
    mb.LIB.morlax_trainer_profile_timeline(t._h, i, name, C.byref(st), C.byref(a), C.byref(b))
    spans.append((a.value, b.value))
spans.sort()
lo, hi = spans[0][0], max(b for _, b in spans)
covered, cur_a, cur_b = 0.0, None, None
for a, b in spans:
    if cur_b is None or a > cur_b:
        if cur_b is not None:
            covered += cur_b - cur_a
        cur_a, cur_b = a, b
    else:
        cur_b = max(cur_b, b)
covered += cur_b - cur_a
print(f"iteration span {hi - lo:.3f} ms, covered by launches {covered:.3f} ms, idle {hi - lo - covered:.3f} ms")
