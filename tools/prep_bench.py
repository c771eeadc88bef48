"""Serialised per-launch times (ncu-free): one config-3 iteration's launches by class, CUDA events per launch."""
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
n = mb.LIB.morlax_trainer_profile_count(t._h)
for i in range(n):
    name = C.create_string_buffer(64)
    pm, pf, pb, pc = C.c_double(), C.c_double(), C.c_double(), C.c_int64()
    mb.LIB.morlax_trainer_profile_get(t._h, i, name, C.byref(pm), C.byref(pf), C.byref(pb), C.byref(pc))
    nm = name.value.decode()
    if any(k in nm for k in sys.argv[1:]):
        print(f"{nm:28s} {pm.value:8.3f} ms / iter  {pc.value:4d} launches  {pm.value / pc.value * 1e3:7.1f} us each")
