"""In-situ timeline of one config-3 iteration from the trainer's per-launch
CUDA events (morlax_trainer_profile_timeline): prints the launches of one
minibatch (stream, start, end, class) and per-stream busy fractions.
  python tools/timeline.py [minibatch index]"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2603_09237_b200 as mb  # noqa: E402

mbi = int(sys.argv[1]) if len(sys.argv) > 1 else 10
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
    spans.append((a.value, b.value, st.value, name.value.decode()))
spans.sort()
gathers = [s for s in spans if s[3].endswith("/gather")]
lo, hi = gathers[mbi][0], gathers[mbi + 1][0]
print(f"minibatch {mbi}: {lo:.3f} .. {hi:.3f} ms ({(hi - lo) * 1e3:.1f} us)")
for a, b, st, nm in spans:
    if lo <= a < hi:
        print(f"  s{st} {(a - lo) * 1e3:8.1f} {(b - lo) * 1e3:8.1f}  {(b - a) * 1e3:7.1f} us  {nm}")
end = max(s[1] for s in spans)
for st in sorted(set(s[2] for s in spans)):
    busy = sum(b - a for a, b, s, _ in spans if s == st)
    print(f"stream {st}: busy {busy:.3f} of {end:.3f} ms")
