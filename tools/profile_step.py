"""One warm + N profiled training iterations of a bench config, for ncu:
  ncu --metrics gpu__time_duration.sum --clock-control none -s <warm launches> ... python tools/profile_step.py
Prints the number of kernel launches of the warm-up so -s can skip them."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2603_09237_b200 as mb  # noqa: E402

cfg_name = sys.argv[1] if len(sys.argv) > 1 else "c3"
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 1
t = mb.Trainer(mb.TrainConfig(**bench.BASE[cfg_name]))
t.iteration(0)
print("warm launches (trainer-counted):", t.kernel_launches, flush=True)
import torch  # noqa: E402

torch.cuda.synchronize()
torch.cuda.profiler.start()  # ncu --profile-from-start off captures only this region
for i in range(iters):
    t.iteration(1 + i)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("total launches:", t.kernel_launches)
