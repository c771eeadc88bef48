"""Config-2 forward a few times (for ncu launch lists)."""
import sys
sys.path.insert(0, ".")
import torch
import bench
import paper_2603_09237_b200 as mb
print(bench.leg_c2(mb, 1500.0)["value"])
torch.cuda.synchronize()
