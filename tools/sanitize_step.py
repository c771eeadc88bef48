"""Small workload for compute-sanitizer (memcheck / racecheck / synccheck):
one training iteration at a small config (k_rollout_tc, k_img_gemm with
every epilogue, k_head, k_dm_adam, the GAE / stats / gather / Adam kernels),
the fused dM + Adam test hook at G = 200 (two K chunks), a 5-objective exact
hypervolume (k_hv_top / k_hv_level1 / k_hv_sub / k_hv_reduce), the dominance
mask and the MC hypervolume."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_09237_b200 as mb  # noqa: E402

cfg = mb.TrainConfig(env_name="mo-humanoid6", N=128, K=2, T=4, epochs=1, minibatch_count=2, seed=3, F=64,
                     feature_hidden=[64], actor_hidden=[128, 128], critic_hidden=[128, 128], entropy_coef=0.01)
t = mb.Trainer(cfg)
st = t.iteration(0)
print("iteration ok", st.actor_loss, st.critic_loss, flush=True)
G, P, F = 200, 300, 32
rng = np.random.default_rng(0)
arrs = [rng.normal(size=s).astype(np.float32) for s in ((G, P), (G, F), (P, F), (P, F))]
m2 = np.abs(rng.normal(size=(P, F))).astype(np.float32)
img = np.zeros((P, F), np.uint16)
rc = mb.LIB.morlax_dm_adam_test(G, P, F, arrs[0].ctypes.data, arrs[1].ctypes.data, arrs[2].ctypes.data,
                                arrs[3].ctypes.data, m2.ctypes.data, 1e-3, 1.0, 1.0, img.ctypes.data)
assert rc == 0
print("dm_adam ok", flush=True)
w = rng.dirichlet(np.ones(5), size=120)
pts = w / np.linalg.norm(w, axis=1, keepdims=True) + rng.normal(0, 0.02, w.shape)
mask = mb.nondominated_mask(pts)
print("hv exact", mb.hypervolume_exact(pts[mask.astype(bool)], -np.ones(5)), flush=True)
print("hv mc", mb.hypervolume_detailed(pts[mask.astype(bool)], -np.ones(5), samples=20000)[:2], flush=True)
