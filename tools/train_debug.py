import sys
sys.path.insert(0, "."); sys.path.insert(0, "tests"); sys.path.insert(0, "oracle")
import paper_2603_09237_b200 as mb
from test_gpu_parity import _tiny, _mbcfg
c = _tiny(N=16, K=2, T=12, epochs=2, minibatch_count=2, F=16, feat_hidden=[16], actor_hidden=[16, 16], critic_hidden=[16, 16])
u = mb.Trainer(_mbcfg(mb, c))
for it in range(3):
    try:
        s = u.iteration(it); print("iter", it, s.actor_loss, s.critic_loss)
    except Exception as e:
        print("iter", it, "ERR", e)
for li in (100, 2):
    try:
        t = mb.train(_mbcfg(mb, c), mb.RunOptions(iterations=3, log_interval=li, grid_resolution=3, episodes_per_point=2), callback=lambda r: print(" cb", r.iteration, r.actor_loss, r.archive_hypervolume))
        print("train ok", li)
    except Exception as e:
        print("train", li, "ERR", e)
