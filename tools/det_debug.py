"""Two identical trainers, one iteration: where do the parameters differ?"""
import sys
sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import numpy as np
import paper_2603_09237_b200 as mb
from test_gpu_parity import _tiny, _mbcfg

c = _tiny(N=32, K=4, T=16)
t1, t2 = mb.Trainer(_mbcfg(mb, c)), mb.Trainer(_mbcfg(mb, c))
print("n_actor", t1.n_actor, "n_critic", t1.n_critic)
for it in range(2):
    s1, s2 = t1.iteration(it), t2.iteration(it)
    print(it, s1.actor_loss, s2.actor_loss, s1.critic_loss, s2.critic_loss)
    for w in ("actor", "critic"):
        a, b = t1.params(w), t2.params(w)
        d = np.nonzero(a != b)[0]
        print(w, "ndiff", len(d), d[:10], d[-10:] if len(d) else "")
