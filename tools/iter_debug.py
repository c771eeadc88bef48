import sys
sys.path.insert(0, "."); sys.path.insert(0, "tests"); sys.path.insert(0, "oracle")
import numpy as np
import paper_2603_09237_b200 as mb
from test_gpu_parity import _tiny, _mbcfg
from pyoracle import Oracle, OracleTrainer
o = Oracle("oracle")
for H in (16, 32, 48):
    c = _tiny(N=32, K=4, T=16, epochs=2, minibatch_count=2, F=16, feat_hidden=[16], actor_hidden=[H, H], critic_hidden=[H, H])
    t = mb.Trainer(_mbcfg(mb, c)); ot = OracleTrainer(o, c)
    st = t.iteration(0); al, cl = ot.iteration(0)
    for which, ref in (("actor", ot.actor_params()), ("critic", ot.critic_params())):
        p = t.params(which); err = np.abs(p - ref)
        lr = c.actor_lr
        big = err > 0.5 * lr
        print(H, which, "n", len(p), "q99/lr", np.quantile(err, 0.99) / lr, "max/lr", err.max() / lr, "frac>0.5lr", big.mean())
        # block split: feature | M | b
        nf = len(p) - 0
        idx = np.nonzero(big)[0]
        print("   first big idx", idx[:10], "last", idx[-5:] if len(idx) else None)
