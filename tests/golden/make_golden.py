"""Generates tests/golden/golden_ref.npz from the COMPILED REFERENCE
(oracle/_ref/libmorlax_ref.so = /root/reference/proj/src/*.cpp + shim).

Run here (where /root/reference exists):  python tests/golden/make_golden.py
The GPU box has no /root/reference; tests there read only the .npz.
Every array is the reference's own output on the listed seeded inputs.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "..", "..", "oracle"))
import ctypes as C  # noqa: E402

from pyoracle import ENV_KINDS, Oracle, TrainCfg  # noqa: E402


def main():
    r = Oracle("ref")
    g = {}
    # ---- RNG (rng.hpp): seeds, words, splits, gaussians, shuffle
    seeds = np.array([0, 1, 2, 3, 4, 7, 0x9E3779B9], np.uint64)
    keys = np.array([r.rng_seed_state(int(s))[0] for s in seeds], np.uint64)
    g["rng_seeds"], g["rng_keys"] = seeds, keys
    k0 = int(keys[0])
    g["rng_words_k0"] = r.rng_words(k0, 0, 256)
    g["rng_words_k0_ctr1000"] = r.rng_words(k0, 1000, 64)
    lanes = np.array([0, 1, 2, 0xA1, 0xA2, 0xE0, 0x10000000, 0x2000_0000, 12345], np.uint64)
    g["rng_split_lanes"] = lanes
    g["rng_split_keys_k0"] = np.array([r.split_key(k0, int(l)) for l in lanes], np.uint64)
    g["rng_gauss_k0"] = r.rng_gaussians(k0, 0, 128)
    g["rng_shuffle_k0"], ctr = r.shuffle(k0, 0, np.arange(100))
    g["rng_shuffle_k0_ctr"] = np.array([ctr], np.uint64)
    # ---- env traces (env.cpp + env_*.cpp; humanoid6 via ref_humanoid6.cpp)
    rng = np.random.default_rng(123)
    for name, steps in (("mo-lqr1d", 205), ("mo-pointmass", 205), ("mo-dst-continuous", 60),
                        ("mo-humanoid6", 48)):
        e = r.env(name, 4)
        reset_key = r.split_key(k0, 0xE0)
        obs0 = e.reset(reset_key)
        acts = rng.uniform(-1.25, 1.25, (steps, 4, e.act_dim))
        if name == "mo-dst-continuous":
            acts = np.abs(acts)  # descend so treasures are reached
        if name == "mo-humanoid6":
            acts = np.sign(acts) * np.minimum(1.2, np.abs(acts) * 2)  # drive towards falls
        O, Rw, Te, Tr = [], [], [], []
        for t in range(steps):
            o, rw, te, tr = e.step(acts[t])
            O.append(o); Rw.append(rw); Te.append(te); Tr.append(tr)
        key = name.replace("-", "_")
        g[f"env_{key}_reset_key"] = np.array([reset_key], np.uint64)
        g[f"env_{key}_obs0"] = obs0
        g[f"env_{key}_actions"] = acts
        g[f"env_{key}_obs"] = np.array(O)
        g[f"env_{key}_reward"] = np.array(Rw)
        g[f"env_{key}_term"] = np.array(Te)
        g[f"env_{key}_trunc"] = np.array(Tr)
        g[f"env_{key}_clamps"] = np.array([e.clamp_count()], np.uint64)
    # ---- tiny trainer config used for hypernet / rollout / losses / train
    cfg = TrainCfg(env="mo-pointmass", N=8, K=2, T=12, epochs=2, minibatch_count=2, F=8,
                   feat_hidden=[8], actor_hidden=[8, 8], critic_hidden=[8, 8], seed=5)
    a, c = cfg.specs()
    root = r.rng_seed_state(cfg.seed)[0]
    aflat = r.init_hypernet(a, r.split_key(root, 0xA1))
    cflat = r.init_hypernet(c, r.split_key(root, 0xA2))
    g["hyper_actor_init"], g["hyper_critic_init"] = aflat, cflat
    W = np.array([[0.25, 0.75], [1.0, 0.0], [0.6, 0.4]])
    g["hyper_w"] = W
    g["hyper_actor_theta"] = np.array([r.hypernet_forward(a, aflat, w) for w in W])
    gth = rng.normal(size=(3, a.P))
    g["hyper_gtheta"] = gth
    g["hyper_actor_grad"] = sum(r.hypernet_backward(a, aflat, W[i], gth[i]) for i in range(3))
    cw = np.array([[0.3, 0.7], [0.9, 0.1]])
    env = r.env("mo-pointmass", 8)
    env.reset(r.split_key(root, 0xE0))
    b = r.collect_rollouts(a, aflat, c, cflat, env, cw, 4, 12, r.split_key(root, 77), 0)
    for k, v in b.items():
        g["roll_" + k] = v
    g["roll_cw"] = cw
    adv, tgt = r.gae(b["reward"], b["value"], b["next_value"], b["term"], b["trunc"], 8, 12, 0.99, 0.95)
    g["gae_adv"], g["gae_tgt"] = adv, tgt
    tw = np.repeat(cw, 4, axis=0)
    sadv = r.normalize_scalarize(adv, tw, 8, 12)
    g["gae_sadv"] = sadv
    rows = rng.permutation(96)[:40].astype(np.int32)
    cl = np.repeat(np.arange(2), 4).astype(np.int32)
    g["loss_rows"] = rows
    la, ga = r.actor_loss(a, aflat, 8, 12, b["obs"], b["action_pre"], b["logprob"], tw, cl, rows, sadv,
                          0.2, 0.1)
    lc, gc = r.critic_loss(c, cflat, 8, 12, b["obs"], tw, cl, rows, tgt)
    g["loss_actor"], g["loss_actor_grad"] = np.array([la]), ga
    g["loss_critic"], g["loss_critic_grad"] = np.array([lc]), gc
    p = rng.normal(size=64)
    gr = rng.normal(size=64)
    g["adam_p0"], g["adam_g"] = p, gr
    g["adam_p1"], g["adam_m1"], g["adam_m2"], _ = r.adam(p, gr, np.zeros(64), np.zeros(64), 0, 1e-3)
    ao, co = np.zeros(a.n_params), np.zeros(c.n_params)
    cc = cfg.c()
    r.check(r.lib.mref_train(C.byref(cc), 2, ao.ctypes.data, co.ctypes.data))
    g["train2_actor"], g["train2_critic"] = ao, co
    # ---- Pareto (pareto.cpp)
    pts = np.round(rng.normal(size=(200, 3)), 2)
    pts[17] = pts[3]
    pts[50] = pts[3]
    g["pareto_pts3"] = pts
    g["pareto_mask3"] = r.nondominated_mask(pts)
    for m in (2, 3, 4):
        q = rng.uniform(0.2, 1.0, (25, m))
        g[f"hv_pts{m}"] = q
        g[f"hv_exact{m}"] = np.array(r.hypervolume_detailed(q, np.zeros(m))[:2])
    q6 = rng.uniform(0.2, 1.0, (30, 6))
    g["hv_pts6"] = q6
    v, se, ex, clp = r.hypervolume_detailed(q6, np.zeros(6), samples=200_000)
    g["hv_mc6"] = np.array([v, se])
    # ---- linear_dominance_filter (pareto.cpp:79-139): 2-D hull with a
    # collinear triple, m = 3 / 4 / 6 grid sweeps with a duplicate point
    lrng = np.random.default_rng(77)
    for m, n in ((2, 40), (3, 60), (4, 40), (6, 16)):
        w = lrng.dirichlet(np.ones(m), size=n)
        q = w / np.linalg.norm(w, axis=1, keepdims=True) + lrng.normal(0, 0.05, (n, m))
        q[5] = q[2]
        if m == 2:
            q[7] = [0.0, 1.0]
            q[8] = [0.5, 0.5 + 0.5]
            q[9] = [1.0, 0.0]
            q[10] = [0.25, 0.75 + 0.25 * 0.5]
        g[f"ldf_pts{m}"] = q
        g[f"ldf_mask{m}"] = r.linear_dominance_mask(q)
    # ---- evaluate_params (evaluate.cpp:17-101): reference envs only
    from pyoracle import HSpec
    for env, od, ad, res, eps in (("mo-pointmass", 4, 2, 4, 3), ("mo-lqr1d", 1, 1, 3, 2)):
        spec = HSpec(2, 16, [16], [od, 32, 32, ad], True, True)
        flat = r.init_hypernet(spec, 0x77)
        W, R = r.evaluate_params(spec, flat, ENV_KINDS[env], res, eps, 0x1234)
        g[f"eval_{env}_flat"], g[f"eval_{env}_W"], g[f"eval_{env}_R"] = flat, W, R
    np.savez_compressed(os.path.join(HERE, "golden_ref.npz"), **g)
    print("wrote", len(g), "arrays")


if __name__ == "__main__":
    main()
