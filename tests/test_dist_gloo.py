"""World-size-2 and 4 (gloo, CPU processes) restatement of the sharded data
plane the CUDA trainer runs per rank (trainer.cu: Trainer::phase_advantages,
HyperNet::backward_multi / adam_step), in fp64 numpy with the
product's own host partitioning (mb.shard_rows, mb.shard_minibatch):

  * rank r owns instances [r N/W, (r+1) N/W) = whole preference clusters
    (the reference's data parallelism over instances, parallel.hpp:15-43);
  * normalisation statistics (gae.cpp:79-96): one partial per cluster,
    all-gathered, summed in cluster order;
  * a minibatch is the global perm slice (train.cpp:161-169); each rank
    keeps its own rows (shard_minibatch) and scales by the GLOBAL 1/B, so the
    per-cluster theta gradients are complete on the owning rank;
  * hypernet backward + Adam (hypernet.cpp:92-122, adam.cpp:8-26,
    train.cpp:28-39): the per-cluster theta gradients are exchanged
    all-to-all by column shard (shard_rows), db / dM / Adam run on the
    rank's M rows and b entries only, the updated rows are all-gathered; the
    per-cluster feature-map output gradients are all-gathered and the feature
    map's backward + Adam run replicated.

Every cross-rank reduction keeps the single-process order, so the result must
equal the single-process computation EXACTLY (==), which is what the CUDA
trainer's loopback tests check on the GPU (tests/test_gpu_multirank.py)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


# ------------------------------------------------------------------ fixed-order fp64 pieces
def seq_sum(rows):
    """sum of the rows of a 2-D array in row order (the device's order)."""
    acc = np.zeros(rows.shape[1:])
    for r in rows:
        acc = acc + r
    return acc


def feature_forward(fp, w):  # tanh MLP m -> h -> F, tanh output (hypernet.cpp:10-17)
    W1, b1, W2, b2 = fp
    h = np.tanh(w @ W1.T + b1)
    return h, np.tanh(h @ W2.T + b2)


def feature_backward(fp, w, h, f, df):
    """weight gradients of the feature map from df_g = M^T gtheta_g, summed
    over the clusters in cluster order."""
    W1, b1, W2, b2 = fp
    gz2 = df * (1.0 - f * f)
    gz1 = (gz2 @ W2) * (1.0 - h * h)
    dW2 = seq_sum(np.einsum("gi,gj->gij", gz2, h))
    dW1 = seq_sum(np.einsum("gi,gj->gij", gz1, w))
    return [dW1, seq_sum(gz1), dW2, seq_sum(gz2)]


def adam(p, g, m1, m2, step, lr):  # adam.cpp:8-26
    m1 = 0.9 * m1 + 0.1 * g
    m2 = 0.999 * m2 + 0.001 * g * g
    p = p - lr * (m1 / (1 - 0.9 ** step)) / (np.sqrt(m2 / (1 - 0.999 ** step)) + 1e-8)
    return p, m1, m2


def problem(K=8, reps=4, T=6, m=2, h=8, F=8, P=300, seed=3):
    rng = np.random.default_rng(seed)
    cw = rng.dirichlet(np.ones(m), size=K)
    fp = [rng.normal(size=(h, m)) * 0.5, rng.normal(size=h) * 0.1, rng.normal(size=(F, h)) * 0.3,
          rng.normal(size=F) * 0.1]
    M = rng.normal(size=(P, F)) * 0.01
    b = rng.normal(size=P) * 0.01
    adv = rng.normal(size=(K * reps * T, m))
    gth = rng.normal(size=(K, P))  # each cluster's theta gradient (complete on its owner)
    return dict(K=K, reps=reps, T=T, m=m, F=F, P=P, cw=cw, fp=fp, M=M, b=b, adv=adv, gth=gth)


def single_process(pb, lr=1e-3):
    K, reps, T = pb["K"], pb["reps"], pb["T"]
    rows = reps * T
    part = np.stack([seq_sum(pb["adv"][g * rows:(g + 1) * rows]) for g in range(K)])
    mean = seq_sum(part) / (K * rows)
    part2 = np.stack([seq_sum((pb["adv"][g * rows:(g + 1) * rows] - mean) ** 2) for g in range(K)])
    inv = 1.0 / (np.sqrt(seq_sum(part2) / (K * rows)) + 1e-8)
    hh, f = feature_forward(pb["fp"], pb["cw"])
    db = seq_sum(pb["gth"])
    dM = seq_sum(np.einsum("gp,gf->gpf", pb["gth"], f))
    df = pb["gth"] @ pb["M"]
    fg = feature_backward(pb["fp"], pb["cw"], hh, f, df)
    M, _, _ = adam(pb["M"], dM, 0, 0, 1, lr)
    b, _, _ = adam(pb["b"], db, 0, 0, 1, lr)
    fp = [adam(x, gx, 0, 0, 1, lr)[0] for x, gx in zip(pb["fp"], fg)]
    return mean, inv, M, b, fp


def _worker(rank, world, port, q):
    import sys
    here = os.path.dirname(os.path.abspath(__file__))
    sys.path.insert(0, os.path.dirname(here))
    sys.path.insert(0, os.path.join(os.path.dirname(here), "oracle"))
    import paper_2603_09237_b200 as mb
    from pyoracle import Oracle, OracleTrainer, TrainCfg

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        out = {}
        # ---------------- the sharded data plane (exact)
        pb = problem()
        K, reps, T, P, F, lr = pb["K"], pb["reps"], pb["T"], pb["P"], pb["F"], 1e-3
        Kl = K // world
        g0 = rank * Kl
        rows = reps * T
        # normalisation partials of this rank's clusters, all-gathered, summed in cluster order
        loc = pb["adv"][g0 * rows:(g0 + Kl) * rows]
        part = torch.tensor(np.stack([seq_sum(loc[k * rows:(k + 1) * rows]) for k in range(Kl)]))
        parts = [torch.zeros_like(part) for _ in range(world)]
        dist.all_gather(parts, part)
        mean = seq_sum(torch.cat(parts).numpy()) / (K * rows)
        part2 = torch.tensor(np.stack([seq_sum((loc[k * rows:(k + 1) * rows] - mean) ** 2) for k in range(Kl)]))
        dist.all_gather(parts, part2)
        inv = 1.0 / (np.sqrt(seq_sum(torch.cat(parts).numpy()) / (K * rows)) + 1e-8)
        # theta-gradient shards: all-to-all by column shard (pack_shards -> grecv [G][S])
        S, lo, hi = mb.shard_rows(P, world, rank)
        assert S % 128 == 0 and all(mb.shard_rows(P, world, r)[0] == S for r in range(world))
        gl = np.zeros((Kl, world * S))
        gl[:, :P] = pb["gth"][g0:g0 + Kl]
        send = torch.tensor(np.ascontiguousarray(gl.reshape(Kl, world, S).transpose(1, 0, 2)))  # [W][Kl][S]
        recv = torch.zeros_like(send)
        dist.all_to_all_single(recv, send)
        grecv = recv.numpy().reshape(K, S)[:, :hi - lo]  # every cluster, this rank's rows
        hh, f = feature_forward(pb["fp"], pb["cw"])  # every rank: f(w) of every cluster
        db = seq_sum(grecv)
        dM = seq_sum(np.einsum("gp,gf->gpf", grecv, f))
        Ms, _, _ = adam(pb["M"][lo:hi], dM, 0, 0, 1, lr)
        bs, _, _ = adam(pb["b"][lo:hi], db, 0, 0, 1, lr)
        # all-gather the updated rows (each rank's block padded to S)
        Mp = torch.zeros(S, F, dtype=torch.float64)
        Mp[:hi - lo] = torch.tensor(Ms)
        bp = torch.zeros(S, dtype=torch.float64)
        bp[:hi - lo] = torch.tensor(bs)
        mg = [torch.zeros_like(Mp) for _ in range(world)]
        bg = [torch.zeros_like(bp) for _ in range(world)]
        dist.all_gather(mg, Mp)
        dist.all_gather(bg, bp)
        M = torch.cat(mg).numpy()[:P]
        b = torch.cat(bg).numpy()[:P]
        # df of this rank's clusters (owner: full M), all-gathered; replicated feature backward
        df_loc = torch.tensor(pb["gth"][g0:g0 + Kl] @ pb["M"])
        dfs = [torch.zeros_like(df_loc) for _ in range(world)]
        dist.all_gather(dfs, df_loc)
        fg = feature_backward(pb["fp"], pb["cw"], hh, f, torch.cat(dfs).numpy())
        fp = [adam(x, gx, 0, 0, 1, lr)[0] for x, gx in zip(pb["fp"], fg)]
        ref = single_process(pb, lr)
        out["exact"] = bool(np.array_equal(mean, ref[0]) and np.array_equal(inv, ref[1]) and
                            np.array_equal(M, ref[2]) and np.array_equal(b, ref[3]) and
                            all(np.array_equal(x, y) for x, y in zip(fp, ref[4])))
        # ---------------- one minibatch of the oracle losses: local rows, global 1/B
        o = Oracle("oracle")
        c = TrainCfg(env="mo-pointmass", N=16, K=4, T=8, F=8, feat_hidden=[8], actor_hidden=[8, 8],
                     critic_hidden=[8, 8], seed=11)
        t = OracleTrainer(o, c)
        t.iteration(0, max_minibatches=0)  # rollout + GAE of iteration 0 (identical on every rank)
        bt = t.batch()
        N, T2, K2 = c.N, c.T, c.K
        reps2 = N // K2
        n_inst = N // world
        lo_i = rank * n_inst
        tw = np.repeat(t.clusters(), reps2, axis=0)
        a_s, c_s = c.specs()
        perm = np.random.default_rng(5).permutation(N * T2).astype(np.int32)
        lo_m, hi_m = 13, 13 + 48
        rws, goff, _ = mb.shard_minibatch(perm, lo_m, hi_m, T2, lo_i, n_inst, reps2, K2 // world)
        grow = (rws + lo_i * T2).astype(np.int32)
        cluster = (np.arange(N) // reps2).astype(np.int32)
        scale = len(grow) / (hi_m - lo_m)
        la, ga = o.actor_loss(a_s, t.actor_params(), N, T2, bt["obs"], bt["action_pre"], bt["logprob"], tw, cluster,
                              grow, bt["sadv"], c.clip_eps, c.entropy_coef)
        lc, gc = o.critic_loss(c_s, t.critic_params(), N, T2, bt["obs"], tw, cluster, grow, bt["targets"])
        vec = torch.tensor(np.concatenate([[la * scale, lc * scale], ga * scale, gc * scale]), dtype=torch.float64)
        dist.all_reduce(vec)
        la_f, ga_f = o.actor_loss(a_s, t.actor_params(), N, T2, bt["obs"], bt["action_pre"], bt["logprob"], tw,
                                  cluster, perm[lo_m:hi_m], bt["sadv"], c.clip_eps, c.entropy_coef)
        lc_f, gc_f = o.critic_loss(c_s, t.critic_params(), N, T2, bt["obs"], tw, cluster, perm[lo_m:hi_m],
                                   bt["targets"])
        full = np.concatenate([[la_f, lc_f], ga_f, gc_f])
        out["loss_err"] = float(np.abs(vec.numpy() - full).max() / np.abs(full).max())
        q.put((rank, out))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_sharded_decomposition_matches_single_process(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=180) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, out in res:
        assert out["exact"], f"rank {rank}: sharded result differs from the single-process one"
        assert out["loss_err"] < 1e-12, out["loss_err"]
