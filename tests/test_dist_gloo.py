"""World-size-2 (gloo, CPU) check of the multi-GPU decomposition the CUDA
trainer uses (trainer.cu: Trainer::phase_advantages / minibatch):

  * each rank owns instances [r*N/W, (r+1)*N/W) = whole preference clusters;
  * advantage-normalisation statistics are per-rank sums, all-reduced;
  * a minibatch is the global perm slice, each rank keeps its own rows
    (shard_minibatch, the C-ABI host helper) and scales by the GLOBAL 1/B;
  * the hypernetwork gradient is linear in the per-cluster theta gradients,
    so each rank's hypernet backward over its own clusters, summed across
    ranks, equals the single-process gradient (checked on the losses);
  * the exchange the trainer actually performs (HyperNet::backward_multi):
    the per-cluster theta-gradient rows are all-gathered so every rank forms
    dM (and db) over all clusters itself, and only the feature-map gradient
    (and db) is all-reduced -- the result equals the single-process
    hypernet_backward; Adam then runs replicated on identical gradients.

Each rank computes with the fp64 C oracle; results are compared with the
single-process oracle on the same seeded inputs."""
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
        o = Oracle("oracle")
        c = TrainCfg(env="mo-pointmass", N=16, K=4, T=8, F=8, feat_hidden=[8], actor_hidden=[8, 8],
                     critic_hidden=[8, 8], seed=11)
        t = OracleTrainer(o, c)
        t.iteration(0, max_minibatches=0)  # rollout + GAE of iteration 0 (identical on every rank)
        b = t.batch()
        N, T, K, m = c.N, c.T, c.K, 2
        reps = N // K
        n_inst = N // world
        lo_i = rank * n_inst
        rows_local = slice(lo_i * T, (lo_i + n_inst) * T)
        cw = t.clusters()
        tw = np.repeat(cw, reps, axis=0)
        # --- normalisation statistics: local sums, all-reduced (gae.cpp:79-96)
        adv = b["adv"][rows_local]
        s1 = torch.tensor(adv.sum(0), dtype=torch.float64)
        cnt = torch.tensor([float(adv.shape[0])], dtype=torch.float64)
        dist.all_reduce(s1)
        dist.all_reduce(cnt)
        mean = (s1 / cnt).numpy()
        s2 = torch.tensor(((adv - mean) ** 2).sum(0), dtype=torch.float64)
        dist.all_reduce(s2)
        inv = 1.0 / (np.sqrt(s2.numpy() / cnt.numpy()) + 1e-8)
        sadv_local = ((adv - mean) * inv * tw[lo_i:lo_i + n_inst].repeat(T, axis=0)).sum(1)
        err_norm = np.abs(sadv_local - b["sadv"][rows_local]).max()
        # --- one minibatch: local rows, global 1/B, summed gradients
        a_s, c_s = c.specs()
        perm = np.random.default_rng(5).permutation(N * T).astype(np.int32)
        lo, hi = 13, 13 + 48
        rows, goff, _ = mb.shard_minibatch(perm, lo, hi, T, lo_i, n_inst, reps, K // world)
        grow = (rows + lo_i * T).astype(np.int32)
        cluster = (np.arange(N) // reps).astype(np.int32)
        scale = len(grow) / (hi - lo)
        la, ga = o.actor_loss(a_s, t.actor_params(), N, T, b["obs"], b["action_pre"], b["logprob"], tw, cluster,
                              grow, b["sadv"], c.clip_eps, c.entropy_coef)
        lc, gc = o.critic_loss(c_s, t.critic_params(), N, T, b["obs"], tw, cluster, grow, b["targets"])
        vec = torch.tensor(np.concatenate([[la * scale, lc * scale], ga * scale, gc * scale]), dtype=torch.float64)
        dist.all_reduce(vec)
        if rank == 0:
            la_f, ga_f = o.actor_loss(a_s, t.actor_params(), N, T, b["obs"], b["action_pre"], b["logprob"], tw,
                                      cluster, perm[lo:hi], b["sadv"], c.clip_eps, c.entropy_coef)
            lc_f, gc_f = o.critic_loss(c_s, t.critic_params(), N, T, b["obs"], tw, cluster, perm[lo:hi],
                                       b["targets"])
            full = np.concatenate([[la_f, lc_f], ga_f, gc_f])
            v = vec.numpy()
            err_grad = float(np.abs(v - full).max() / np.abs(full).max())
        else:
            err_grad = 0.0
        # --- the exchange of HyperNet::backward_multi on seeded per-cluster theta gradients
        Kl = K // world
        gth = np.random.default_rng(100).normal(size=(K, a_s.P))  # every cluster's dloss / dtheta
        mine = torch.tensor(gth[rank * Kl:(rank + 1) * Kl])
        parts = [torch.zeros_like(mine) for _ in range(world)]
        dist.all_gather(parts, mine)  # the bf16-row all-gather (fp64 here)
        rows_all = torch.cat(parts).numpy()
        flat = t.actor_params()

        def hb(ws, gs):  # hypernet_backward is per preference (hypernet.cpp:92-122): sum over clusters
            return sum(o.hypernet_backward(a_s, flat, wv, gv) for wv, gv in zip(ws, gs))
        g_all = hb(cw, rows_all)  # dM / db over every cluster, on every rank
        g_loc = hb(cw[rank * Kl:(rank + 1) * Kl], gth[rank * Kl:(rank + 1) * Kl])
        nfe = a_s.n_feature
        feat = torch.tensor(g_loc[:nfe])
        dist.all_reduce(feat)  # the feature-map gradient: per-rank partials
        db_loc = torch.tensor(gth[rank * Kl:(rank + 1) * Kl].sum(0))
        dist.all_reduce(db_loc)  # db: per-rank partial sums
        got = np.concatenate([feat.numpy(), g_all[nfe:nfe + a_s.P * a_s.F], db_loc.numpy()])
        ref = hb(cw, gth)
        err_x = float(np.abs(got - ref).max() / np.abs(ref).max())
        q.put((float(err_norm), max(err_grad, err_x)))
    finally:
        dist.destroy_process_group()


def test_two_rank_decomposition_matches_single_process():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for err_norm, err_grad in res:
        assert err_norm < 1e-12, err_norm
        assert err_grad < 1e-12, err_grad
