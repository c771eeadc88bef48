"""The sharded multi-GPU data plane at W = 2 and 4
ranks on ONE GPU through the in-process loopback communicator: each rank is
a host thread driving its own Trainer; the collectives (all-to-all of the
per-cluster gradient shards, all-gathers of the normalisation partials, the
feature-map gradients, the refreshed M image rows and b entries, the loss
all-reduce) are device copies ordered by events and host barriers.

Partitioning follows the reference's data parallelism over env instances
(parallel.hpp:15-43, rollout.cpp:98) at cluster granularity, with the
minibatch rows of train.cpp:161-184 split by owning rank. Every reduction
keeps the single-rank order, so parameters, rollouts and advantages must
equal the single-GPU trainer's BIT FOR BIT; only the reported minibatch
losses (a sum of per-rank partial sums) may differ in the last bits."""
import threading

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def mb():
    import paper_2603_09237_b200 as mb
    return mb


def _cfg(mb, F, env="mo-pointmass", **kw):
    base = dict(env_name=env, N=64, K=8, T=16, epochs=2, minibatch_count=2, seed=7, F=F, feature_hidden=[16],
                actor_hidden=[32, 32], critic_hidden=[32, 32])
    base.update(kw)
    return mb.TrainConfig(**base)


def _run_ranks(trainers, fn):
    """fn(rank, trainer) on one thread per rank; re-raises the first error."""
    out, errs = [None] * len(trainers), []

    def work(r):
        try:
            out[r] = fn(r, trainers[r])
        except Exception as e:  # noqa: BLE001 -- re-raised below
            errs.append(e)

    th = [threading.Thread(target=work, args=(r,)) for r in range(len(trainers))]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
    assert not any(t.is_alive() for t in th), "a rank hung"
    if errs:
        raise errs[0]
    return out


def _sharded(mb, cfg, W, iters):
    g = mb.LoopbackGroup(W)
    ts = [mb.Trainer(cfg, W, r, loopback=g) for r in range(W)]

    def body(r, t):
        st = [t.iteration(it) for it in range(iters)]
        batch = {k: t.get(k) for k in ("obs", "action_pre", "reward", "advantages", "scalar_advantage",
                                        "terminated", "truncated", "env_ctr")}
        return st, batch, t.params("actor"), t.params("critic")  # params(): collective gather of the M shards

    res = _run_ranks(ts, body)
    del ts
    return res


@pytest.mark.parametrize("F,W", [(64, 2), (64, 4), (16, 2), (32, 4)])
def test_sharded_ranks_match_single_gpu_bit_exact(mb, F, W):
    """F = 64: the fused dM + Adam kernel on each rank's M-row shard (K = all
    clusters); F = 16 / 32: the tcgen05 dM GEMM on the shard + Adam."""
    cfg = _cfg(mb, F)
    iters = 2
    ref = mb.Trainer(cfg)
    ref_st = [ref.iteration(it) for it in range(iters)]
    res = _sharded(mb, cfg, W, iters)
    for name in ("obs", "action_pre", "reward", "advantages", "scalar_advantage", "terminated", "truncated",
                 "env_ctr"):
        whole = ref.get(name)
        got = np.concatenate([r[1][name] for r in res])
        assert np.array_equal(got, whole), name
    for r in range(W):
        _, _, pa, pc = res[r]
        assert np.array_equal(pa, ref.params("actor")), f"rank {r} actor params"
        assert np.array_equal(pc, ref.params("critic")), f"rank {r} critic params"
        for it in range(iters):
            st = res[r][0][it]
            assert st.minibatches == ref_st[it].minibatches
            assert abs(st.actor_loss - ref_st[it].actor_loss) <= 1e-6 * max(1.0, abs(ref_st[it].actor_loss))
            assert abs(st.critic_loss - ref_st[it].critic_loss) <= 1e-6 * max(1.0, abs(ref_st[it].critic_loss))


def test_eight_ranks_with_k_chunked_optimizer(mb):
    """W = 8 ranks, 256 clusters (more than one 128-cluster K chunk of the
    fused dM + Adam: the K-chunked walker on every rank's M-row shard),
    mo-humanoid6 (obs 45, act 12, m 6): bit-exact against one GPU."""
    cfg = _cfg(mb, 64, env="mo-humanoid6", N=512, K=256, T=4, epochs=1, minibatch_count=2, feature_hidden=[32],
               actor_hidden=[64, 64], critic_hidden=[64, 64])
    ref = mb.Trainer(cfg)
    ref.iteration(0)
    res = _sharded(mb, cfg, 8, 1)
    for r in range(8):
        _, _, pa, pc = res[r]
        assert np.array_equal(pa, ref.params("actor")), f"rank {r} actor params"
        assert np.array_equal(pc, ref.params("critic")), f"rank {r} critic params"
    got = np.concatenate([r[1]["scalar_advantage"] for r in res])
    assert np.array_equal(got, ref.get("scalar_advantage"))


def test_single_rank_loopback_is_the_single_gpu_path(mb):
    """W = 1 with a communicator runs every sharded code path (exchanges are
    self-copies) and must equal the no-communicator trainer bit for bit."""
    cfg = _cfg(mb, 64, env="mo-humanoid6", N=64, K=4, T=8, feature_hidden=[64], actor_hidden=[64, 64],
               critic_hidden=[64, 64])
    ref = mb.Trainer(cfg)
    for it in range(2):
        ref.iteration(it)
    (st, _, pa, pc), = _sharded(mb, cfg, 1, 2)
    assert np.array_equal(pa, ref.params("actor")) and np.array_equal(pc, ref.params("critic"))


def test_sharded_checkpoint_gathers_every_shard(mb, tmp_path):
    """save_checkpoint on a sharded rank writes the full parameter vectors
    (every rank's M rows), identical to the single-GPU trainer's file."""
    cfg = _cfg(mb, 64)
    ref = mb.Trainer(cfg)
    ref.iteration(0)
    ref.save_checkpoint(str(tmp_path / "ref.bin"), 1)
    g = mb.LoopbackGroup(2)
    ts = [mb.Trainer(cfg, 2, r, loopback=g) for r in range(2)]

    def body(r, t):
        t.iteration(0)
        t.save_checkpoint(str(tmp_path / f"r{r}.bin"), 1)

    _run_ranks(ts, body)
    want = (tmp_path / "ref.bin").read_bytes()
    assert (tmp_path / "r0.bin").read_bytes() == want and (tmp_path / "r1.bin").read_bytes() == want


def test_loopback_group_errors(mb):
    with pytest.raises(mb.ConfigError):
        mb.LoopbackGroup(0)
    g = mb.LoopbackGroup(2)
    with pytest.raises(mb.ConfigError):
        mb.Trainer(_cfg(mb, 64), 3, 0, loopback=g)
    with pytest.raises(mb.ConfigError):
        mb.Trainer(_cfg(mb, 64, K=6, N=48), 4, 0, loopback=mb.LoopbackGroup(4))  # K % world
