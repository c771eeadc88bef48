"""GPU parity at the configuration the bench measures (config 3: mo-humanoid6,
obs 45 / act 12 / m 6, policy 45-256-256-12, critic 45-256-256-6, hypernet
6-256-F256, 64 environments per preference cluster), shrinking only the
cluster count K and the horizon T so the oracle finishes in seconds, plus
episode boundaries inside the fused rollout.

* Rollout, teacher-forced (rollout.cpp:98-151, env.cpp:60-92): every step
  the oracle restarts from the DEVICE's recorded observation and uses the
  device's generated weights (bf16 weights as the tensor cores see them,
  fp32 biases / log-std), so per-step errors do not compound: actions,
  log-probs, values and next values within the bf16 tolerance per step;
  terminated / truncated flags, auto-reset observations, stream counters and
  step counters bit-exact; completed-episode returns exact.
* Losses and hypernet gradients at bench widths on the device's own rollout
  batch (losses.cpp:46-189): the head kernel at act_dim 12, the 256-wide
  backward epilogues and grouped weight gradients.
* The fused dM + Adam kernel at the bench shape (G = 128, P = 80,664,
  F = 256) and at multi-rank cluster counts (K chunks) against numpy fp64.
* A full training iteration at bench widths against the oracle, compared in
  update space (tests/helpers.py: update_errors).
"""
import ctypes as C

import numpy as np
import pytest

from helpers import REL_BF16, REL_F32, assert_close, assert_normwise, assert_update_close, bf16, hyper_blocks
from pyoracle import ENV_KINDS, ENV_SPECS, Oracle, OracleEnv, OracleTrainer, TrainCfg

pytestmark = pytest.mark.gpu

LOG_SQRT_2PI = 0.9189385332046727


@pytest.fixture(scope="module")
def mb():
    import paper_2603_09237_b200 as mb
    return mb


@pytest.fixture(scope="module")
def o():
    return Oracle("oracle")


def _mbcfg(mb, c: TrainCfg):
    return mb.TrainConfig(env_name=c.env, N=c.N, K=c.K, kappa=c.kappa, T=c.T, epochs=c.epochs,
                          minibatch_count=c.minibatch_count, gamma=c.gamma, gae_lambda=c.lam,
                          clip_eps=c.clip_eps, actor_lr=c.actor_lr, critic_lr=c.critic_lr,
                          entropy_coef=c.entropy_coef, seed=c.seed, F=c.F,
                          feature_hidden=c.feat_hidden, actor_hidden=c.actor_hidden,
                          critic_hidden=c.critic_hidden)


def bench_cfg(K=4, T=8, **kw):
    """Config-3 widths (bench.py BASE["c3"]) with 64 envs per cluster."""
    base = dict(env="mo-humanoid6", N=64 * K, K=K, T=T, epochs=2, minibatch_count=2, clip_eps=0.2,
                actor_lr=3e-4, critic_lr=1e-3, entropy_coef=0.01, seed=2, F=256, feat_hidden=[256],
                actor_hidden=[256, 256], critic_hidden=[256, 256])
    base.update(kw)
    return TrainCfg(**base)


# ------------------------------------------------------------------ fused dM + Adam (dm_adam.cu)
@pytest.mark.parametrize("G,P,F", [(128, 80664, 256), (128, 79110, 256), (5, 1000, 64), (1024, 4133, 64),
                                   (200, 300, 32)])
def test_dm_adam_matches_numpy(mb, G, P, F):
    """dM = gtheta^T f on the bf16 images (hypernet.cpp:92-122) consumed by
    Adam (adam.cpp:8-26) in one kernel. G = 128 / F = 256 / P = 80,664 is the
    bench's launch; G = 1024 is the 8-rank cluster count (8 K chunks)."""
    rng = np.random.default_rng(G + P)
    gth = (rng.normal(size=(G, P)) * 1e-3).astype(np.float32)
    f = np.tanh(rng.normal(size=(G, F))).astype(np.float32)
    p = (rng.normal(size=(P, F)) * 0.01).astype(np.float32)
    m1 = (rng.normal(size=(P, F)) * 1e-3).astype(np.float32)
    m2 = (rng.random(size=(P, F)) * 1e-5).astype(np.float32)
    lr, step = 3e-4, 7
    ibc1, ibc2 = np.float32(1 / (1 - 0.9 ** step)), np.float32(1 / (1 - 0.999 ** step))
    pd, ad, bd = p.copy(), m1.copy(), m2.copy()
    img = np.zeros((P, F), np.uint16)
    rc = mb.LIB.morlax_dm_adam_test(G, P, F, gth.ctypes.data, f.ctypes.data, pd.ctypes.data, ad.ctypes.data,
                                    bd.ctypes.data, lr, ibc1, ibc2, img.ctypes.data)
    assert rc == 0, mb.LIB.morlax_last_error()
    g = bf16(gth).T @ bf16(f)  # fp64 product of the bf16 operands
    a_ref = 0.9 * m1.astype(np.float64) + 0.1 * g
    b_ref = 0.999 * m2.astype(np.float64) + 0.001 * g * g
    d_ref = -lr * float(ibc1) * a_ref / (np.sqrt(b_ref * float(ibc2)) + 1e-8)
    # fp32 accumulation of exact bf16 products: |dM_dev - dM| <= G eps sum_k |gtheta_k f_k|
    S = np.abs(bf16(gth)).T @ np.abs(bf16(f))
    eg = G * 2.0 ** -24 * S
    assert np.all(np.abs(ad - a_ref) <= 0.1 * eg + 2e-7 * np.abs(a_ref) + 1e-12), "m1"
    assert np.all(np.abs(bd - b_ref) <= 0.002 * np.abs(g) * eg + 2e-7 * b_ref + 1e-15), "m2"
    # the update itself (not p, which hides it), propagated from those bounds
    # plus the fp32 Adam arithmetic (hardware sqrt / divide: a few ulp)
    den = np.sqrt(b_ref * float(ibc2)) + 1e-8
    du = lr * float(ibc1) * (0.1 * eg / den + np.abs(a_ref) * 0.5 * (0.002 * np.abs(g) * eg) * float(ibc2) / den ** 3)
    upd = pd.astype(np.float64) - p
    assert np.all(np.abs(upd - d_ref) <= du + 1e-5 * np.abs(d_ref) + 2e-9), "p update"
    # the refreshed M image holds bf16(p_new) exactly
    exp = np.ascontiguousarray(pd).view(np.uint32).astype(np.uint64)
    exp = (((exp + 0x7FFF + ((exp >> 16) & 1)) >> 16) & 0xFFFF).astype(np.uint16)
    assert np.array_equal(img, exp)


# ------------------------------------------------------------------ teacher-forced rollout
def _mlp(theta, sizes, x):
    """nn.cpp:60-92 on the device's operands: every tensor-core operand in
    bf16 as the device holds it (observation, weights, hidden activations:
    north star "bf16 in, fp32 accumulate"), fp32 biases, fp64 arithmetic;
    returns the output layer's pre-activation. What remains between the two
    is accumulation order and the device's tanh."""
    off = 0
    a = bf16(x)
    L = len(sizes) - 1
    th = np.asarray(theta, np.float32)
    for layer in range(L):
        i, o_ = sizes[layer], sizes[layer + 1]
        W = bf16(th[off:off + i * o_]).reshape(o_, i)
        b = th[off + i * o_:off + i * o_ + o_].astype(np.float64)
        off += (i + 1) * o_
        a = a @ W.T + b
        if layer < L - 1:
            a = bf16(np.tanh(a))
    return a


def _per_cluster(fn, theta, sizes, x, reps):
    return np.concatenate([fn(theta[c], sizes, x[c * reps:(c + 1) * reps]) for c in range(len(theta))])


def _rollout_keys(o, seed, it, N):
    root = o.rng_seed_state(seed)[0]
    lane = o.split_key(o.split_key(root, 0x10000000 + it), 1)  # train.cpp:120,146
    return [o.split_key(lane, i) for i in range(N)]  # rollout.cpp:101


def _normwise_step(a, b, rel, what):
    scale = max(float(np.abs(b).max()), 1e-30)
    e = float(np.abs(np.asarray(a, np.float64) - b).max()) / scale
    assert e <= rel, f"{what}: normwise rel err {e:.3g} > {rel}"
    return e


def _teacher_forced(mb, o, c: TrainCfg, prepare=None, it=0):
    t = mb.Trainer(_mbcfg(mb, c))
    es = t.es
    N, T, K = c.N, c.T, c.K
    reps = N // K
    od, ad, m = es.obs_dim, es.act_dim, es.m
    if prepare:
        prepare(t)
    steps0 = t.get("env_steps").copy()
    ctr0 = t.get("env_ctr").copy()
    keys = t.get("env_key").copy()
    trk0 = t.get("tracker").copy()
    t.phase(it, 1)  # sampling + hypernet + fused rollout (train.cpp:130-150)
    a_s, c_s = c.specs()
    th_a, th_c = t.theta("actor"), t.theta("critic")
    cw = t.get("clusters")
    obs = t.get("obs").reshape(N, T, od).astype(np.float64)
    z = t.get("action_pre").reshape(N, T, ad).astype(np.float64)
    lp = t.get("logprob").reshape(N, T)
    rew = t.get("reward").reshape(N, T, m)
    val = t.get("value").reshape(N, T, m)
    nval = t.get("next_value").reshape(N, T, m)
    term = t.get("terminated").reshape(N, T)
    trunc = t.get("truncated").reshape(N, T)
    rk = _rollout_keys(o, c.seed, it, N)
    eps = np.stack([o.rng_gaussians(k, 0, T * ad) for k in rk]).reshape(N, T, ad)
    ls = np.clip(th_a[:, a_s.mlp_n:a_s.mlp_n + ad].astype(np.float64), -5.0, 1.0)  # nn.cpp:185-188
    ls_i = np.repeat(ls, reps, axis=0)
    env = OracleEnv(o, ENV_KINDS[c.env], N)
    steps, ctrs = steps0.astype(np.int32), ctr0.astype(np.uint64)
    errs = {"action_pre": 0.0, "mean": 0.0, "logprob": 0.0, "value": 0.0, "next_value": 0.0}
    n_term = n_trunc = 0
    for s in range(T):
        x = obs[:, s]
        mu = _per_cluster(_mlp, th_a, a_s.target_sizes, x, reps)
        z_o = mu + np.exp(ls_i) * eps[:, s]  # nn.cpp:192-202
        errs["action_pre"] = max(errs["action_pre"], _normwise_step(z[:, s], z_o, REL_BF16, f"action_pre t={s}"))
        mu_dev = z[:, s] - np.exp(ls_i) * eps[:, s]  # the policy mean alone (fp32 sampling arithmetic)
        errs["mean"] = max(errs["mean"], _normwise_step(mu_dev, mu, REL_BF16, f"policy mean t={s}"))
        zs = z[:, s]  # teacher forcing: the device's sample drives the oracle from here on
        lp_o = np.sum(-0.5 * ((zs - mu) / np.exp(ls_i)) ** 2 - ls_i - LOG_SQRT_2PI
                      - np.log(1.0 - np.tanh(zs) ** 2 + 1e-6), axis=1)  # nn.cpp:204-219
        errs["logprob"] = max(errs["logprob"], _normwise_step(lp[:, s], lp_o, REL_BF16, f"logprob t={s}"))
        v_o = _per_cluster(_mlp, th_c, c_s.target_sizes, x, reps)
        errs["value"] = max(errs["value"], _normwise_step(val[:, s], v_o, REL_BF16, f"value t={s}"))
        env.set_instances(state=x, steps=steps, keys=keys, ctrs=ctrs)
        fobs, r_o, te_o, tr_o = env.step(np.tanh(zs))  # env.cpp:60-92
        _, ctrs, steps = env.streams()
        assert np.array_equal(term[:, s], te_o), f"terminated t={s}"
        assert np.array_equal(trunc[:, s], tr_o), f"truncated t={s}"
        n_term += int(te_o.sum())
        n_trunc += int(tr_o.sum())
        assert_close(rew[:, s], r_o, REL_F32, floor=1e-2, what=f"reward t={s}")
        nv_o = _per_cluster(_mlp, th_c, c_s.target_sizes, fobs, reps)  # V at the pre-reset final obs
        errs["next_value"] = max(errs["next_value"], _normwise_step(nval[:, s], nv_o, REL_BF16, f"next_value t={s}"))
        cur = env.current_obs()
        done = (te_o | tr_o).astype(bool)
        nxt = obs[:, s + 1] if s + 1 < T else t.get("env_state").T.astype(np.float64)
        # auto-reset observations come from the persistent stream: bit-exact
        assert np.array_equal(nxt[done], cur[done].astype(np.float32).astype(np.float64)), f"reset obs t={s}"
        assert_close(nxt[~done], cur[~done], REL_F32, floor=1e-2, what=f"next obs t={s}")
    assert np.array_equal(t.get("env_ctr"), ctrs), "stream counters"
    assert np.array_equal(t.get("env_steps"), steps), "step counters"
    # episode tracker and completed-return merge (rollout.cpp:143-159), fp32
    # running sums in step order, fp64 scalarised return per completed episode
    run = trk0.astype(np.float32)
    rs = np.zeros(N)
    rc = np.zeros(N, np.int32)
    w = np.repeat(cw.astype(np.float32), reps, axis=0).astype(np.float64)
    for s in range(T):
        run = (run + rew[:, s]).astype(np.float32)
        d = (term[:, s] | trunc[:, s]).astype(bool)
        rs[d] += np.sum(w[d] * run[d].astype(np.float64), axis=1)
        rc[d] += 1
        run[d] = 0
    assert np.array_equal(t.get("ret_cnt"), rc)
    assert_close(t.get("ret_sum"), rs, 1e-12, floor=1e-12, what="completed returns")
    assert np.array_equal(t.get("tracker"), run)
    return errs, n_term, n_trunc


def test_rollout_teacher_forced_humanoid6_bench_widths(mb, o):
    """64 envs per cluster and H = 256 (two 128-feature tiles, nepad 64), T = 64,
    with truncations and falls forced inside the window: the step counters of
    every other instance are set close to the 1000-step horizon and some
    instances start tilted past the fall threshold."""
    c = bench_cfg(K=8, T=64)

    def prepare(t):
        N = c.N
        steps = np.zeros(N, np.int32)
        steps[::2] = 1000 - 1 - (np.arange(0, N, 2) * 7) % 90  # truncate at t = 0..89
        t.set("env_steps", steps)
        st = t.get("env_state")  # SoA [state][N]
        fall = np.arange(N) % 16 == 3
        st[40, fall] = 0.995  # roll
        st[42, fall] = 0.8    # roll rate: |roll| > 1 within a few steps
        t.set("env_state", st)

    errs, n_term, n_trunc = _teacher_forced(mb, o, c, prepare)
    assert n_term > 0 and n_trunc > 0, (n_term, n_trunc)
    print("humanoid6 teacher-forced max normwise errors:", errs, "term", n_term, "trunc", n_trunc)


def _force_boundaries(c):
    """Truncations and falls inside the window (mo-humanoid6)."""
    def prepare(t):
        N = c.N
        steps = np.zeros(N, np.int32)
        steps[::2] = 1000 - 1 - (np.arange(0, N, 2) * 7) % 90
        t.set("env_steps", steps)
        st = t.get("env_state")
        fall = np.arange(N) % 16 == 3
        st[40, fall] = 0.995
        st[42, fall] = 0.8
        t.set("env_state", st)
    return prepare


def test_rollout_teacher_forced_deep_ragged_nets(mb, o):
    """Three hidden layers of unequal widths (the in-place hidden buffer
    changes its padded K between layers: 200 -> 256 -> 100 features, one or
    two 128-feature tiles, zeros in the padded features) and 40 instances
    per cluster (nepad 48, a partial 8-env block)."""
    c = bench_cfg(K=4, T=24, N=160, F=64, feat_hidden=[64], actor_hidden=[200, 256, 100],
                  critic_hidden=[96, 256, 40], seed=5)
    errs, n_term, n_trunc = _teacher_forced(mb, o, c, _force_boundaries(c))
    assert n_term > 0 and n_trunc > 0, (n_term, n_trunc)
    print("deep / ragged teacher-forced max normwise errors:", errs, "term", n_term, "trunc", n_trunc)


def test_rollout_teacher_forced_two_ctas_per_cluster(mb, o):
    """100 instances per cluster at bench widths: two rollout CTAs (64 + 36
    instances) stream the same cluster's weights; boundaries forced in both."""
    c = bench_cfg(K=2, T=32, N=200, seed=12)
    errs, n_term, n_trunc = _teacher_forced(mb, o, c, _force_boundaries(c))
    assert n_term > 0 and n_trunc > 0, (n_term, n_trunc)
    print("two-CTA teacher-forced max normwise errors:", errs, "term", n_term, "trunc", n_trunc)


def test_rollout_teacher_forced_pointmass_truncation(mb, o):
    """mo-pointmass past its 200-step horizon: every instance truncates and
    auto-resets inside the fused rollout (T = 210)."""
    c = TrainCfg(env="mo-pointmass", N=128, K=4, T=210, F=64, feat_hidden=[64], actor_hidden=[64, 64],
                 critic_hidden=[64, 64], seed=9)
    errs, n_term, n_trunc = _teacher_forced(mb, o, c)
    assert n_trunc == c.N, n_trunc
    print("pointmass teacher-forced max normwise errors:", errs)


def test_rollout_teacher_forced_dst_terminals(mb, o):
    """mo-dst-continuous: terminal treasures and the 50-step truncation at T = 64."""
    c = TrainCfg(env="mo-dst-continuous", N=128, K=2, T=64, F=32, feat_hidden=[32], actor_hidden=[64, 64],
                 critic_hidden=[64, 64], seed=4)
    errs, n_term, n_trunc = _teacher_forced(mb, o, c)
    assert n_trunc > 0, (n_term, n_trunc)
    print("dst teacher-forced max normwise errors:", errs, "term", n_term, "trunc", n_trunc)


# ------------------------------------------------------------------ losses / gradients at bench widths
# ragged widths: partial 128-row / 256-column GEMM tiles everywhere, a
# last hidden layer that is not a multiple of 16 (k_head's K loop), a
# 3-hidden-layer actor, F = 192 (the fused dM + Adam's 64-wide tiles)
RAGGED = dict(F=192, feat_hidden=[100], actor_hidden=[200, 136, 72], critic_hidden=[96, 40])


@pytest.mark.parametrize("widths", ["bench", "ragged"])
def test_losses_and_grads_bench_widths(mb, o, widths):
    """actor_loss / critic_loss + hypernet backward (losses.cpp:46-189) at
    config-3 widths on the device's own rollout batch (fed unchanged to the
    oracle): the act_dim-12 head, 256-wide dX epilogues and grouped dW; and
    at ragged widths."""
    c = bench_cfg(K=4, T=8, **(RAGGED if widths == "ragged" else {}))
    t = mb.Trainer(_mbcfg(mb, c))
    t.phase(0, 1)
    t.phase(0, 2)
    a_s, c_s = c.specs()
    N, T = c.N, c.T
    reps = N // c.K
    af, cf = t.params("actor"), t.params("critic")
    obs = t.get("obs").astype(np.float64)
    act = t.get("action_pre").astype(np.float64)
    lpo = t.get("logprob").astype(np.float64)
    sadv = t.get("scalar_advantage").astype(np.float64)
    tgt = t.get("value_targets").astype(np.float64)
    cw = t.get("clusters").astype(np.float64)
    cw /= cw.sum(axis=1, keepdims=True)  # fp64 simplex check of the oracle (hypernet.cpp:58)
    tw = np.repeat(cw, reps, axis=0)
    cl = np.repeat(np.arange(c.K), reps).astype(np.int32)
    rows = np.random.default_rng(0).permutation(N * T)[:1024].astype(np.int32)
    la, lc = t.losses(rows)
    ga, gc = t.grad("actor"), t.grad("critic")
    la_o, ga_o = o.actor_loss(a_s, af, N, T, obs, act, lpo, tw, cl, rows, sadv, c.clip_eps, c.entropy_coef)
    lc_o, gc_o = o.critic_loss(c_s, cf, N, T, obs, tw, cl, rows, tgt)
    assert abs(la - la_o) <= REL_BF16 * max(1.0, abs(la_o)), (la, la_o)
    assert abs(lc - lc_o) <= REL_BF16 * max(1.0, abs(lc_o)), (lc, lc_o)
    for which, g, g_o, spec in (("actor", ga, ga_o, a_s), ("critic", gc, gc_o, c_s)):
        for name, (lo, hi) in hyper_blocks(spec).items():
            assert_normwise(g[lo:hi], g_o[lo:hi], REL_BF16, what=f"{which} grad {name}")


# ------------------------------------------------------------------ full iteration at bench widths
@pytest.mark.parametrize("widths", ["bench", "ragged"])
def test_full_iteration_bench_widths(mb, o, widths):
    """One whole training iteration (rollout -> GAE -> 2 x 2 minibatches of
    both losses + Adam) at config-3 widths (and at ragged widths) vs the fp64
    oracle, compared in update space per hypernet block."""
    c = bench_cfg(K=4, T=8, **(RAGGED if widths == "ragged" else {}))
    t = mb.Trainer(_mbcfg(mb, c))
    ot = OracleTrainer(o, c)
    a0, c0 = t.params("actor"), t.params("critic")
    st = t.iteration(0)
    al, cl = ot.iteration(0)
    assert st.minibatches == 4
    assert np.array_equal(t.get("perm"), ot.perm())
    assert abs(st.actor_loss - al) <= 2e-2 * max(1, abs(al)), (st.actor_loss, al)
    assert abs(st.critic_loss - cl) <= 2e-2 * max(1, abs(cl)), (st.critic_loss, cl)
    a_s, c_s = c.specs()
    ea = assert_update_close(t.params("actor"), ot.actor_params(), a0, c.actor_lr, hyper_blocks(a_s),
                             rel_l2=0.1, sign_agree=0.999, what="actor")
    ec = assert_update_close(t.params("critic"), ot.critic_params(), c0, c.critic_lr, hyper_blocks(c_s),
                             rel_l2=0.1, sign_agree=0.999, what="critic")
    print(widths, "iteration update errors: actor", ea, "critic", ec)
