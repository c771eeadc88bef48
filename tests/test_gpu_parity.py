"""GPU parity: the CUDA path (through the C-ABI) vs the C oracle on identical
seeded inputs. Integer outputs (RNG words, flags, perms, masks, hit counts)
are compared bit-exactly; float outputs within the tolerances of
tests/helpers.py. Inputs fed to both sides are fp32-representable so the
only difference is device arithmetic."""
import numpy as np
import pytest

from helpers import (REL_BF16, REL_CHAIN, REL_F32, assert_close, assert_normwise, assert_update_close, golden,
                     hyper_blocks)
from pyoracle import Oracle, OracleTrainer, TrainCfg

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def mb():
    import paper_2603_09237_b200 as mb
    return mb


@pytest.fixture(scope="module")
def o():
    return Oracle("oracle")


@pytest.fixture(scope="module")
def g():
    return golden()


def r32(x):
    return np.asarray(x, np.float32).astype(np.float64)


# ------------------------------------------------------------------ RNG
def test_rng_words_bit_exact(mb, o, g):
    k0 = int(g["rng_keys"][0])
    assert np.array_equal(mb.rng_words(k0, 0, 256), g["rng_words_k0"])
    assert np.array_equal(mb.rng_words(k0, 1000, 64), g["rng_words_k0_ctr1000"])
    big = mb.rng_words(0x1234567, 99, 1 << 20)
    assert np.array_equal(big, o.rng_words(0x1234567, 99, 1 << 20))


def test_rng_gaussians(mb, g):
    k0 = int(g["rng_keys"][0])
    got = mb.rng_gaussians(k0, 0, 128)
    # same words; fp64 log/cos may differ from glibc in the last ulp
    assert_close(got, g["rng_gauss_k0"], 1e-14, floor=1e-12, what="box-muller")


# ------------------------------------------------------------------ env (K1)
@pytest.mark.parametrize("name", ["mo-lqr1d", "mo-pointmass", "mo-dst-continuous", "mo-humanoid6"])
def test_env_step_parity(mb, o, g, name):
    key = name.replace("-", "_")
    acts = r32(g[f"env_{key}_actions"])
    rk = int(g[f"env_{key}_reset_key"][0])
    e, eo = mb.BatchedEnv(name, 4), o.env(name, 4)
    assert_close(e.reset(rk), eo.reset(rk), 1e-7, what="reset obs")
    for t in range(len(acts)):
        s = e.step(acts[t])
        ob, rw, te, tr = eo.step(acts[t])
        assert np.array_equal(s.terminated, te) and np.array_equal(s.truncated, tr), t
        # per-step error <= 1e-5; fp32 state accumulated over up to 205 steps
        # drifts from the fp64 reference, so the bound grows to 1e-4 after 32 steps
        tol = REL_F32 if t < 32 else 10 * REL_F32
        assert_close(s.obs, ob, tol, floor=1e-2, what=f"{name} obs t={t}")
        assert_close(s.reward, rw, tol, floor=1e-2, what=f"{name} reward t={t}")
    assert e.clamp_count() == eo.clamp_count()


def test_env_large_batch_auto_reset(mb, o):
    n = 8192
    e, eo = mb.BatchedEnv("mo-pointmass", n), o.env("mo-pointmass", n)
    e.reset(77)
    eo.reset(77)
    rng = np.random.default_rng(0)
    for t in range(201):
        a = r32(rng.uniform(-1, 1, (n, 2)))
        s = e.step(a)
        ob, rw, te, tr = eo.step(a)
        assert np.array_equal(s.truncated, tr)
    assert_close(e.current_obs(), eo.current_obs(), REL_F32, floor=1e-4, what="post-reset obs")


def test_env_rejects_non_finite_action(mb):
    e = mb.BatchedEnv("mo-pointmass", 2)
    e.reset(1)
    with pytest.raises(mb.NumericError):
        e.step(np.array([[0.1, np.nan], [0.0, 0.0]]))


# ------------------------------------------------------------------ hypernet (K2/K6)
@pytest.mark.parametrize("F,fh,ah,od,ad,m", [(8, [8], [8, 8], 4, 2, 2), (64, [64], [64, 64], 4, 2, 2),
                                             (256, [256], [256, 256], 45, 12, 6)])
def test_hypernet_forward_backward(mb, o, F, fh, ah, od, ad, m):
    from pyoracle import HSpec
    spec_o = HSpec(m, F, fh, [od] + ah + [ad], True, True)
    spec = mb.HypernetSpec(m, F, fh, [od] + ah + [ad], True, True)
    flat = o.init_hypernet(spec_o, 0xBEEF)
    dev_init = mb.init_hypernet(spec, 0xBEEF)
    assert_close(dev_init, flat, 1e-6, floor=1e-9, what="init_hypernet")
    flat = r32(flat)
    rng = np.random.default_rng(3)
    W = rng.dirichlet(np.ones(m), size=5)
    th = mb.hypernet_forward(spec, flat, W)
    th_o = np.array([o.hypernet_forward(spec_o, flat, w) for w in W])
    assert_normwise(th, th_o, REL_BF16, what="theta")
    gth = r32(rng.normal(size=th.shape))
    gr = mb.hypernet_backward(spec, flat, W, gth)
    gr_o = sum(o.hypernet_backward(spec_o, flat, W[i], gth[i]) for i in range(len(W)))
    assert_normwise(gr, gr_o, REL_BF16, what="hypernet grad")


def _mlp_pre(theta, sizes, x):
    """nn.cpp:60-92 mlp_forward restated in numpy (fp64): tanh hidden layers,
    identity output (the pre-squash Gaussian mean)."""
    off = 0
    a = x
    L = len(sizes) - 1
    for l in range(L):
        i, o_ = sizes[l], sizes[l + 1]
        W = theta[off:off + i * o_].reshape(o_, i)
        b = theta[off + i * o_:off + i * o_ + o_]
        off += (i + 1) * o_
        a = a @ W.T + b
        if l < L - 1:
            a = np.tanh(a)
    return a


@pytest.mark.parametrize("F,fh,ah,od,ad,m,G,R", [(16, [16], [32, 32], 4, 2, 2, 3, 50),
                                                 (256, [256], [256, 256], 48, 12, 3, 8, 256)])
def test_group_policy_forward(mb, o, F, fh, ah, od, ad, m, G, R):
    """Per-preference-group policy forward (config-2 shapes scaled down):
    theta from the oracle's hypernet_forward, then the reference MLP."""
    from pyoracle import HSpec
    sizes = [od] + ah + [ad]
    spec_o = HSpec(m, F, fh, sizes, True, True)
    spec = mb.HypernetSpec(m, F, fh, sizes, True, True)
    flat = r32(o.init_hypernet(spec_o, 0x51))
    rng = np.random.default_rng(1)
    W = rng.dirichlet(np.ones(m), size=G)
    obs = r32(rng.normal(size=(G * R, od)))
    pf = mb.PolicyForward(spec, G, R)
    pf.set_params(flat)
    pre = pf.forward(W, obs)
    ref = np.concatenate([_mlp_pre(o.hypernet_forward(spec_o, flat, W[g]), sizes, obs[g * R:(g + 1) * R])
                          for g in range(G)])
    assert pre.shape == ref.shape
    assert_normwise(pre, ref, REL_BF16, what="policy pre-activation")
    with pytest.raises(mb.DomainError):
        pf.forward(np.full((G, m), 0.9), obs)


# ------------------------------------------------------------------ GAE / normalise (K4)
# (T <= 256 with the staged blocks under 48 KB: the per-instance staged
# kernel; T = 300 and the m = 8, T = 64 case: the warp-scan kernel)
@pytest.mark.parametrize("T,m", [(1, 6), (16, 6), (32, 6), (64, 6), (100, 6), (300, 6), (64, 2), (64, 8)])
def test_gae_scan_parity(mb, o, T, m):
    rng = np.random.default_rng(T)
    N = 37
    r, v, nv = (r32(rng.normal(size=(N * T, m))) for _ in range(3))
    u = rng.random(N * T)
    te = (u < 0.03).astype(np.uint8)
    tr = ((u >= 0.03) & (u < 0.06)).astype(np.uint8)
    adv, tg = mb.gae_per_objective(r, v, nv, te, tr, N, T, 0.99, 0.95)
    adv_o, tg_o = o.gae(r, v, nv, te, tr, N, T, 0.99, 0.95)
    # floor = natural scale of the data (rewards/values ~ N(0, 1))
    assert_close(adv, adv_o, REL_F32, floor=1.0, what="advantages")
    assert_close(tg, tg_o, REL_F32, floor=1.0, what="targets")
    tw = rng.dirichlet(np.ones(m), size=N)
    s = mb.normalize_and_scalarize(r32(adv_o), tw, N, T)
    s_o = o.normalize_scalarize(r32(adv_o), r32(tw), N, T)
    assert_close(s, s_o, REL_F32, floor=1.0, what="scalar advantages")


def test_gae_reference_hand_fixture(mb):  # test_gae.cpp:109-134
    adv, tg = mb.gae_per_objective([[1.0], [1.0]], [[2.0], [1.0]], [[3.0], [4.0]], [0, 0], [0, 1],
                                   1, 2, 0.5, 0.5)
    assert adv[:, 0].tolist() == [1.0, 2.0] and tg[:, 0].tolist() == [3.0, 3.0]
    adv, tg = mb.gae_per_objective([[1.0], [1.0]], [[2.0], [1.0]], [[3.0], [4.0]], [0, 1], [0, 0],
                                   1, 2, 0.5, 0.5)
    assert adv[:, 0].tolist() == [0.5, 0.0] and tg[:, 0].tolist() == [2.5, 1.0]


# ------------------------------------------------------------------ Adam (K7)
def test_adam_parity(mb, o):
    rng = np.random.default_rng(5)
    n = 1003
    p = r32(rng.normal(size=n))
    m1 = np.zeros(n)
    m2 = np.zeros(n)
    po, m1o, m2o, st, sto = p.copy(), m1.copy(), m2.copy(), 0, 0
    for _ in range(5):
        gr = r32(rng.normal(size=n))
        p, m1, m2, st = mb.adam_apply(p, gr, m1, m2, st, 1e-3)
        po, m1o, m2o, sto = o.adam(po, gr, m1o, m2o, sto, 1e-3)
    assert st == sto == 5
    assert_close(p, po, REL_F32, floor=1e-3, what="adam params")


def test_adam_first_step_moves_by_lr(mb):  # test_trainer.cpp:486-497
    p, _, _, _ = mb.adam_apply([0.0], [1.0], [0.0], [0.0], 0, 0.1)
    assert abs(p[0] + 0.1) < 1e-6


# ------------------------------------------------------------------ trainer pieces
def _tiny(env="mo-pointmass", **kw):
    base = dict(env=env, N=8, K=2, T=12, epochs=2, minibatch_count=1, F=8, feat_hidden=[8],
                actor_hidden=[8, 8], critic_hidden=[8, 8], seed=5)
    base.update(kw)
    return TrainCfg(**base)


def _mbcfg(mb, c: TrainCfg):
    return mb.TrainConfig(env_name=c.env, N=c.N, K=c.K, kappa=c.kappa, T=c.T, epochs=c.epochs,
                          minibatch_count=c.minibatch_count, gamma=c.gamma, gae_lambda=c.lam,
                          clip_eps=c.clip_eps, actor_lr=c.actor_lr, critic_lr=c.critic_lr,
                          entropy_coef=c.entropy_coef, seed=c.seed, F=c.F,
                          feature_hidden=c.feat_hidden, actor_hidden=c.actor_hidden,
                          critic_hidden=c.critic_hidden)


def test_trainer_init_matches_reference_init(mb, o, g):
    t = mb.Trainer(_mbcfg(mb, _tiny()))
    assert_close(t.params("actor"), g["hyper_actor_init"], 1e-6, floor=1e-9, what="actor init")
    assert_close(t.params("critic"), g["hyper_critic_init"], 1e-6, floor=1e-9, what="critic init")


def test_losses_and_grads_parity(mb, o, g):
    """actor_loss / critic_loss through the hypernet on the reference rollout batch."""
    c = _tiny()
    a_s, c_s = c.specs()
    t = mb.Trainer(_mbcfg(mb, c))
    af, cf = r32(g["hyper_actor_init"]), r32(g["hyper_critic_init"])
    t.set_params("actor", af)
    t.set_params("critic", cf)
    obs, act, lp = r32(g["roll_obs"]), r32(g["roll_action_pre"]), r32(g["roll_logprob"])
    sadv, tgt = r32(g["gae_sadv"]), r32(g["gae_tgt"])
    cw = r32(g["roll_cw"])
    t.set("obs", obs)
    t.set("action_pre", act)
    t.set("logprob", lp)
    t.set("scalar_advantage", sadv)
    t.set("value_targets", tgt)
    t.set("clusters", cw)
    rows = g["loss_rows"]
    la, lc = t.losses(rows)
    tw = np.repeat(cw, 4, axis=0)
    cl = np.repeat(np.arange(2), 4).astype(np.int32)
    tw = np.repeat(g["roll_cw"], 4, axis=0)  # oracle keeps its fp64 simplex check
    la_o, ga_o = o.actor_loss(a_s, af, 8, 12, obs, act, lp, tw, cl, rows, sadv, 0.2, 0.1)
    lc_o, gc_o = o.critic_loss(c_s, cf, 8, 12, obs, tw, cl, rows, tgt)
    assert abs(la - la_o) <= REL_BF16 * max(1.0, abs(la_o))
    assert abs(lc - lc_o) <= REL_BF16 * max(1.0, abs(lc_o))
    assert_normwise(t.grad("actor"), ga_o, REL_BF16, what="actor grad")
    assert_normwise(t.grad("critic"), gc_o, REL_BF16, what="critic grad")


@pytest.mark.parametrize("env", ["mo-pointmass", "mo-humanoid6"])
def test_rollout_and_advantages_parity(mb, o, env):
    kw = dict(N=32, K=4, T=16, F=16, feat_hidden=[16], actor_hidden=[32, 32], critic_hidden=[32, 32])
    c = _tiny(env, **kw)
    t = mb.Trainer(_mbcfg(mb, c))
    ot = OracleTrainer(o, c)
    t.phase(0, 1)
    t.phase(0, 2)
    ot.iteration(0, max_minibatches=0)
    b = ot.batch()
    assert_close(t.get("clusters"), ot.clusters(), 1e-7, floor=1e-9, what="clusters")
    assert np.array_equal(t.get("terminated"), b["term"])
    assert np.array_equal(t.get("truncated"), b["trunc"])
    for name, key in (("obs", "obs"), ("action_pre", "action_pre"), ("logprob", "logprob"),
                      ("reward", "reward"), ("value", "value"), ("next_value", "next_value"),
                      ("advantages", "adv"), ("value_targets", "targets"),
                      ("scalar_advantage", "sadv")):
        assert_normwise(t.get(name), b[key], REL_CHAIN, what=name)


@pytest.mark.parametrize("F,fused,H", [(16, "1", 32), (64, "1", 32), (64, "0", 32), (16, "1", 48), (16, "1", 16)])
def test_full_iteration_parity(mb, o, monkeypatch, F, fused, H):
    """F = 64 takes the single-rank fused dM + Adam kernel (dm_adam.cu) unless
    MORLAX_FUSED_ADAM=0 (the tcgen05 dM GEMM + separate Adam); H = 48 / 16
    cover the head kernel's partial 32-column group of the output layer's
    backward."""
    monkeypatch.setenv("MORLAX_FUSED_ADAM", fused)
    c = _tiny(N=32, K=4, T=16, epochs=2, minibatch_count=2, F=F, feat_hidden=[16],
              actor_hidden=[H, H], critic_hidden=[H, H])
    t = mb.Trainer(_mbcfg(mb, c))
    ot = OracleTrainer(o, c)
    a0, c0 = t.params("actor"), t.params("critic")
    st = t.iteration(0)
    al, cl = ot.iteration(0)
    assert st.minibatches == 4
    assert abs(st.actor_loss - al) <= REL_CHAIN * max(1, abs(al))
    assert abs(st.critic_loss - cl) <= REL_CHAIN * max(1, abs(cl))
    assert np.array_equal(t.get("perm"), ot.perm())
    a_s, c_s = c.specs()
    for which, ref, p0, spec, lr in (("actor", ot.actor_params(), a0, a_s, c.actor_lr),
                                     ("critic", ot.critic_params(), c0, c_s, c.critic_lr)):
        # update space: (p - p0) vs (ref - p0) per hypernet block (helpers.update_errors)
        e = assert_update_close(t.params(which), ref, p0, lr, hyper_blocks(spec), rel_l2=0.1, sign_agree=0.995,
                                what=which)
        print(f"F={F} fused={fused} H={H} {which} update errors: {e}")


@pytest.mark.parametrize("F", [8, 64])
def test_iteration_is_deterministic(mb, F):
    c = _tiny(N=32, K=4, T=16, F=F)
    t1, t2 = mb.Trainer(_mbcfg(mb, c)), mb.Trainer(_mbcfg(mb, c))
    for it in range(2):
        s1, s2 = t1.iteration(it), t2.iteration(it)
        assert s1.actor_loss == s2.actor_loss and s1.critic_loss == s2.critic_loss
    assert np.array_equal(t1.params("actor"), t2.params("actor"))
    assert np.array_equal(t1.params("critic"), t2.params("critic"))


def test_trainer_config_errors(mb):
    with pytest.raises(mb.ConfigError):
        mb.Trainer(mb.TrainConfig(N=10, K=3))
    with pytest.raises(mb.ConfigError):
        mb.Trainer(mb.TrainConfig(env_name="nope"))


# ------------------------------------------------------------------ Pareto / HV (K8/K9)
def _front(n, m, seed):  # config-5 recipe: Dirichlet -> unit sphere + N(0, 0.02^2)
    rng = np.random.default_rng(seed)
    w = rng.dirichlet(np.ones(m), size=n)
    p = w / np.linalg.norm(w, axis=1, keepdims=True)
    return p + rng.normal(0, 0.02, p.shape)


def test_pareto_mask_bit_exact(mb, o, g):
    assert np.array_equal(mb.nondominated_mask(g["pareto_pts3"]), g["pareto_mask3"])
    p = _front(1024, 6, 4)
    p[100] = p[7]  # exact duplicate
    p[200] = np.round(p[200], 1)
    assert np.array_equal(mb.nondominated_mask(p), o.nondominated_mask(p))
    q = np.round(np.random.default_rng(1).normal(size=(600, 2)), 1)  # many ties
    assert np.array_equal(mb.nondominated_mask(q), o.nondominated_mask(q))


def test_hypervolume_mc_bit_exact(mb, o, g):
    key = o.rng_seed_state(0x9E3779B9)[0]
    v, se, _ = mb.hypervolume_mc(g["hv_pts6"], np.zeros(6), 200_000, key, 0)
    assert v == g["hv_mc6"][0] and se == g["hv_mc6"][1]
    p = _front(1024, 6, 4)
    ref = -np.ones(6)
    v, se, hits = mb.hypervolume_mc(p, ref, 1_000_000, key, 0)
    vo, seo, ho = o.hypervolume_mc(p, ref, 1_000_000, key, 0)
    assert hits == ho and v == vo and se == seo
    vd, sed, ex, cl = mb.hypervolume_detailed(p, ref)
    assert (vd, sed, ex) == (vo, seo, False) and cl == 0


# ------------------------------------------------------------------ exact hypervolume (device WFG)
def test_hypervolume_exact_known_answer(mb):  # test_pareto.cpp:130-137
    pts = np.array([[3.0, 1.0], [1.0, 3.0], [2.0, 2.0]])
    assert mb.hypervolume_exact(pts, np.zeros(2)) == (6.0, 0)
    v, se, ex, cl = mb.hypervolume_detailed(pts, np.zeros(2))
    assert (v, se, ex, cl) == (6.0, 0.0, True, 0)
    # 3-D: one point is its box; a dominated point and a duplicate add nothing
    p3 = np.array([[2.0, 3.0, 4.0], [1.0, 1.0, 1.0], [2.0, 3.0, 4.0]])
    assert mb.hypervolume_exact(p3, np.zeros(3))[0] == 24.0


@pytest.mark.parametrize("m", [2, 3, 4])
def test_hypervolume_exact_matches_reference_recursion(mb, o, g, m):
    # golden: the reference's own exact hv_recursive (pareto.cpp:145-189)
    v, se, ex, cl = mb.hypervolume_detailed(g[f"hv_pts{m}"], np.zeros(m))
    assert ex and se == 0.0
    assert abs(v - g[f"hv_exact{m}"][0]) <= 1e-12 * abs(g[f"hv_exact{m}"][0])
    p = _front(300, m, 11 + m)
    ref = -np.ones(m)
    vo = o.hypervolume_detailed(p, ref)[0]
    assert abs(mb.hypervolume_exact(p, ref)[0] - vo) <= 1e-12 * vo


def test_hypervolume_exact_m6_matches_oracle_wfg(mb, o, g):
    v = mb.hypervolume_exact(g["hv_pts6"], np.zeros(6))[0]
    vo = o.hypervolume_wfg(g["hv_pts6"], np.zeros(6))
    assert abs(v - vo) <= 1e-12 * abs(vo)
    # config 5: 1024 points on the 6-simplex projected onto the unit sphere
    # + N(0, 0.02^2), reference -1^6; exact vs the MC estimate within 4 sigma
    p = _front(1024, 6, 4)
    ref = -np.ones(6)
    v, cl = mb.hypervolume_exact(p, ref)
    vo = o.hypervolume_wfg(p, ref)
    assert cl == 0 and abs(v - vo) <= 1e-12 * vo
    vm, se, _, _ = mb.hypervolume_detailed(p, ref)
    assert abs(vm - v) <= 4 * se


def test_hypervolume_exact_edge_cases(mb):
    assert mb.hypervolume_exact(np.zeros((0, 3)), np.zeros(3)) == (0.0, 0)
    # every point below the reference in some coordinate: clipped, volume 0
    assert mb.hypervolume_exact(np.array([[1.0, -1.0, 1.0], [-2.0, 1.0, 1.0]]), np.zeros(3)) == (0.0, 2)
    assert mb.hypervolume_exact(np.array([[5.0], [3.0]]), np.array([1.0]))[0] == 4.0
    q = np.round(np.random.default_rng(5).uniform(0, 1, (200, 4)), 1)  # heavy ties and duplicates
    v = mb.hypervolume_exact(q, np.zeros(4))[0]
    vd = mb.hypervolume_detailed(q, np.zeros(4))[0]
    assert v == vd
    with pytest.raises(mb.ShapeError):
        mb.hypervolume_exact(np.zeros((3, 9)), np.zeros(9))


# ------------------------------------------------------------------ linear dominance filter (pareto.cpp:79-139)
@pytest.mark.parametrize("m", [2, 3, 4, 6])
def test_linear_dominance_bit_exact(mb, o, g, m):
    assert np.array_equal(mb.linear_dominance_mask(g[f"ldf_pts{m}"]), g[f"ldf_mask{m}"])


def test_linear_dominance_edge_cases(mb, o):
    line = np.array([[0.0, 1.0], [0.25, 0.75], [0.5, 0.5], [1.0, 0.0], [0.2, 0.2]])  # collinear: all kept
    assert list(mb.linear_dominance_mask(line)) == [1, 1, 1, 1, 0]
    q = np.round(np.random.default_rng(8).normal(size=(300, 2)), 1)  # ties / duplicates
    assert np.array_equal(mb.linear_dominance_mask(q), o.linear_dominance_mask(q))
    p3 = _front(200, 3, 9)
    p3[10] = p3[4]
    assert np.array_equal(mb.linear_dominance_mask(p3), o.linear_dominance_mask(p3))
    assert list(mb.linear_dominance_mask(np.array([[1.0, 2.0], [2.0, 1.0]]))) == [1, 1]  # |nd| <= 2
    assert mb.linear_dominance_mask(np.zeros((0, 3))).size == 0


# ------------------------------------------------------------------ evaluate_params (evaluate.cpp:17-101)
@pytest.mark.parametrize("env,od,ad,res,eps", [("mo-pointmass", 4, 2, 4, 3), ("mo-lqr1d", 1, 1, 3, 2)])
def test_evaluate_params_matches_reference(mb, g, env, od, ad, res, eps):
    """Deterministic first-episode returns over the simplex grid: bf16
    generated weights on the device vs the fp64 reference (chain tolerance:
    200-step trajectories through the policy)."""
    spec = mb.HypernetSpec(2, 16, [16], [od, 32, 32, ad], True, True)
    W, R = mb.evaluate_params(spec, r32(g[f"eval_{env}_flat"]), env, res, eps, 0x1234)
    assert np.array_equal(W, g[f"eval_{env}_W"])
    assert_normwise(R, g[f"eval_{env}_R"], REL_CHAIN, what=f"{env} mean returns")


def test_evaluate_params_oracle_envs(mb, o):
    """DST (terminal treasures) and mo-humanoid6 against the C oracle, and
    more episodes than one CTA holds (partial sums across CTAs)."""
    from pyoracle import ENV_KINDS, HSpec
    spec_o = HSpec(2, 16, [16], [1, 32, 32, 1], True, True)
    spec = mb.HypernetSpec(2, 16, [16], [1, 32, 32, 1], True, True)
    flat = r32(o.init_hypernet(spec_o, 0x99))
    W, R = mb.evaluate_params(spec, flat, "mo-dst-continuous", 5, 20, 7)
    Wo, Ro = o.evaluate_params(spec_o, flat, ENV_KINDS["mo-dst-continuous"], 5, 20, 7)
    assert np.array_equal(W, Wo)
    assert_normwise(R, Ro, REL_CHAIN, what="dst mean returns")
    spec_o = HSpec(6, 32, [32], [45, 64, 64, 12], True, True)
    spec = mb.HypernetSpec(6, 32, [32], [45, 64, 64, 12], True, True)
    flat = r32(o.init_hypernet(spec_o, 0x98))
    W, R = mb.evaluate_params(spec, flat, "mo-humanoid6", 1, 2, 5)
    Wo, Ro = o.evaluate_params(spec_o, flat, ENV_KINDS["mo-humanoid6"], 1, 2, 5)
    assert np.array_equal(W, Wo) and len(W) == 6
    assert_normwise(R, Ro, REL_CHAIN, what="humanoid6 mean returns")


def test_evaluate_params_errors(mb):
    spec = mb.HypernetSpec(2, 16, [16], [4, 32, 32, 2], True, True)
    flat = mb.init_hypernet(spec, 1)
    with pytest.raises(mb.ConfigError):
        mb.evaluate_params(spec, flat, "mo-pointmass", 4, 0, 1)
    with pytest.raises(mb.ShapeError):
        mb.evaluate_params(spec, flat, "mo-humanoid6", 4, 1, 1)


@pytest.mark.parametrize("F", [16, 64])
def test_single_rank_nccl_path_matches(mb, F):
    """The multi-GPU code path (NCCL all-reduces of the normalisation sums
    and the losses; the per-minibatch exchange: all-gather of the clusters'
    bf16 theta-gradient rows re-tiled for dM, all-reduces of db and the
    feature-map gradient; all on one stream) with a single-rank communicator
    gives bit-identical results to the no-NCCL run. F = 64 takes the fused
    dM + Adam kernel over the gathered rows."""
    cfg = mb.TrainConfig(env_name="mo-pointmass", N=64, K=4, T=16, epochs=2, minibatch_count=2, seed=5, F=F,
                         feature_hidden=[16], actor_hidden=[32, 32], critic_hidden=[32, 32])
    a = mb.Trainer(cfg)
    b = mb.Trainer(cfg, 1, 0, mb.nccl_unique_id())
    for it in range(2):
        sa, sb = a.iteration(it), b.iteration(it)
        assert sa.actor_loss == sb.actor_loss and sa.critic_loss == sb.critic_loss
    assert np.array_equal(a.params("actor"), b.params("actor"))
    assert np.array_equal(a.params("critic"), b.params("critic"))


# ------------------------------------------------------------------ checkpoint wire format (checkpoint.cpp)
def test_checkpoint_is_the_reference_format(mb, tmp_path):
    from helpers import ref_available
    cfg = mb.TrainConfig(env_name="mo-pointmass", N=32, K=4, T=8, epochs=1, minibatch_count=2, seed=3, F=16,
                         feature_hidden=[16], actor_hidden=[32, 32], critic_hidden=[32, 32])
    t = mb.Trainer(cfg)
    t.iteration(0)
    path = str(tmp_path / "ck.bin")
    t.save_checkpoint(path, 1, iterations=7, pareto_reference=[-1.0, -2.0])
    u = mb.Trainer(cfg)
    assert u.load_checkpoint(path) == 1
    assert np.array_equal(u.params("actor"), t.params("actor"))
    assert np.array_equal(u.params("critic"), t.params("critic"))
    bad = tmp_path / "bad.bin"
    bad.write_bytes(b"NOTACKPT" + open(path, "rb").read()[8:])
    with pytest.raises(mb.ConfigError):
        u.load_checkpoint(str(bad))
    trunc = tmp_path / "trunc.bin"
    trunc.write_bytes(open(path, "rb").read()[:100])
    with pytest.raises(mb.ConfigError):
        u.load_checkpoint(str(trunc))
    if ref_available():  # the compiled reference reads it and writes back the identical bytes
        r = Oracle("ref")
        out = str(tmp_path / "ref.bin")
        a, c, it = r.checkpoint_resave(path, out, t.n_actor, t.n_critic)
        assert it == 1 and np.array_equal(a, t.params("actor")) and np.array_equal(c, t.params("critic"))
        assert open(out, "rb").read() == open(path, "rb").read()


# ------------------------------------------------------------------ train() loop (train.cpp:55-229)
def _train_cfg():
    return _tiny(N=16, K=2, T=12, epochs=2, minibatch_count=2, F=16, feat_hidden=[16],
                 actor_hidden=[16, 16], critic_hidden=[16, 16])


def test_train_loop_drives_the_iteration_loop(mb, tmp_path):
    """train() = Trainer.iteration(0..n-1) (bit-identical params) + the
    evaluation / archive / files / callback around it."""
    c = _train_cfg()
    recs = []
    t = mb.train(_mbcfg(mb, c), mb.RunOptions(out_dir=str(tmp_path), iterations=3, grid_resolution=3,
                                              episodes_per_point=2, log_interval=2, deterministic=True),
                 callback=recs.append)
    u = mb.Trainer(_mbcfg(mb, c))
    for it in range(3):
        su = u.iteration(it)
        assert recs[it].iteration == it
        assert recs[it].actor_loss == su.actor_loss and recs[it].critic_loss == su.critic_loss
    assert np.array_equal(t.params("actor"), u.params("actor"))
    assert np.array_equal(t.params("critic"), u.params("critic"))
    lines = (tmp_path / "metrics.csv").read_text().splitlines()
    assert lines[0] == "iteration,wall_ms,cluster_0_return,cluster_1_return,archive_hypervolume"
    assert [ln.split(",")[:2] for ln in lines[1:]] == [[str(i), "0"] for i in range(3)]
    assert recs[0].archive_hypervolume > 0 and recs[1].archive_hypervolume == recs[0].archive_hypervolume
    v = mb.Trainer(_mbcfg(mb, c))
    assert v.load_checkpoint(str(tmp_path / "checkpoint.bin")) == 3
    assert np.array_equal(v.params("actor"), t.params("actor"))

    class Stop(Exception):
        pass

    def boom(r):
        if r.iteration == 1:
            raise Stop()
    with pytest.raises(Stop):
        mb.train(_mbcfg(mb, c), mb.RunOptions(iterations=3, log_interval=5), callback=boom)
    with pytest.raises(mb.ConfigError):
        mb.train(_mbcfg(mb, c), mb.RunOptions(iterations=1, pareto_reference=[0.0]))


def test_train_loop_matches_the_reference_train(mb, tmp_path):
    """metrics.csv (layout, iteration / wall_ms columns, cluster returns,
    archive hypervolume) and checkpoint.bin of train() vs the compiled
    reference train() on the same config (fp32 device path vs fp64)."""
    from helpers import ref_available
    if not ref_available():
        pytest.skip("compiled reference (oracle/_ref) not built")
    c = _train_cfg()
    its = 3
    recs = []
    t = mb.train(_mbcfg(mb, c), mb.RunOptions(out_dir=str(tmp_path / "gpu"), iterations=its, grid_resolution=3,
                                              episodes_per_point=2, log_interval=2, deterministic=True),
                 callback=recs.append)
    r = Oracle("ref")
    hv_ref, a_ref, c_ref = r.train_run(c, its, 3, 2, 2, str(tmp_path / "ref"), t.n_actor, t.n_critic)
    g = (tmp_path / "gpu" / "metrics.csv").read_text().splitlines()
    q = (tmp_path / "ref" / "metrics.csv").read_text().splitlines()
    assert g[0] == q[0] and len(g) == len(q) == its + 1
    for lg, lq in zip(g[1:], q[1:]):
        fg, fq = lg.split(","), lq.split(",")
        assert fg[:2] == fq[:2]
        vg, vq = np.array(fg[2:], float), np.array(fq[2:], float)
        assert np.array_equal(np.isnan(vg), np.isnan(vq))
        ok = ~np.isnan(vq)
        assert np.allclose(vg[ok], vq[ok], rtol=2e-2, atol=1e-2)
    assert np.allclose([x.archive_hypervolume for x in recs], hv_ref, rtol=2e-2)
    a, cc, it = r.checkpoint_resave(str(tmp_path / "gpu" / "checkpoint.bin"), str(tmp_path / "re.bin"),
                                    t.n_actor, t.n_critic)
    assert it == its
    a_s, c_s = c.specs()
    p0 = Oracle("oracle")
    a0 = p0.init_hypernet(a_s, p0.split_key(p0.rng_seed_state(c.seed)[0], 0xA1))  # train.cpp:67-70
    c0 = p0.init_hypernet(c_s, p0.split_key(p0.rng_seed_state(c.seed)[0], 0xA2))
    for p, ref, init, spec, lr in ((a, a_ref, a0, a_s, c.actor_lr), (cc, c_ref, c0, c_s, c.critic_lr)):
        e = assert_update_close(p, ref, init, lr, hyper_blocks(spec), rel_l2=0.1, sign_agree=0.995,
                                what="train() checkpoint")
        print("train() vs reference update errors:", e)
