"""Pins the C oracle (oracle/morlax_oracle.c) against fixtures produced by
the compiled reference (tests/golden/make_golden.py). CPU only; runs on the
GPU box too (no /root/reference needed)."""
import numpy as np
import pytest

from helpers import golden
from pyoracle import Oracle, TrainCfg

import ctypes as C


@pytest.fixture(scope="module")
def o():
    return Oracle("oracle")


@pytest.fixture(scope="module")
def g():
    return golden()


def test_rng_words_splits_gaussians_shuffle(o, g):
    keys = [o.rng_seed_state(int(s))[0] for s in g["rng_seeds"]]
    assert np.array_equal(np.array(keys, np.uint64), g["rng_keys"])
    k0 = int(g["rng_keys"][0])
    assert np.array_equal(o.rng_words(k0, 0, 256), g["rng_words_k0"])
    assert np.array_equal(o.rng_words(k0, 1000, 64), g["rng_words_k0_ctr1000"])
    sk = [o.split_key(k0, int(l)) for l in g["rng_split_lanes"]]
    assert np.array_equal(np.array(sk, np.uint64), g["rng_split_keys_k0"])
    assert np.array_equal(o.rng_gaussians(k0, 0, 128), g["rng_gauss_k0"])
    v, ctr = o.shuffle(k0, 0, np.arange(100))
    assert np.array_equal(v, g["rng_shuffle_k0"]) and ctr == int(g["rng_shuffle_k0_ctr"][0])


@pytest.mark.parametrize("name", ["mo-lqr1d", "mo-pointmass", "mo-dst-continuous", "mo-humanoid6"])
def test_env_traces(o, g, name):
    key = name.replace("-", "_")
    e = o.env(name, 4)
    obs0 = e.reset(int(g[f"env_{key}_reset_key"][0]))
    assert np.array_equal(obs0, g[f"env_{key}_obs0"])
    acts = g[f"env_{key}_actions"]
    for t in range(len(acts)):
        ob, rw, te, tr = e.step(acts[t])
        assert np.array_equal(ob, g[f"env_{key}_obs"][t])
        assert np.array_equal(rw, g[f"env_{key}_reward"][t])
        assert np.array_equal(te, g[f"env_{key}_term"][t])
        assert np.array_equal(tr, g[f"env_{key}_trunc"][t])
    assert e.clamp_count() == int(g[f"env_{key}_clamps"][0])


def _tiny():
    return TrainCfg(env="mo-pointmass", N=8, K=2, T=12, epochs=2, minibatch_count=2, F=8,
                    feat_hidden=[8], actor_hidden=[8, 8], critic_hidden=[8, 8], seed=5)


def test_hypernet_init_forward_backward(o, g):
    cfg = _tiny()
    a, c = cfg.specs()
    root = o.rng_seed_state(cfg.seed)[0]
    assert np.array_equal(o.init_hypernet(a, o.split_key(root, 0xA1)), g["hyper_actor_init"])
    assert np.array_equal(o.init_hypernet(c, o.split_key(root, 0xA2)), g["hyper_critic_init"])
    aflat = g["hyper_actor_init"]
    th = np.array([o.hypernet_forward(a, aflat, w) for w in g["hyper_w"]])
    assert np.array_equal(th, g["hyper_actor_theta"])
    gr = sum(o.hypernet_backward(a, aflat, g["hyper_w"][i], g["hyper_gtheta"][i]) for i in range(3))
    np.testing.assert_allclose(gr, g["hyper_actor_grad"], rtol=1e-13, atol=1e-15)


def test_rollout_gae_losses_adam(o, g):
    cfg = _tiny()
    a, c = cfg.specs()
    root = o.rng_seed_state(cfg.seed)[0]
    aflat, cflat = g["hyper_actor_init"], g["hyper_critic_init"]
    env = o.env("mo-pointmass", 8)
    env.reset(o.split_key(root, 0xE0))
    b = o.collect_rollouts(a, aflat, c, cflat, env, g["roll_cw"], 4, 12, o.split_key(root, 77), 0)
    for k, v in b.items():
        assert np.array_equal(v, g["roll_" + k]), k
    adv, tgt = o.gae(b["reward"], b["value"], b["next_value"], b["term"], b["trunc"], 8, 12, 0.99, 0.95)
    assert np.array_equal(adv, g["gae_adv"]) and np.array_equal(tgt, g["gae_tgt"])
    tw = np.repeat(g["roll_cw"], 4, axis=0)
    sadv = o.normalize_scalarize(adv, tw, 8, 12)
    assert np.array_equal(sadv, g["gae_sadv"])
    cl = np.repeat(np.arange(2), 4).astype(np.int32)
    la, ga = o.actor_loss(a, aflat, 8, 12, b["obs"], b["action_pre"], b["logprob"], tw, cl,
                          g["loss_rows"], sadv, 0.2, 0.1)
    lc, gc = o.critic_loss(c, cflat, 8, 12, b["obs"], tw, cl, g["loss_rows"], tgt)
    assert la == g["loss_actor"][0] and lc == g["loss_critic"][0]
    assert np.array_equal(ga, g["loss_actor_grad"]) and np.array_equal(gc, g["loss_critic_grad"])
    p1, m1, m2, st = o.adam(g["adam_p0"], g["adam_g"], np.zeros(64), np.zeros(64), 0, 1e-3)
    assert st == 1
    assert np.array_equal(p1, g["adam_p1"]) and np.array_equal(m1, g["adam_m1"])
    assert np.array_equal(m2, g["adam_m2"])


def test_train_two_iterations_matches_reference_train(o, g):
    """The oracle's train-loop restatement equals the reference train() (2 iterations)."""
    from pyoracle import OracleTrainer
    t = OracleTrainer(o, _tiny())
    t.iteration(0)
    t.iteration(1)
    assert np.array_equal(t.actor_params(), g["train2_actor"])
    assert np.array_equal(t.critic_params(), g["train2_critic"])


def test_pareto_mask_and_hypervolume(o, g):
    assert np.array_equal(o.nondominated_mask(g["pareto_pts3"]), g["pareto_mask3"])
    for m in (2, 3, 4):
        v, se, ex, _ = o.hypervolume_detailed(g[f"hv_pts{m}"], np.zeros(m))
        assert ex and se == 0.0
        assert abs(v - g[f"hv_exact{m}"][0]) <= 1e-12 * abs(v)
    v, se, ex, _ = o.hypervolume_detailed(g["hv_pts6"], np.zeros(6), samples=200_000)
    assert not ex
    assert v == g["hv_mc6"][0] and se == g["hv_mc6"][1]


def test_wfg_exact_matches_reference_exact_for_small_m(o, g):
    for m in (2, 3, 4):
        v = o.hypervolume_wfg(g[f"hv_pts{m}"], np.zeros(m))
        assert abs(v - g[f"hv_exact{m}"][0]) <= 1e-12 * abs(v)
    # m = 6: exact within 4 stderr of the reference Monte-Carlo
    v = o.hypervolume_wfg(g["hv_pts6"], np.zeros(6))
    assert abs(v - g["hv_mc6"][0]) <= 4 * g["hv_mc6"][1]


@pytest.mark.parametrize("m", [2, 3, 4, 6])
def test_linear_dominance_oracle_matches_reference(o, g, m):
    # golden: the reference's linear_dominance_filter (pareto.cpp:79-139)
    assert np.array_equal(o.linear_dominance_mask(g[f"ldf_pts{m}"]), g[f"ldf_mask{m}"])


@pytest.mark.parametrize("env,od,ad,res,eps", [("mo-pointmass", 4, 2, 4, 3), ("mo-lqr1d", 1, 1, 3, 2)])
def test_evaluate_params_oracle_matches_reference(o, g, env, od, ad, res, eps):
    # golden: the reference's evaluate_params (evaluate.cpp:17-101)
    from pyoracle import ENV_KINDS, HSpec
    spec = HSpec(2, 16, [16], [od, 32, 32, ad], True, True)
    W, R = o.evaluate_params(spec, g[f"eval_{env}_flat"], ENV_KINDS[env], res, eps, 0x1234)
    assert np.array_equal(W, g[f"eval_{env}_W"])
    assert np.array_equal(R, g[f"eval_{env}_R"])
