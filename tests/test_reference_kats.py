"""Known-answer fixtures from the reference's own unit tests, run through
the C oracle (CPU). Each test cites the reference test it restates."""
import numpy as np
import pytest

from pyoracle import Oracle, TrainCfg


@pytest.fixture(scope="module")
def o():
    return Oracle("oracle")


def test_gae_single_terminal_step(o):  # test_gae.cpp:57-67
    adv, tg = o.gae(np.array([[1.0, 0.0]]), np.zeros((1, 2)), np.array([[5.0, 5.0]]),
                    np.array([1], np.uint8), np.array([0], np.uint8), 1, 1, 0.99, 0.95)
    assert adv.tolist() == [[1.0, 0.0]] and tg.tolist() == [[1.0, 0.0]]


@pytest.mark.parametrize("term,trunc,adv_exp,tgt_exp", [
    ([0, 0], [0, 1], [1.0, 2.0], [3.0, 3.0]),   # truncated final step keeps its bootstrap
    ([0, 1], [0, 0], [0.5, 0.0], [2.5, 1.0]),   # terminated final step zeroes it
])
def test_gae_hand_fixture(o, term, trunc, adv_exp, tgt_exp):  # test_gae.cpp:109-134
    adv, tg = o.gae(np.array([[1.0], [1.0]]), np.array([[2.0], [1.0]]), np.array([[3.0], [4.0]]),
                    np.array(term, np.uint8), np.array(trunc, np.uint8), 1, 2, 0.5, 0.5)
    assert adv[:, 0].tolist() == adv_exp and tg[:, 0].tolist() == tgt_exp


def test_gae_lambda_zero_is_td_residual(o):  # test_gae.cpp:69-79
    rng = np.random.default_rng(41)
    N, T, m = 3, 17, 2
    r, v, nv = (rng.uniform(-2, 2, (N * T, m)) for _ in range(3))
    u = rng.random(N * T)
    te = (u < 0.1).astype(np.uint8)
    tr = ((u >= 0.1) & (u < 0.2)).astype(np.uint8)
    adv, _ = o.gae(r, v, nv, te, tr, N, T, 0.9, 0.0)
    exp = r + 0.9 * nv * (1 - te)[:, None] - v
    assert np.array_equal(adv, exp)


def test_hypervolume_spec_fixture_is_six(o):  # test_pareto.cpp:130-137
    v, se, ex, cl = o.hypervolume_detailed(np.array([[3, 1], [1, 3], [2, 2]], float), np.zeros(2))
    assert v == 6.0 and ex and cl == 0


def test_hypervolume_clipping(o):  # test_pareto.cpp:151-156
    v, _, _, cl = o.hypervolume_detailed(np.array([[-1, 2], [3, 1]], float), np.zeros(2))
    assert cl == 1 and abs(v - 3.0) < 1e-12


def test_lqr_step_law(o):  # test_envs.cpp:168-203 (reward on the pre-transition state)
    e = o.env("mo-lqr1d", 1)
    e.reset(11)
    for t in range(20):
        x0 = e.current_obs()[0, 0]
        u = np.sin(0.7 * t) * 0.9
        ob, rw, te, tr = e.step([[u]])
        assert rw[0, 0] == -x0 * x0 and rw[0, 1] == -u * u
        assert ob[0, 0] == 0.9 * x0 + 0.5 * u


def test_pointmass_integrator(o):  # test_envs.cpp:232-254
    e = o.env("mo-pointmass", 1)
    e.reset(23)
    px, py = e.current_obs()[0, :2]
    vx = vy = 0.0
    for t in range(40):
        ux, uy = np.cos(0.3 * t), np.sin(0.5 * t) * 0.8
        ob, rw, _, _ = e.step([[ux, uy]])
        vx += 0.05 * ux
        vy += 0.05 * uy
        px += 0.05 * vx
        py += 0.05 * vy
        assert rw[0, 0] == vx and rw[0, 1] == -(ux * ux + uy * uy)
        assert ob[0].tolist() == [px, py, vx, vy]


def test_pointmass_truncates_at_200_and_auto_resets(o):  # test_envs.cpp:332-376
    e = o.env("mo-pointmass", 2)
    e.reset(5)
    for t in range(200):
        ob, rw, te, tr = e.step(np.zeros((2, 2)))
        assert te.sum() == 0
        assert tr.tolist() == ([1, 1] if t == 199 else [0, 0])
    assert np.all(e.current_obs()[:, 2:] == 0)


def test_dst_min_capture_times(o):  # test_oracles.cpp:201-212 (full-throttle descent)
    e = o.env("mo-dst-continuous", 1)
    e.reset(0)
    captured = None
    for t in range(50):
        _, rw, te, _ = e.step([[1.0]])
        if te[0]:
            captured = (t + 1, rw[0, 0])
            break
    assert captured == (1, 0.7)  # the first treasure sits at depth 1


def test_adam_first_step_is_lr_sign(o):  # test_trainer.cpp:486-497
    p, _, _, _ = o.adam([0.0], [1.0], [0.0], [0.0], 0, 0.1)
    assert abs(p[0] + 0.1) < 1e-6
    p, _, _, _ = o.adam([0.0], [-1.0], [0.0], [0.0], 0, 0.1)
    assert abs(p[0] - 0.1) < 1e-6


def test_adam_zero_grad_leaves_params(o):  # test_trainer.cpp:475-484
    p = np.array([0.5, -1.25, 3.0])
    m1 = np.zeros(3)
    m2 = np.zeros(3)
    st = 0
    for _ in range(3):
        p2, m1, m2, st = o.adam(p, np.zeros(3), m1, m2, st, 0.01)
        assert np.array_equal(p2, p)
    assert st == 3


def test_first_epoch_actor_loss_is_minus_mean_adv(o):  # test_trainer.cpp:279-292
    cfg = TrainCfg(env="mo-lqr1d", N=4, K=2, T=12, F=3, feat_hidden=[3, 3], actor_hidden=[4],
                   critic_hidden=[4])
    a, c = cfg.specs()
    af, cf = o.init_hypernet(a, 50), o.init_hypernet(c, 51)
    env = o.env("mo-lqr1d", 4)
    env.reset(51)
    cw = np.array([[0.7, 0.3], [0.2, 0.8]])
    b = o.collect_rollouts(a, af, c, cf, env, cw, 2, 12, 52, 0)
    adv, tg = o.gae(b["reward"], b["value"], b["next_value"], b["term"], b["trunc"], 4, 12, 0.99, 0.95)
    tw = np.repeat(cw, 2, axis=0)
    sadv = o.normalize_scalarize(adv, tw, 4, 12)
    rows = np.arange(48, dtype=np.int32)
    cl = np.repeat(np.arange(2), 2).astype(np.int32)
    la, _ = o.actor_loss(a, af, 4, 12, b["obs"], b["action_pre"], b["logprob"], tw, cl, rows, sadv,
                         0.2, 0.0)
    assert abs(la - (-sadv.mean())) < 1e-12


def test_hypernet_zero_M_collapses_to_b(o):  # test_hypernet.cpp:32-44
    cfg = TrainCfg(F=4, feat_hidden=[4], actor_hidden=[5], critic_hidden=[5])
    a, _ = cfg.specs()
    flat = o.init_hypernet(a, 9)
    flat[a.n_feature:a.n_feature + a.P * a.F] = 0.0
    b = flat[a.n_feature + a.P * a.F:]
    for w in ([0.5, 0.5], [1.0, 0.0], [0.1, 0.9]):
        assert np.array_equal(o.hypernet_forward(a, flat, w), b)


def test_hypernet_rejects_off_simplex_weights(o):  # test_hypernet.cpp:321-330
    cfg = TrainCfg(F=4, feat_hidden=[4], actor_hidden=[5], critic_hidden=[5])
    a, _ = cfg.specs()
    flat = o.init_hypernet(a, 9)
    with pytest.raises(Exception):
        o.hypernet_forward(a, flat, [0.6, 0.6])
