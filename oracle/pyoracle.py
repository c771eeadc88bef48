"""TEST INFRASTRUCTURE ONLY: ctypes bindings over oracle/liboracle.so (the C
restatement, prefix ``mo_``) and oracle/_ref/libmorlax_ref.so (the compiled
reference + shim, prefix ``mref_``). Both expose the same flat signatures, so
``Oracle(lib="oracle")`` and ``Oracle(lib="ref")`` are interchangeable.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` leg may import this module.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libmorlax_ref.so")
REF_SRC = "/root/reference/proj"

ENV_KINDS = {"mo-lqr1d": 0, "mo-lqr1d-m1": 1, "mo-pointmass": 2, "mo-dst-continuous": 3,
             "mo-humanoid6": 4}
ENV_SPECS = {  # kind -> (obs_dim, act_dim, m, max_steps)
    0: (1, 1, 2, 200), 1: (1, 1, 1, 200), 2: (4, 2, 2, 200), 3: (1, 1, 2, 50), 4: (45, 12, 6, 1000)}

MAXL = 8


class MlpSpecC(C.Structure):
    _fields_ = [("n_sizes", C.c_int), ("sizes", C.c_int * (MAXL + 1)), ("out_tanh", C.c_int)]


class HSpecC(C.Structure):
    _fields_ = [("m", C.c_int), ("F", C.c_int), ("n_feat_hidden", C.c_int),
                ("feat_hidden", C.c_int * MAXL), ("target", MlpSpecC), ("has_log_std", C.c_int)]


class BatchC(C.Structure):
    _fields_ = [(n, C.POINTER(C.c_double)) for n in
                ("obs", "action_pre", "logprob", "reward", "value", "next_value")] + \
               [("term", C.POINTER(C.c_uint8)), ("trunc", C.POINTER(C.c_uint8))]


class TrainCfgC(C.Structure):
    _fields_ = [("env_kind", C.c_int), ("N", C.c_int), ("K", C.c_int), ("kappa", C.c_int),
                ("T", C.c_int), ("epochs", C.c_int), ("minibatch_count", C.c_int),
                ("gamma", C.c_double), ("lambda_", C.c_double), ("clip_eps", C.c_double),
                ("actor_lr", C.c_double), ("critic_lr", C.c_double), ("entropy_coef", C.c_double),
                ("seed", C.c_uint64), ("F", C.c_int),
                ("n_feat_hidden", C.c_int), ("feat_hidden", C.c_int * MAXL),
                ("n_actor_hidden", C.c_int), ("actor_hidden", C.c_int * MAXL),
                ("n_critic_hidden", C.c_int), ("critic_hidden", C.c_int * MAXL)]


@dataclass
class HSpec:
    m: int
    F: int
    feat_hidden: list
    target_sizes: list
    out_tanh: bool
    has_log_std: bool

    def c(self) -> HSpecC:
        h = HSpecC()
        h.m, h.F = self.m, self.F
        h.n_feat_hidden = len(self.feat_hidden)
        for i, v in enumerate(self.feat_hidden):
            h.feat_hidden[i] = v
        h.target.n_sizes = len(self.target_sizes)
        for i, v in enumerate(self.target_sizes):
            h.target.sizes[i] = v
        h.target.out_tanh = int(self.out_tanh)
        h.has_log_std = int(self.has_log_std)
        return h

    @property
    def feature_sizes(self):
        return [self.m] + list(self.feat_hidden) + [self.F]

    @staticmethod
    def mlp_count(sizes):
        return sum((sizes[i] + 1) * sizes[i + 1] for i in range(len(sizes) - 1))

    @property
    def n_feature(self):
        return self.mlp_count(self.feature_sizes)

    @property
    def mlp_n(self):
        return self.mlp_count(self.target_sizes)

    @property
    def P(self):
        return self.mlp_n + (self.target_sizes[-1] if self.has_log_std else 0)

    @property
    def n_params(self):
        return self.n_feature + self.P * self.F + self.P


def actor_spec(env_kind, F, feat_hidden, actor_hidden):
    od, ad, m, _ = ENV_SPECS[env_kind]
    return HSpec(m, F, list(feat_hidden), [od] + list(actor_hidden) + [ad], True, True)


def critic_spec(env_kind, F, feat_hidden, critic_hidden):
    od, ad, m, _ = ENV_SPECS[env_kind]
    return HSpec(m, F, list(feat_hidden), [od] + list(critic_hidden) + [m], False, False)


@dataclass
class TrainCfg:
    env: str = "mo-pointmass"
    N: int = 256
    K: int = 16
    kappa: int = 0
    T: int = 32
    epochs: int = 4
    minibatch_count: int = 4
    gamma: float = 0.99
    lam: float = 0.95
    clip_eps: float = 0.2
    actor_lr: float = 3e-4
    critic_lr: float = 3e-4
    entropy_coef: float = 0.1
    seed: int = 0
    F: int = 64
    feat_hidden: list = field(default_factory=lambda: [64])
    actor_hidden: list = field(default_factory=lambda: [64, 64])
    critic_hidden: list = field(default_factory=lambda: [64, 64])

    def c(self) -> TrainCfgC:
        t = TrainCfgC()
        t.env_kind = ENV_KINDS[self.env]
        for k in ("N", "K", "kappa", "T", "epochs", "minibatch_count", "clip_eps", "actor_lr",
                  "critic_lr", "entropy_coef", "seed", "F", "gamma"):
            setattr(t, k, getattr(self, k))
        t.lambda_ = self.lam
        for name in ("feat_hidden", "actor_hidden", "critic_hidden"):
            v = getattr(self, name)
            setattr(t, "n_" + name, len(v))
            arr = getattr(t, name)
            for i, x in enumerate(v):
                arr[i] = x
        return t

    @property
    def kind(self):
        return ENV_KINDS[self.env]

    def specs(self):
        return (actor_spec(self.kind, self.F, self.feat_hidden, self.actor_hidden),
                critic_spec(self.kind, self.F, self.feat_hidden, self.critic_hidden))


def _p(a, t=C.c_double):
    return a.ctypes.data_as(C.POINTER(t)) if a is not None else None


def build(quiet=True):
    """Build liboracle.so (always possible) and the reference shim (only when
    the reference sources are present, i.e. in the build container)."""
    targets = ["liboracle.so"]
    if os.path.isdir(REF_SRC):
        targets.append("ref")
    subprocess.run(["make", "-C", HERE, "-j8"] + targets, check=True,
                   stdout=subprocess.DEVNULL if quiet else None)


class OracleError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"[{code}] {msg}")
        self.code = code


class Oracle:
    """Same API over the C restatement (lib='oracle') or the compiled reference (lib='ref')."""

    def __init__(self, lib="oracle"):
        self.kind = lib
        path = ORACLE_SO if lib == "oracle" else REF_SO
        if not os.path.exists(path):
            build()
        self.lib = C.CDLL(path)
        self.pre = "mo_" if lib == "oracle" else "mref_"
        L = self.lib
        f = self.fn
        f("last_error").restype = C.c_char_p
        f("rng_split_key").restype = C.c_uint64
        f("rng_split_key").argtypes = [C.c_uint64, C.c_uint64]
        f("env_create").restype = C.c_void_p
        f("env_create").argtypes = [C.c_int, C.c_int]
        f("env_destroy").argtypes = [C.c_void_p]
        f("env_clamp_count").restype = C.c_uint64
        f("env_clamp_count").argtypes = [C.c_void_p]
        for n in ("rng_words", "rng_gaussians"):
            f(n).argtypes = [C.c_uint64, C.c_uint64, C.c_int64, C.c_void_p]
        f("rng_shuffle").argtypes = [C.c_uint64, C.POINTER(C.c_uint64), C.c_void_p, C.c_int64]
        f("env_reset").argtypes = [C.c_void_p, C.c_uint64, C.c_uint64, C.c_void_p]
        f("env_step").argtypes = [C.c_void_p] + [C.c_void_p] * 5
        f("env_current_obs").argtypes = [C.c_void_p, C.c_void_p]
        if lib == "oracle":
            L.mo_trainer_create.restype = C.c_void_p
            for n in ("mo_trainer_actor_params", "mo_trainer_critic_params", "mo_trainer_sadv",
                      "mo_trainer_advantages", "mo_trainer_targets", "mo_trainer_clusters",
                      "mo_trainer_tracker"):
                getattr(L, n).restype = C.POINTER(C.c_double)
                getattr(L, n).argtypes = [C.c_void_p]
            L.mo_trainer_perm.restype = C.POINTER(C.c_int32)
            L.mo_trainer_perm.argtypes = [C.c_void_p]
            L.mo_trainer_batch.restype = C.POINTER(BatchC)
            L.mo_trainer_batch.argtypes = [C.c_void_p]
            L.mo_trainer_env.restype = C.c_void_p
            L.mo_trainer_env.argtypes = [C.c_void_p]
            L.mo_trainer_iteration.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_void_p, C.c_void_p]
            L.mo_trainer_destroy.argtypes = [C.c_void_p]
            L.mo_env_get_streams.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
            L.mo_env_set_instances.argtypes = [C.c_void_p] * 5
            L.mo_hypervolume_wfg.argtypes = [C.c_int, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p]
        else:
            L.mref_trainer_create.restype = C.c_void_p
            L.mref_trainer_create.argtypes = [C.c_void_p, C.c_int]
            L.mref_trainer_destroy.argtypes = [C.c_void_p]
            L.mref_trainer_iteration.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_void_p,
                                                 C.c_void_p, C.c_void_p]
            L.mref_trainer_params.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p]
            L.mref_trainer_perm.argtypes = [C.c_void_p, C.c_void_p]
            L.mref_dirichlet.argtypes = [C.c_uint64, C.c_uint64, C.c_int, C.c_int, C.c_void_p]
        f("hypervolume_mc").argtypes = [C.c_int, C.c_int, C.c_void_p, C.c_void_p, C.c_uint64,
                                        C.c_uint64, C.c_uint64, C.c_void_p, C.c_void_p] + \
            ([C.c_void_p] if lib == "oracle" else [])
        f("hypervolume_detailed").argtypes = [C.c_int, C.c_int, C.c_void_p, C.c_void_p, C.c_uint64,
                                              C.c_uint64, C.c_void_p, C.c_void_p, C.c_void_p,
                                              C.c_void_p]
        f("adam").argtypes = [C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                              C.POINTER(C.c_int64), C.c_double]
        f("gae").argtypes = [C.c_int, C.c_int, C.c_int] + [C.c_void_p] * 5 + \
            [C.c_double, C.c_double, C.c_void_p, C.c_void_p]
        f("actor_loss").argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_int] + [C.c_void_p] * 6 + \
            [C.c_int, C.c_void_p, C.c_double, C.c_double, C.c_void_p, C.c_void_p]
        f("critic_loss").argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_int] + [C.c_void_p] * 4 + \
            [C.c_int, C.c_void_p, C.c_void_p, C.c_void_p]
        args = [C.c_void_p] * 5 + [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_uint64, C.c_uint64,
                                   C.c_void_p, C.c_void_p if lib == "oracle" else C.c_int]
        f("collect_rollouts").argtypes = args

    def fn(self, name):
        return getattr(self.lib, self.pre + name)

    def check(self, rc):
        if rc != 0:
            raise OracleError(rc, self.fn("last_error")().decode())

    # ---------------- rng ----------------
    def rng_seed_state(self, seed):
        k, c = C.c_uint64(), C.c_uint64()
        self.fn("rng_seed_state")(C.c_uint64(seed), C.byref(k), C.byref(c))
        return k.value, c.value

    def split_key(self, key, lane):
        return self.fn("rng_split_key")(key, lane)

    def rng_words(self, key, ctr, n):
        out = np.zeros(n, np.uint64)
        self.fn("rng_words")(key, ctr, n, out.ctypes.data)
        return out

    def rng_gaussians(self, key, ctr, n):
        out = np.zeros(n, np.float64)
        self.fn("rng_gaussians")(key, ctr, n, out.ctypes.data)
        return out

    def shuffle(self, key, ctr, v):
        v = np.ascontiguousarray(v, np.int32).copy()
        c = C.c_uint64(ctr)
        self.fn("rng_shuffle")(key, C.byref(c), v.ctypes.data, len(v))
        return v, c.value

    # ---------------- hypernet ----------------
    def init_hypernet(self, spec: HSpec, key, ctr=0):
        out = np.zeros(spec.n_params, np.float64)
        h = spec.c()
        self.check(self.fn("init_hypernet")(C.byref(h), C.c_uint64(key), C.c_uint64(ctr), _p(out)))
        return out

    def hypernet_forward(self, spec, flat, w):
        out = np.zeros(spec.P, np.float64)
        h = spec.c()
        w = np.ascontiguousarray(w, np.float64)
        flat = np.ascontiguousarray(flat, np.float64)
        self.check(self.fn("hypernet_forward")(C.byref(h), _p(flat), _p(w), _p(out)))
        return out

    def hypernet_backward(self, spec, flat, w, gtheta):
        out = np.zeros(spec.n_params, np.float64)
        h = spec.c()
        w = np.ascontiguousarray(w, np.float64)
        flat = np.ascontiguousarray(flat, np.float64)
        gtheta = np.ascontiguousarray(gtheta, np.float64)
        self.check(self.fn("hypernet_backward")(C.byref(h), _p(flat), _p(w), _p(gtheta), _p(out)))
        return out

    # ---------------- env ----------------
    def env(self, name, n):
        return OracleEnv(self, ENV_KINDS[name], n)

    # ---------------- rollout ----------------
    def collect_rollouts(self, aspec, aflat, cspec, cflat, env, cluster_w, reps, T, key, ctr,
                         tracker=None, threads=1):
        K = len(cluster_w)
        N = K * reps
        od, ad, m, _ = ENV_SPECS[env.kind]
        R = N * T
        out = {"obs": np.zeros((R, od)), "action_pre": np.zeros((R, ad)), "logprob": np.zeros(R),
               "reward": np.zeros((R, m)), "value": np.zeros((R, m)), "next_value": np.zeros((R, m)),
               "term": np.zeros(R, np.uint8), "trunc": np.zeros(R, np.uint8)}
        b = BatchC(*[_p(out[k]) for k in ("obs", "action_pre", "logprob", "reward", "value",
                                           "next_value")],
                   _p(out["term"], C.c_uint8), _p(out["trunc"], C.c_uint8))
        a, c = aspec.c(), cspec.c()
        cw = np.ascontiguousarray(cluster_w, np.float64)
        last = (tracker.ctypes.data if tracker is not None else None) if self.kind == "oracle" \
            else threads
        self.check(self.fn("collect_rollouts")(C.byref(a), aflat.ctypes.data, C.byref(c),
                                               cflat.ctypes.data, env.h, cw.ctypes.data, K, reps, T,
                                               key, ctr, C.byref(b), last))
        return out

    # ---------------- gae ----------------
    def gae(self, reward, value, next_value, term, trunc, N, T, gamma, lam):
        m = reward.shape[-1]
        adv = np.zeros((N * T, m))
        tg = np.zeros((N * T, m))
        arrs = [np.ascontiguousarray(x, np.float64) for x in (reward, value, next_value)]
        fl = [np.ascontiguousarray(x, np.uint8) for x in (term, trunc)]
        self.check(self.fn("gae")(N, T, m, *[a.ctypes.data for a in arrs],
                                  *[f.ctypes.data for f in fl], gamma, lam, adv.ctypes.data,
                                  tg.ctypes.data))
        return adv, tg

    def normalize_scalarize(self, adv, tradeoffs, N, T):
        m = adv.shape[-1]
        out = np.zeros(N * T)
        adv = np.ascontiguousarray(adv, np.float64)
        tw = np.ascontiguousarray(tradeoffs, np.float64)
        self.check(self.fn("normalize_scalarize")(N, T, m, _p(adv), _p(tw), _p(out)))
        return out

    # ---------------- losses ----------------
    def actor_loss(self, spec, flat, N, T, obs, action_pre, logprob_old, tradeoffs, cluster, rows,
                   sadv, clip, ent):
        g = np.zeros(spec.n_params)
        loss = C.c_double()
        h = spec.c()
        arrs = [np.ascontiguousarray(x, np.float64) for x in (flat, obs, action_pre, logprob_old,
                                                              tradeoffs)]
        cl = np.ascontiguousarray(cluster, np.int32)
        rw = np.ascontiguousarray(rows, np.int32)
        sa = np.ascontiguousarray(sadv, np.float64)
        self.check(self.fn("actor_loss")(C.byref(h), arrs[0].ctypes.data, N, T,
                                         arrs[1].ctypes.data, arrs[2].ctypes.data,
                                         arrs[3].ctypes.data, arrs[4].ctypes.data, cl.ctypes.data,
                                         rw.ctypes.data, len(rw), sa.ctypes.data, clip, ent,
                                         C.byref(loss), g.ctypes.data))
        return loss.value, g

    def critic_loss(self, spec, flat, N, T, obs, tradeoffs, cluster, rows, targets):
        g = np.zeros(spec.n_params)
        loss = C.c_double()
        h = spec.c()
        arrs = [np.ascontiguousarray(x, np.float64) for x in (flat, obs, tradeoffs, targets)]
        cl = np.ascontiguousarray(cluster, np.int32)
        rw = np.ascontiguousarray(rows, np.int32)
        self.check(self.fn("critic_loss")(C.byref(h), arrs[0].ctypes.data, N, T,
                                          arrs[1].ctypes.data, arrs[2].ctypes.data,
                                          cl.ctypes.data, rw.ctypes.data, len(rw),
                                          arrs[3].ctypes.data, C.byref(loss), g.ctypes.data))
        return loss.value, g

    def adam(self, p, g, m1, m2, step, lr):
        p, m1, m2 = (np.ascontiguousarray(x, np.float64).copy() for x in (p, m1, m2))
        g = np.ascontiguousarray(g, np.float64)
        st = C.c_int64(step)
        self.check(self.fn("adam")(len(p), p.ctypes.data, g.ctypes.data, m1.ctypes.data,
                                   m2.ctypes.data, C.byref(st), lr))
        return p, m1, m2, st.value

    # ---------------- pareto ----------------
    def nondominated_mask(self, pts):
        pts = np.ascontiguousarray(pts, np.float64)
        n, m = pts.shape
        mask = np.zeros(n, np.uint8)
        self.check(self.fn("nondominated_mask")(n, m, _p(pts), _p(mask, C.c_uint8)))
        return mask

    def evaluate_params(self, spec, flat, env_kind, res, episodes, key):
        m = spec.m
        f = self.fn("simplex_grid_size")
        f.restype = C.c_int64
        n = 1 if m == 1 else int(f(m, res))
        W = np.zeros((n, m))
        R = np.zeros((n, m))
        npts = C.c_int64()
        flat = np.ascontiguousarray(flat, np.float64)
        self.check(self.fn("evaluate_params")(C.byref(spec.c()), _p(flat), env_kind, res, episodes,
                                              C.c_uint64(key), _p(W), _p(R), C.byref(npts)))
        return W[:npts.value], R[:npts.value]

    def checkpoint_resave(self, src, dst, n_actor, n_critic):
        """The reference's load_checkpoint(src) + save_checkpoint(dst) (ref lib only)."""
        a, c = np.zeros(n_actor), np.zeros(n_critic)
        it = C.c_int64()
        self.check(self.lib.mref_checkpoint_resave(src.encode(), dst.encode(), _p(a), C.c_int64(n_actor), _p(c),
                                                   C.c_int64(n_critic), C.byref(it)))
        return a, c, it.value

    def train_run(self, cfg, iterations, grid, episodes, log_interval, out_dir, n_actor, n_critic):
        """The reference train() with out_dir, evaluation and the archive
        (train.cpp:55-229; ref lib only): per-iteration archive HV, final params."""
        hv, a, c = np.zeros(iterations), np.zeros(n_actor), np.zeros(n_critic)
        self.check(self.lib.mref_train_run(C.byref(cfg.c()), iterations, grid, episodes, log_interval,
                                           out_dir.encode(), _p(hv), _p(a), _p(c)))
        return hv, a, c

    def linear_dominance_mask(self, pts):
        pts = np.ascontiguousarray(pts, np.float64)
        n, m = pts.shape
        mask = np.zeros(n, np.uint8)
        self.check(self.fn("linear_dominance_mask")(n, m, _p(pts), _p(mask, C.c_uint8)))
        return mask

    def hypervolume_detailed(self, pts, ref, samples=1_000_000, seed=0x9E3779B9):
        pts = np.ascontiguousarray(pts, np.float64).reshape(-1, len(ref))
        ref = np.ascontiguousarray(ref, np.float64)
        v, se = C.c_double(), C.c_double()
        ex, cl = C.c_int(), C.c_int()
        self.check(self.fn("hypervolume_detailed")(len(pts), len(ref), pts.ctypes.data,
                                                   ref.ctypes.data, samples, seed, C.byref(v),
                                                   C.byref(se), C.byref(ex), C.byref(cl)))
        return v.value, se.value, bool(ex.value), cl.value

    def hypervolume_mc(self, pts, ref, samples, key, ctr):
        pts = np.ascontiguousarray(pts, np.float64).reshape(-1, len(ref))
        ref = np.ascontiguousarray(ref, np.float64)
        v, se = C.c_double(), C.c_double()
        extra = []
        hits = C.c_uint64()
        if self.kind == "oracle":
            extra = [C.byref(hits)]
        self.check(self.fn("hypervolume_mc")(len(pts), len(ref), pts.ctypes.data, ref.ctypes.data,
                                             samples, key, ctr, C.byref(v), C.byref(se), *extra))
        return v.value, se.value, hits.value

    def hypervolume_wfg(self, pts, ref):
        pts = np.ascontiguousarray(pts, np.float64).reshape(-1, len(ref))
        ref = np.ascontiguousarray(ref, np.float64)
        v = C.c_double()
        self.lib.mo_hypervolume_wfg(len(pts), len(ref), pts.ctypes.data, ref.ctypes.data,
                                    C.byref(v))
        return v.value


class OracleEnv:
    def __init__(self, o: Oracle, kind, n):
        self.o, self.kind, self.n = o, kind, n
        self.h = o.fn("env_create")(kind, n)
        if not self.h:
            raise OracleError(2, o.fn("last_error")().decode())
        self.obs_dim, self.act_dim, self.m, self.max_steps = ENV_SPECS[kind]

    def __del__(self):
        try:
            self.o.fn("env_destroy")(self.h)
        except Exception:
            pass

    def reset(self, key, ctr=0):
        out = np.zeros((self.n, self.obs_dim))
        self.o.check(self.o.fn("env_reset")(self.h, C.c_uint64(key), C.c_uint64(ctr),
                                            out.ctypes.data))
        return out

    def step(self, actions):
        a = np.ascontiguousarray(actions, np.float64).reshape(self.n, self.act_dim)
        obs = np.zeros((self.n, self.obs_dim))
        rew = np.zeros((self.n, self.m))
        term = np.zeros(self.n, np.uint8)
        trunc = np.zeros(self.n, np.uint8)
        self.o.check(self.o.fn("env_step")(self.h, a.ctypes.data, obs.ctypes.data, rew.ctypes.data,
                                           term.ctypes.data, trunc.ctypes.data))
        return obs, rew, term, trunc

    def current_obs(self):
        out = np.zeros((self.n, self.obs_dim))
        self.o.fn("env_current_obs")(self.h, out.ctypes.data)
        return out

    def clamp_count(self):
        return self.o.fn("env_clamp_count")(self.h)

    def streams(self):
        assert self.o.kind == "oracle"
        keys = np.zeros(self.n, np.uint64)
        ctrs = np.zeros(self.n, np.uint64)
        steps = np.zeros(self.n, np.int32)
        self.o.lib.mo_env_get_streams(self.h, keys.ctypes.data, ctrs.ctypes.data, steps.ctypes.data)
        return keys, ctrs, steps

    def set_instances(self, state=None, steps=None, keys=None, ctrs=None):
        """Teacher-forcing test hook: restart every instance from the given
        state (obs == state) / step counter / stream position."""
        assert self.o.kind == "oracle"
        arrs = []
        for v, dt in ((state, np.float64), (steps, np.int32), (keys, np.uint64), (ctrs, np.uint64)):
            arrs.append(None if v is None else np.ascontiguousarray(v, dt))
        self.o.lib.mo_env_set_instances(self.h, *[None if a is None else a.ctypes.data for a in arrs])


class OracleTrainer:
    """The C restatement of train()'s loop body (oracle only)."""

    def __init__(self, o: Oracle, cfg: TrainCfg):
        assert o.kind == "oracle"
        self.o, self.cfg = o, cfg
        self._c = cfg.c()
        self.h = o.lib.mo_trainer_create(C.byref(self._c))
        if not self.h:
            raise OracleError(2, o.lib.mo_last_error().decode())
        self.aspec, self.cspec = cfg.specs()
        self.od, self.ad, self.m, _ = ENV_SPECS[cfg.kind]

    def __del__(self):
        try:
            self.o.lib.mo_trainer_destroy(self.h)
        except Exception:
            pass

    def iteration(self, it, max_minibatches=-1):
        a, c = C.c_double(), C.c_double()
        self.o.check(self.o.lib.mo_trainer_iteration(self.h, it, max_minibatches, C.byref(a),
                                                     C.byref(c)))
        return a.value, c.value

    def _arr(self, ptr, n, dtype=np.float64):
        return np.ctypeslib.as_array(ptr, shape=(n,)).astype(dtype, copy=True)

    def actor_params(self):
        return self._arr(self.o.lib.mo_trainer_actor_params(self.h), self.aspec.n_params)

    def critic_params(self):
        return self._arr(self.o.lib.mo_trainer_critic_params(self.h), self.cspec.n_params)

    def perm(self):
        return self._arr(self.o.lib.mo_trainer_perm(self.h), self.cfg.N * self.cfg.T, np.int32)

    def clusters(self):
        return self._arr(self.o.lib.mo_trainer_clusters(self.h), self.cfg.K * self.m).reshape(
            self.cfg.K, self.m)

    def tracker(self):
        return self._arr(self.o.lib.mo_trainer_tracker(self.h), self.cfg.N * self.m)

    def batch(self):
        b = self.o.lib.mo_trainer_batch(self.h).contents
        R = self.cfg.N * self.cfg.T
        m, od, ad = self.m, self.od, self.ad
        return {"obs": self._arr(b.obs, R * od).reshape(R, od),
                "action_pre": self._arr(b.action_pre, R * ad).reshape(R, ad),
                "logprob": self._arr(b.logprob, R),
                "reward": self._arr(b.reward, R * m).reshape(R, m),
                "value": self._arr(b.value, R * m).reshape(R, m),
                "next_value": self._arr(b.next_value, R * m).reshape(R, m),
                "term": self._arr(b.term, R, np.uint8), "trunc": self._arr(b.trunc, R, np.uint8),
                "adv": self._arr(self.o.lib.mo_trainer_advantages(self.h), R * m).reshape(R, m),
                "targets": self._arr(self.o.lib.mo_trainer_targets(self.h), R * m).reshape(R, m),
                "sadv": self._arr(self.o.lib.mo_trainer_sadv(self.h), R)}

    def env_state(self):
        e = OracleEnv.__new__(OracleEnv)
        e.o, e.kind, e.n = self.o, self.cfg.kind, self.cfg.N
        e.h = self.o.lib.mo_trainer_env(self.h)
        e.obs_dim, e.act_dim, e.m, e.max_steps = ENV_SPECS[self.cfg.kind]
        keys, ctrs, steps = OracleEnv.streams(e)
        return e.current_obs(), keys, ctrs, steps


class RefTrainer:
    """The compiled reference's train() loop body (ref shim), for the CPU baseline."""

    def __init__(self, o: Oracle, cfg: TrainCfg, threads=1):
        assert o.kind == "ref"
        self.o, self.cfg = o, cfg
        self._c = cfg.c()
        self.h = o.lib.mref_trainer_create(C.byref(self._c), threads)
        if not self.h:
            raise OracleError(2, o.lib.mref_last_error().decode())
        self.aspec, self.cspec = cfg.specs()

    def __del__(self):
        try:
            self.o.lib.mref_trainer_destroy(self.h)
        except Exception:
            pass

    def iteration(self, it, max_minibatches=-1):
        secs = np.zeros(6)
        a, c = C.c_double(), C.c_double()
        self.o.check(self.o.lib.mref_trainer_iteration(self.h, it, max_minibatches, 0,
                                                       secs.ctypes.data, C.byref(a), C.byref(c)))
        return secs, a.value, c.value

    def params(self):
        a = np.zeros(self.aspec.n_params)
        c = np.zeros(self.cspec.n_params)
        self.o.lib.mref_trainer_params(self.h, a.ctypes.data, c.ctypes.data)
        return a, c

    def perm(self):
        p = np.zeros(self.cfg.N * self.cfg.T, np.int32)
        self.o.lib.mref_trainer_perm(self.h, p.ctypes.data)
        return p
