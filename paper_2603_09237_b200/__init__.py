"""B200-native MORLAX data-parallel training step.

Python mirror of the reference C++ API (``/root/reference/proj/include/morlax``)
over the C-ABI in ``include/morlax_b200.h`` (``libmorlax_b200.so``: sm_100a
CUDA kernels + C++ host orchestration). Names, argument meaning and error
behaviour follow the reference:

* ``BatchedEnv`` / ``make_env`` / ``env_spec``      -> env.hpp:37-99, registry.cpp
* ``hypernet_forward`` / ``hypernet_backward`` / ``init_hypernet`` -> hypernet.hpp
* ``gae_per_objective`` / ``normalize_and_scalarize`` -> trainer.hpp:154-161
* ``adam_apply``                                     -> trainer.hpp:211-212
* ``Trainer`` (``train()`` loop body)                -> train.cpp:118-184
* ``nondominated_filter`` / ``hypervolume_mc`` / ``hypervolume_detailed`` -> pareto.hpp

There is no CPU fallback: importing this package loads the CUDA library
(building it with nvcc if the in-tree .so is missing) and every compute call
runs on the GPU; without a GPU, calls fail with ``CudaError``.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from ._lib import LIB, LIB_PATH  # noqa: F401  (loads / builds the CUDA library)

__all__ = [
    "ConfigError", "ShapeError", "NumericError", "DomainError", "CudaError", "EnvSpec", "env_spec",
    "BatchedEnv", "make_env", "HypernetSpec", "PolicyForward", "evaluate_params", "simplex_grid_size", "init_hypernet", "hypernet_forward", "hypernet_backward",
    "gae_per_objective", "normalize_and_scalarize", "adam_apply", "TrainConfig", "Trainer",
    "nondominated_mask", "nondominated_filter", "linear_dominance_mask", "linear_dominance_filter", "hypervolume_mc", "hypervolume_detailed", "hypervolume_exact",
    "rng_words", "rng_gaussians", "shard_minibatch", "LIB_PATH",
]


# ---------------------------------------------------------------- errors (errors.hpp:10-30)
class MorlaxError(RuntimeError):
    code = 1


class ConfigError(MorlaxError):
    code = 2


class ShapeError(MorlaxError):
    code = 2


class DomainError(MorlaxError):
    code = 2


class NumericError(MorlaxError):
    code = 3


class CudaError(MorlaxError):
    code = 1


_KINDS = {"ConfigError": ConfigError, "ShapeError": ShapeError, "DomainError": DomainError,
          "NumericError": NumericError, "CudaError": CudaError}


def _check(rc):
    if rc != 0:
        kind = LIB.morlax_last_error_kind().decode()
        msg = LIB.morlax_last_error().decode()
        raise _KINDS.get(kind, MorlaxError)(msg)


def _ptr(a):
    return C.c_void_p(a.ctypes.data) if a is not None else None


def _f32(a, shape=None):
    a = np.ascontiguousarray(a, dtype=np.float32)
    return a if shape is None else a.reshape(shape)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


# ---------------------------------------------------------------- RNG (rng.hpp)
def rng_words(key: int, ctr: int, n: int) -> np.ndarray:
    out = np.zeros(n, np.uint64)
    _check(LIB.morlax_rng_words(C.c_uint64(key), C.c_uint64(ctr), n, _ptr(out)))
    return out


def rng_gaussians(key: int, ctr: int, n: int) -> np.ndarray:
    out = np.zeros(n, np.float64)
    _check(LIB.morlax_rng_gaussians(C.c_uint64(key), C.c_uint64(ctr), n, _ptr(out)))
    return out


# ---------------------------------------------------------------- env (env.hpp)
@dataclass
class EnvSpec:
    name: str
    obs_dim: int
    act_dim: int
    m: int
    max_episode_steps: int


def env_spec(name: str) -> EnvSpec:
    v = [C.c_int() for _ in range(4)]
    _check(LIB.morlax_env_spec(name.encode(), *[C.byref(x) for x in v]))
    return EnvSpec(name, *[x.value for x in v])


@dataclass
class StepOut:
    obs: np.ndarray
    reward: np.ndarray
    terminated: np.ndarray
    truncated: np.ndarray


class BatchedEnv:
    """N instances of one environment stepped in lockstep on the GPU, with
    per-instance counter-based RNG streams and auto-reset (env.hpp:26-99)."""

    def __init__(self, name: str, num_envs: int):
        self.spec = env_spec(name)
        self.num_envs = num_envs
        h = C.c_void_p()
        _check(LIB.morlax_env_create(name.encode(), num_envs, C.byref(h)))
        self._h = h

    def __del__(self):
        if getattr(self, "_h", None):
            LIB.morlax_env_destroy(self._h)
            self._h = None

    def reset(self, key: int, ctr: int = 0) -> np.ndarray:
        obs = np.zeros((self.num_envs, self.spec.obs_dim), np.float32)
        _check(LIB.morlax_env_reset(self._h, C.c_uint64(key), C.c_uint64(ctr), _ptr(obs)))
        return obs

    def step(self, actions) -> StepOut:
        s = self.spec
        a = _f32(actions)
        if a.size != self.num_envs * s.act_dim:
            raise ShapeError("BatchedEnv::step: actions must be N x act_dim")
        out = StepOut(np.zeros((self.num_envs, s.obs_dim), np.float32),
                      np.zeros((self.num_envs, s.m), np.float32),
                      np.zeros(self.num_envs, np.uint8), np.zeros(self.num_envs, np.uint8))
        _check(LIB.morlax_env_step(self._h, _ptr(a), _ptr(out.obs), _ptr(out.reward),
                                   _ptr(out.terminated), _ptr(out.truncated)))
        return out

    def step_device(self, d_actions, d_obs, d_reward, d_term, d_trunc, stream=0):
        """Device-pointer variant (e.g. torch tensors' data_ptr())."""
        _check(LIB.morlax_env_step_device(self._h, C.c_void_p(d_actions), C.c_void_p(d_obs),
                                          C.c_void_p(d_reward), C.c_void_p(d_term),
                                          C.c_void_p(d_trunc), C.c_void_p(stream)))

    def current_obs(self) -> np.ndarray:
        obs = np.zeros((self.num_envs, self.spec.obs_dim), np.float32)
        _check(LIB.morlax_env_current_obs(self._h, _ptr(obs)))
        return obs

    def clamp_count(self) -> int:
        return int(LIB.morlax_env_clamp_count(self._h))


def make_env(name: str, num_envs: int) -> BatchedEnv:
    return BatchedEnv(name, num_envs)


# ---------------------------------------------------------------- hypernet (hypernet.hpp)
class _HSpecC(C.Structure):
    _fields_ = [("m", C.c_int), ("F", C.c_int), ("n_feature_hidden", C.c_int),
                ("feature_hidden", C.c_int * 8), ("n_target_sizes", C.c_int),
                ("target_sizes", C.c_int * 9), ("target_tanh", C.c_int), ("has_log_std", C.c_int)]


@dataclass
class HypernetSpec:
    m: int
    F: int
    feature_hidden: list
    target_sizes: list  # [in, hidden..., out]
    target_tanh: bool
    has_log_std: bool

    def c(self):
        h = _HSpecC()
        h.m, h.F = self.m, self.F
        h.n_feature_hidden = len(self.feature_hidden)
        for i, v in enumerate(self.feature_hidden):
            h.feature_hidden[i] = v
        h.n_target_sizes = len(self.target_sizes)
        for i, v in enumerate(self.target_sizes):
            h.target_sizes[i] = v
        h.target_tanh = int(self.target_tanh)
        h.has_log_std = int(self.has_log_std)
        return h

    @property
    def target_param_count(self) -> int:
        return int(LIB.morlax_hypernet_target_count(C.byref(self.c())))

    @property
    def param_count(self) -> int:
        return int(LIB.morlax_hypernet_param_count(C.byref(self.c())))


def init_hypernet(spec: HypernetSpec, key: int, ctr: int = 0) -> np.ndarray:
    out = np.zeros(spec.param_count)
    _check(LIB.morlax_init_hypernet(C.byref(spec.c()), C.c_uint64(key), C.c_uint64(ctr), _ptr(out)))
    return out


def hypernet_forward(spec: HypernetSpec, flat, w) -> np.ndarray:
    w = _f64(w).reshape(-1, spec.m)
    out = np.zeros((len(w), spec.target_param_count))
    _check(LIB.morlax_hypernet_forward(C.byref(spec.c()), _ptr(_f64(flat)), _ptr(w), len(w),
                                       _ptr(out)))
    return out


class PolicyForward:
    """Per-preference-group policy forward (BASELINE config 2): G preference
    vectors, R observations each, through the weights the hypernetwork
    generates for each preference (policy_forward nn.cpp:162-190 over
    hypernet_forward hypernet.cpp:69-90). forward() returns the Gaussian mean
    before the tanh squash, [G*R][out]."""

    def __init__(self, spec: HypernetSpec, groups: int, rows_per_group: int):
        self.spec, self.G, self.R = spec, groups, rows_per_group
        h = C.c_void_p()
        _check(LIB.morlax_policy_create(C.byref(spec.c()), groups, rows_per_group, C.byref(h)))
        self._h = h

    def __del__(self):
        if getattr(self, "_h", None):
            LIB.morlax_policy_destroy(self._h)
            self._h = None

    def set_params(self, flat):
        f = _f64(flat)
        if f.size != self.spec.param_count:
            raise ShapeError("policy forward: flat parameter vector has the wrong length")
        _check(LIB.morlax_policy_set_params(self._h, _ptr(f)))

    def forward(self, w, obs) -> np.ndarray:
        w = _f64(w).reshape(self.G, self.spec.m)
        od, out = self.spec.target_sizes[0], self.spec.target_sizes[-1]
        o = np.ascontiguousarray(obs, np.float32).reshape(self.G * self.R, od)
        pre = np.zeros((self.G * self.R, out), np.float32)
        _check(LIB.morlax_policy_forward(self._h, _ptr(w), _ptr(o), _ptr(pre)))
        return pre

    def forward_device(self, w_ptr: int, obs_ptr: int, pre_ptr: int, stream: int = 0):
        _check(LIB.morlax_policy_forward_device(self._h, C.c_void_p(w_ptr), C.c_void_p(obs_ptr),
                                                C.c_void_p(pre_ptr), C.c_void_p(stream)))

    @property
    def flops(self) -> float:
        return float(LIB.morlax_policy_flops(self._h))


def simplex_grid_size(m: int, resolution: int) -> int:
    return int(LIB.morlax_simplex_grid_size(m, resolution))


def evaluate_params(spec: HypernetSpec, flat, env_name: str, grid_resolution: int, episodes_per_point: int,
                    key: int):
    """evaluate_params (evaluate.cpp:68-101) on the device: returns (W, mean_return),
    both [n_points][m], W in simplex_grid order; Rng(key).split(g) resets point g."""
    n = 1 if spec.m == 1 else simplex_grid_size(spec.m, grid_resolution)
    W = np.zeros((max(n, 1), spec.m))
    R = np.zeros((max(n, 1), spec.m))
    npts = C.c_int64()
    _check(LIB.morlax_evaluate_params(C.byref(spec.c()), _ptr(_f64(flat)), env_name.encode(), grid_resolution,
                                      episodes_per_point, C.c_uint64(key), _ptr(W), _ptr(R), C.byref(npts)))
    return W[:npts.value], R[:npts.value]


def hypernet_backward(spec: HypernetSpec, flat, w, gtheta) -> np.ndarray:
    w = _f64(w).reshape(-1, spec.m)
    g = _f64(gtheta).reshape(len(w), -1)
    out = np.zeros(spec.param_count)
    _check(LIB.morlax_hypernet_backward(C.byref(spec.c()), _ptr(_f64(flat)), _ptr(w), len(w),
                                        _ptr(g), _ptr(out)))
    return out


# ---------------------------------------------------------------- GAE (gae.cpp)
def gae_per_objective(reward, value, next_value, terminated, truncated, N, T, gamma, lam):
    m = np.asarray(reward).reshape(N * T, -1).shape[1]
    adv = np.zeros((N * T, m), np.float32)
    tgt = np.zeros((N * T, m), np.float32)
    r, v, nv = (_f32(x) for x in (reward, value, next_value))
    te = np.ascontiguousarray(terminated, np.uint8)
    tr = np.ascontiguousarray(truncated, np.uint8)
    _check(LIB.morlax_gae(N, T, m, _ptr(r), _ptr(v), _ptr(nv), _ptr(te), _ptr(tr), C.c_double(gamma),
                          C.c_double(lam), _ptr(adv), _ptr(tgt)))
    return adv, tgt


def normalize_and_scalarize(advantages, tradeoffs, N, T):
    a = _f32(advantages)
    m = a.reshape(N * T, -1).shape[1]
    out = np.zeros(N * T, np.float32)
    _check(LIB.morlax_normalize_scalarize(N, T, m, _ptr(a), _ptr(_f64(tradeoffs)), _ptr(out)))
    return out


def adam_apply(params, grad, m1, m2, step, lr):
    p, m1, m2 = (_f64(x).copy() for x in (params, m1, m2))
    st = C.c_int64(step)
    _check(LIB.morlax_adam(len(p), _ptr(p), _ptr(_f64(grad)), _ptr(m1), _ptr(m2), C.byref(st),
                           C.c_double(lr)))
    return p, m1, m2, st.value


# ---------------------------------------------------------------- trainer (train.cpp)
class _TrainCfgC(C.Structure):
    _fields_ = [("env_name", C.c_char_p), ("N", C.c_int), ("K", C.c_int), ("kappa", C.c_int),
                ("T", C.c_int), ("epochs", C.c_int), ("minibatch_count", C.c_int),
                ("gamma", C.c_double), ("gae_lambda", C.c_double), ("clip_eps", C.c_double),
                ("actor_lr", C.c_double), ("critic_lr", C.c_double), ("entropy_coef", C.c_double),
                ("seed", C.c_uint64), ("F", C.c_int), ("n_feature_hidden", C.c_int),
                ("feature_hidden", C.c_int * 8), ("n_actor_hidden", C.c_int),
                ("actor_hidden", C.c_int * 8), ("n_critic_hidden", C.c_int),
                ("critic_hidden", C.c_int * 8)]


class _IterStatsC(C.Structure):
    _fields_ = [("actor_loss", C.c_double), ("critic_loss", C.c_double), ("minibatches", C.c_int),
                ("numeric_error", C.c_int), ("kernel_launches", C.c_int64)]


@dataclass
class TrainConfig:
    """RunConfig subset of the hot path (trainer.hpp:21-77). Defaults = PR1."""
    env_name: str = "mo-pointmass"
    N: int = 256
    K: int = 16
    kappa: int = 0
    T: int = 32
    gamma: float = 0.99
    gae_lambda: float = 0.95
    clip_eps: float = 0.2
    epochs: int = 4
    minibatch_count: int = 4
    actor_lr: float = 3e-4
    critic_lr: float = 3e-4
    entropy_coef: float = 0.1
    seed: int = 0
    F: int = 64
    feature_hidden: list = field(default_factory=lambda: [64])
    actor_hidden: list = field(default_factory=lambda: [64, 64])
    critic_hidden: list = field(default_factory=lambda: [64, 64])

    def c(self):
        c = _TrainCfgC()
        self._name = self.env_name.encode()
        c.env_name = self._name
        for k in ("N", "K", "kappa", "T", "epochs", "minibatch_count", "gamma", "gae_lambda",
                  "clip_eps", "actor_lr", "critic_lr", "entropy_coef", "seed", "F"):
            setattr(c, k, getattr(self, k))
        for name in ("feature_hidden", "actor_hidden", "critic_hidden"):
            v = getattr(self, name)
            setattr(c, "n_" + name, len(v))
            arr = getattr(c, name)
            for i, x in enumerate(v):
                arr[i] = x
        return c

    def specs(self):
        es = env_spec(self.env_name)
        a = HypernetSpec(es.m, self.F, list(self.feature_hidden),
                         [es.obs_dim] + list(self.actor_hidden) + [es.act_dim], True, True)
        c = HypernetSpec(es.m, self.F, list(self.feature_hidden),
                         [es.obs_dim] + list(self.critic_hidden) + [es.m], False, False)
        return a, c


@dataclass
class IterationStats:
    actor_loss: float
    critic_loss: float
    minibatches: int
    numeric_error: int
    kernel_launches: int


def nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    _check(LIB.morlax_nccl_unique_id(buf))
    return buf.raw


class _CkExtraC(C.Structure):
    _fields_ = [("iterations", C.c_int), ("grid_resolution", C.c_int), ("episodes_per_point", C.c_int),
                ("log_interval", C.c_int), ("n_pareto_reference", C.c_int),
                ("pareto_reference", C.POINTER(C.c_double))]


class LoopbackGroup:
    """W ranks of the sharded data plane as host threads on ONE device
    (morlax_loopback_create): each rank's Trainer(cfg, W, r, loopback=group)
    must be driven from its own thread; results equal the single-rank
    trainer's bit for bit. For tests of the multi-GPU code path."""

    def __init__(self, world: int):
        self.world = world
        h = C.c_void_p()
        _check(LIB.morlax_loopback_create(world, C.byref(h)))
        self._h = h

    def __del__(self):
        if getattr(self, "_h", None):
            LIB.morlax_loopback_destroy(self._h)
            self._h = None


class Trainer:
    """The reference train() loop body on the GPU (train.cpp:118-184).
    world > 1: one Trainer per GPU/rank (environments and preference clusters
    sharded; NCCL exchange of the per-cluster hypernetwork gradients)."""

    _F32 = {"obs", "action_pre", "logprob", "reward", "value", "next_value", "advantages",
            "value_targets", "scalar_advantage", "env_state", "tracker", "clusters"}

    def __init__(self, cfg: TrainConfig, world: int = 1, rank: int = 0, nccl_id: bytes = None,
                 _handle=None, loopback: "LoopbackGroup" = None):
        self.cfg = cfg
        self._c = cfg.c()
        h = C.c_void_p()
        self._group = loopback  # keeps the group alive while this rank exists
        if _handle is not None:  # adopt a trainer made by morlax_train
            h = _handle
        elif loopback is not None:
            if world != loopback.world:
                raise ConfigError("world must equal the loopback group's size")
            _check(LIB.morlax_trainer_create_loopback(C.byref(self._c), loopback._h, rank, C.byref(h)))
        else:
            idb = C.create_string_buffer(nccl_id, 128) if nccl_id else None
            _check(LIB.morlax_trainer_create(C.byref(self._c), world, rank, idb, C.byref(h)))
        self._h = h
        self.es = env_spec(cfg.env_name)
        ap, cp = C.c_int64(), C.c_int64()
        le, lc, rows = C.c_int(), C.c_int(), C.c_int()
        _check(LIB.morlax_trainer_sizes(h, C.byref(ap), C.byref(cp), C.byref(le), C.byref(lc),
                                        C.byref(rows)))
        self.n_actor, self.n_critic = ap.value, cp.value
        self.local_envs, self.local_clusters, self.rows = le.value, lc.value, rows.value

    def __del__(self):
        if getattr(self, "_h", None):
            LIB.morlax_trainer_destroy(self._h)
            self._h = None

    def iteration(self, it: int) -> IterationStats:
        st = _IterStatsC()
        _check(LIB.morlax_trainer_iteration(self._h, it, C.byref(st)))
        return IterationStats(st.actor_loss, st.critic_loss, st.minibatches, st.numeric_error,
                              st.kernel_launches)

    def phase(self, it: int, phase: int, max_minibatches: int = -1):
        st = _IterStatsC()
        _check(LIB.morlax_trainer_phase(self._h, it, phase, max_minibatches, C.byref(st)))
        return IterationStats(st.actor_loss, st.critic_loss, st.minibatches, st.numeric_error,
                              st.kernel_launches)

    def params(self, which: str = "actor") -> np.ndarray:
        n = self.n_actor if which == "actor" else self.n_critic
        out = np.zeros(n)
        _check(LIB.morlax_trainer_get_params(self._h, 0 if which == "actor" else 1, _ptr(out)))
        return out

    def set_params(self, which: str, flat):
        _check(LIB.morlax_trainer_set_params(self._h, 0 if which == "actor" else 1,
                                             _ptr(_f64(flat))))

    def theta(self, which: str = "actor") -> np.ndarray:
        """Generated target-net weights of the local clusters (last hypernet
        forward), fp32 [local K][P] in the reference flat layout."""
        P = self.cfg.specs()[0 if which == "actor" else 1].target_param_count
        out = np.zeros((self.local_clusters, P), np.float32)
        _check(LIB.morlax_trainer_get_theta(self._h, 0 if which == "actor" else 1, _ptr(out)))
        return out

    def grad(self, which: str = "actor") -> np.ndarray:
        n = self.n_actor if which == "actor" else self.n_critic
        out = np.zeros(n)
        _check(LIB.morlax_trainer_get_grad(self._h, 0 if which == "actor" else 1, _ptr(out)))
        return out

    def _shape(self, name):
        es, R, N = self.es, self.rows, self.local_envs
        return {"obs": (R, es.obs_dim), "action_pre": (R, es.act_dim), "logprob": (R,),
                "reward": (R, es.m), "value": (R, es.m), "next_value": (R, es.m),
                "advantages": (R, es.m), "value_targets": (R, es.m), "scalar_advantage": (R,),
                "terminated": (R,), "truncated": (R,), "clusters": (self.cfg.K, es.m),
                "perm": (self.cfg.N * self.cfg.T,), "env_ctr": (N,), "env_steps": (N,),
                "env_key": (N,), "ret_sum": (N,), "ret_cnt": (N,), "tracker": (N, es.m),
                "env_state": (es.obs_dim, N)}[name]  # obs == state for every env

    def _dtype(self, name):
        if name in self._F32:
            return np.float32
        if name in ("terminated", "truncated"):
            return np.uint8
        if name in ("env_ctr", "env_key"):
            return np.uint64
        return np.float64 if name == "ret_sum" else np.int32

    def get(self, name: str) -> np.ndarray:
        """Device field -> host copy. env_state is the SoA [state_dim][N] layout."""
        out = np.zeros(self._shape(name), self._dtype(name))
        _check(LIB.morlax_trainer_get(self._h, name.encode(), _ptr(out)))
        return out

    def set(self, name: str, value):
        v = np.ascontiguousarray(value, self._dtype(name)).reshape(self._shape(name))
        _check(LIB.morlax_trainer_set(self._h, name.encode(), _ptr(v)))

    def save_checkpoint(self, path: str, iteration: int, iterations: int = 300, grid_resolution: int = 10,
                        episodes_per_point: int = 8, log_interval: int = 10, pareto_reference=None):
        """save_checkpoint (checkpoint.cpp:200-213): the reference's MRLXCKPT v1 bytes."""
        ref = _f64(pareto_reference if pareto_reference is not None else [])
        x = _CkExtraC(iterations, grid_resolution, episodes_per_point, log_interval, len(ref),
                      ref.ctypes.data_as(C.POINTER(C.c_double)) if len(ref) else None)
        _check(LIB.morlax_trainer_save_checkpoint(self._h, path.encode(), C.c_int64(iteration), C.byref(x)))

    def load_checkpoint(self, path: str) -> int:
        """load_checkpoint (checkpoint.cpp:215-241) into this trainer's hypernets; returns the iteration."""
        it = C.c_int64()
        _check(LIB.morlax_trainer_load_checkpoint(self._h, path.encode(), C.byref(it)))
        return it.value

    def losses(self, rows):
        r = np.ascontiguousarray(rows, np.int32)
        a, c = C.c_double(), C.c_double()
        _check(LIB.morlax_trainer_losses(self._h, _ptr(r), len(r), C.byref(a), C.byref(c)))
        return a.value, c.value

    @property
    def kernel_launches(self) -> int:
        return int(LIB.morlax_trainer_kernel_launches(self._h))


def shard_rows(P: int, world: int, rank: int):
    """The sharded optimizer's partition of the P hypernet rows (M rows / b
    entries): (S, row_lo, row_hi), S a multiple of 128 (trainer.cu shard_rows)."""
    S, lo, hi = C.c_int64(), C.c_int64(), C.c_int64()
    _check(LIB.morlax_shard_rows(C.c_int64(P), world, rank, C.byref(S), C.byref(lo), C.byref(hi)))
    return S.value, lo.value, hi.value


def shard_minibatch(perm, lo, hi, T, inst_lo, n_inst, reps, n_groups):
    perm = np.ascontiguousarray(perm, np.int32)
    rows = np.zeros(max(hi - lo, 1), np.int32)
    goff = np.zeros(n_groups + 1, np.int32)
    n, mx = C.c_int(), C.c_int()
    _check(LIB.morlax_shard_minibatch(_ptr(perm), lo, hi, T, inst_lo, n_inst, reps, n_groups,
                                      _ptr(rows), _ptr(goff), C.byref(n), C.byref(mx)))
    return rows[:n.value], goff, mx.value


# ---------------------------------------------------------------- pareto (pareto.hpp)
def nondominated_mask(points) -> np.ndarray:
    p = _f64(points)
    n, m = p.shape
    mask = np.zeros(n, np.uint8)
    _check(LIB.morlax_pareto_mask(n, m, _ptr(p), _ptr(mask)))
    return mask


def nondominated_filter(points) -> np.ndarray:
    p = _f64(points)
    return p[nondominated_mask(p).astype(bool)]


def linear_dominance_mask(points) -> np.ndarray:
    """linear_dominance_filter (pareto.cpp:79-139) survivors as a mask."""
    p = _f64(points)
    n, m = p.shape
    mask = np.zeros(n, np.uint8)
    _check(LIB.morlax_linear_dominance_mask(n, m, _ptr(p), _ptr(mask)))
    return mask


def linear_dominance_filter(points) -> np.ndarray:
    p = _f64(points)
    return p[linear_dominance_mask(p).astype(bool)]


def hypervolume_mc(points, reference, samples, key, ctr=0):
    p = _f64(points).reshape(-1, len(reference))
    ref = _f64(reference)
    v, se, h = C.c_double(), C.c_double(), C.c_uint64()
    _check(LIB.morlax_hypervolume_mc(len(p), len(ref), _ptr(p), _ptr(ref), C.c_uint64(samples),
                                     C.c_uint64(key), C.c_uint64(ctr), C.byref(v), C.byref(se),
                                     C.byref(h)))
    return v.value, se.value, h.value


def hypervolume_exact(points, reference):
    """Exact hypervolume for any m <= 8 on the device (WFG recursion; the
    reference is exact only for m <= 4). Returns (value, clipped)."""
    p = _f64(points).reshape(-1, len(reference))
    ref = _f64(reference)
    v, cl = C.c_double(), C.c_int()
    _check(LIB.morlax_hypervolume_exact(len(p), len(ref), _ptr(p), _ptr(ref), C.byref(v), C.byref(cl)))
    return v.value, cl.value


def hypervolume_detailed(points, reference, samples=1_000_000, seed=0x9E3779B9):
    p = _f64(points).reshape(-1, len(reference))
    ref = _f64(reference)
    v, se = C.c_double(), C.c_double()
    ex, cl = C.c_int(), C.c_int()
    _check(LIB.morlax_hypervolume_detailed(len(p), len(ref), _ptr(p), _ptr(ref), C.c_uint64(samples),
                                           C.c_uint64(seed), C.byref(v), C.byref(se), C.byref(ex),
                                           C.byref(cl)))
    return v.value, se.value, bool(ex.value), cl.value


# ---------------------------------------------------------------- train()
@dataclass
class RunOptions:
    """TrainOptions + EvalConfig + TrainerConfig::iterations + the Pareto
    reference of RunConfig (trainer.hpp:59-77, 237-241); defaults = the
    reference's."""
    out_dir: str = ""
    iterations: int = 300
    grid_resolution: int = 10
    episodes_per_point: int = 8
    log_interval: int = 10
    pareto_reference: list = None
    deterministic: bool = False


@dataclass
class IterationRecord:
    """IterationStats (trainer.hpp:243-249)."""
    iteration: int
    actor_loss: float
    critic_loss: float
    archive_hypervolume: float
    cluster_returns: np.ndarray


class _RunOptsC(C.Structure):
    _fields_ = [("out_dir", C.c_char_p), ("iterations", C.c_int), ("grid_resolution", C.c_int),
                ("episodes_per_point", C.c_int), ("log_interval", C.c_int),
                ("n_pareto_reference", C.c_int), ("pareto_reference", C.POINTER(C.c_double)),
                ("deterministic", C.c_int)]


class _IterRecC(C.Structure):
    _fields_ = [("iteration", C.c_int), ("actor_loss", C.c_double), ("critic_loss", C.c_double),
                ("archive_hypervolume", C.c_double), ("n_clusters", C.c_int),
                ("cluster_returns", C.POINTER(C.c_double))]


_ITER_CB = C.CFUNCTYPE(C.c_int, C.POINTER(_IterRecC), C.c_void_p)


def train(cfg: TrainConfig, opts: RunOptions = None, callback=None) -> "Trainer":
    """train(RunConfig, TrainOptions, IterationCallback) (train.cpp:55-229) on
    one GPU: returns the trained Trainer (params(), save_checkpoint(), ...).
    With opts.out_dir, writes metrics.csv and checkpoint.bin there like the
    reference (on a NumericError: the last healthy checkpoint, then raises).
    An exception raised by `callback(IterationRecord)` stops training and
    propagates."""
    opts = opts or RunOptions()
    ref = None
    if opts.pareto_reference is not None:
        ref = np.ascontiguousarray(opts.pareto_reference, dtype=np.float64)
    o = _RunOptsC(opts.out_dir.encode() if opts.out_dir else None, opts.iterations, opts.grid_resolution,
                  opts.episodes_per_point, opts.log_interval, 0 if ref is None else len(ref),
                  None if ref is None else ref.ctypes.data_as(C.POINTER(C.c_double)),
                  1 if opts.deterministic else 0)
    err = []

    def _cb(p, _user):
        if callback is None:
            return 0
        r = p.contents
        rec = IterationRecord(r.iteration, r.actor_loss, r.critic_loss, r.archive_hypervolume,
                              np.ctypeslib.as_array(r.cluster_returns, (r.n_clusters,)).copy())
        try:
            callback(rec)
        except BaseException as e:  # noqa: BLE001 -- re-raised below
            err.append(e)
            return 1
        return 0

    cb = _ITER_CB(_cb)
    h = C.c_void_p()
    c = cfg.c()
    rc = LIB.morlax_train(C.byref(c), C.byref(o), cb, None, C.byref(h))
    if err:
        raise err[0]
    _check(rc)
    return Trainer(cfg, _handle=h)
