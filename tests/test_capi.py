"""CPU checks of the C-ABI boundary (no GPU compute): the library loads,
exports every symbol include/morlax_b200.h declares, validates configs with
the reference's exception taxonomy, and its host-side sharding helper
partitions minibatch rows exactly."""
import ctypes as C
import re

import numpy as np
import pytest

import paper_2603_09237_b200 as mb
from paper_2603_09237_b200._lib import HEADER, LIB_PATH, exported_symbols


def test_library_exports_every_header_symbol():
    syms = exported_symbols()
    assert len(syms) >= 40
    lib = C.CDLL(LIB_PATH)
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing


def test_header_is_plain_c():
    src = open(HEADER).read()
    assert 'extern "C"' in src
    assert not re.search(r"\b(std::|torch::|at::|c10::)", src)


def test_env_specs_match_reference_registry():  # registry.cpp / env_*.cpp make_spec
    assert mb.env_spec("mo-lqr1d") == mb.EnvSpec("mo-lqr1d", 1, 1, 2, 200)
    assert mb.env_spec("mo-lqr1d-m1") == mb.EnvSpec("mo-lqr1d-m1", 1, 1, 1, 200)
    assert mb.env_spec("mo-pointmass") == mb.EnvSpec("mo-pointmass", 4, 2, 2, 200)
    assert mb.env_spec("mo-dst-continuous") == mb.EnvSpec("mo-dst-continuous", 1, 1, 2, 50)
    assert mb.env_spec("mo-humanoid6") == mb.EnvSpec("mo-humanoid6", 45, 12, 6, 1000)
    with pytest.raises(mb.ConfigError):
        mb.env_spec("no-such-env")


@pytest.mark.parametrize("kw,msg", [
    (dict(N=10, K=3), "K must divide N"),
    (dict(K=1, N=4), "K must be > 1"),
    (dict(kappa=3), "kappa must be <= m"),
    (dict(gamma=1.0), "gamma"),
    (dict(clip_eps=0.0), "clip_eps"),
    (dict(epochs=0), "epochs"),
    (dict(env_name="mo-lqr1d-m1", N=4, K=2), "K must equal trainer.N"),
])
def test_trainer_config_validation(kw, msg):  # config.cpp:17-45, simplex.cpp:44-53
    with pytest.raises(mb.ConfigError, match=msg):
        mb.Trainer(mb.TrainConfig(**kw))


def test_hypernet_param_counts():  # hypernet.cpp:44-48
    a = mb.HypernetSpec(6, 256, [256], [45, 256, 256, 12], True, True)
    assert a.target_param_count == 80664
    c = mb.HypernetSpec(6, 256, [256], [45, 256, 256, 6], False, False)
    assert c.target_param_count == 79110
    assert a.param_count == (7 * 256 + 257 * 256) + 80664 * 256 + 80664


def test_shard_minibatch_partitions_rows():
    rng = np.random.default_rng(0)
    N, K, T, world = 64, 8, 16, 4
    reps = N // K
    perm = rng.permutation(N * T).astype(np.int32)
    lo, hi = 100, 700
    seen = []
    for r in range(world):
        n_inst = N // world
        rows, goff, mx = mb.shard_minibatch(perm, lo, hi, T, r * n_inst, n_inst, reps, K // world)
        assert goff[0] == 0 and goff[-1] == len(rows)
        # rows are local ids, grouped by local cluster, minibatch order kept in a group
        for z in range(K // world):
            seg = rows[goff[z]:goff[z + 1]]
            assert np.all(seg // T // reps == z)
            glob = seg + r * n_inst * T
            pos = [np.where(perm[lo:hi] == x)[0][0] for x in glob]
            assert pos == sorted(pos)
        seen.extend((rows + r * n_inst * T).tolist())
    assert sorted(seen) == sorted(perm[lo:hi].tolist())


def test_no_gpu_calls_fail_loudly():
    if mb.LIB.morlax_device_count() > 0:
        pytest.skip("GPU present")
    with pytest.raises(mb.CudaError):
        mb.BatchedEnv("mo-pointmass", 4)
