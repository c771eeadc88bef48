"""The drop-in boundary, compiled: integration/train_b200.cpp (the adapter a
reference maintainer adds next to proj/src/train.cpp) built against the
reference headers and linked with the compiled reference and
libmorlax_b200.so by oracle/Makefile (`adapter`), run against the
reference's own train() / nondominated_filter / evaluate_params on the same
configuration, including the CLI exit-code contract (tools/commands.hpp:12-32:
ConfigError -> 2, NumericError -> 3) through the reference's guarded()."""
import json
import os
import subprocess

import numpy as np
import pytest

from helpers import REL_CHAIN, ROOT, assert_update_close, hyper_blocks
from pyoracle import Oracle, TrainCfg

pytestmark = pytest.mark.gpu
BIN = os.path.join(ROOT, "oracle", "_ref", "train_b200_check")


@pytest.fixture(scope="module")
def run(tmp_path_factory):
    if not os.path.exists(BIN):
        pytest.skip("adapter check binary not built (make -C oracle adapter, needs /root/reference)")
    prefix = str(tmp_path_factory.mktemp("adapter") / "ck")
    out = subprocess.run([BIN, prefix], capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    return json.loads(out.stdout.strip().splitlines()[-1]), prefix


def test_adapter_train_matches_reference_train(run):
    d, prefix = run
    assert d["iteration_b200"] == d["iteration_ref"] == 3
    for k in ("actor_loss", "critic_loss"):
        b, r = np.array(d[k + "_b200"]), np.array(d[k + "_ref"])
        assert len(b) == len(r) == 3
        assert np.all(np.abs(b - r) <= REL_CHAIN * np.maximum(1.0, np.abs(r))), (k, b, r)
    assert np.allclose(d["hv_b200"], d["hv_ref"], rtol=REL_CHAIN)
    rb, rr = np.array(d["returns_b200"]), np.array(d["returns_ref"])
    assert np.array_equal(rb == -1e300, rr == -1e300)  # episodes completed in the same windows
    ok = rr != -1e300
    assert np.allclose(rb[ok], rr[ok], rtol=REL_CHAIN, atol=1e-2)
    c = TrainCfg(env="mo-pointmass", N=16, K=2, T=12, epochs=2, minibatch_count=2, F=16, feat_hidden=[16],
                 actor_hidden=[16, 16], critic_hidden=[16, 16], seed=5)
    o = Oracle("oracle")
    root = o.rng_seed_state(5)[0]
    for which, lane, spec, lr in (("actor", 0xA1, c.specs()[0], c.actor_lr), ("critic", 0xA2, c.specs()[1], c.critic_lr)):
        p0 = o.init_hypernet(spec, o.split_key(root, lane))  # train.cpp:67-70
        pb = np.fromfile(f"{prefix}_{which}_b200.bin", np.float64)
        pr = np.fromfile(f"{prefix}_{which}_ref.bin", np.float64)
        assert len(pb) == len(pr) == spec.n_params
        assert_update_close(pb, pr, p0, lr, hyper_blocks(spec), rel_l2=0.1, sign_agree=0.995, what=f"adapter {which}")


def test_adapter_exit_codes_match_the_cli_contract(run):
    d, _ = run
    assert d["config_exit_b200"] == d["config_exit_ref"] == 2
    assert d["numeric_exit_b200"] == d["numeric_exit_ref"] == 3


def test_adapter_pareto_and_evaluation(run):
    d, _ = run
    assert d["nondominated_equal"]
    assert d["eval_grid_equal"]
    assert d["eval_max_abs"] <= REL_CHAIN * max(d["eval_scale"], 1e-12)
