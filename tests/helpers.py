"""Shared test helpers. Tolerances are stated here once:
bit-exact for integer words / indices / flags / masks / hit counts; fp32
device arithmetic vs the fp64 reference within REL (relative, with an
absolute floor like tests/support/fd.hpp:29-39 of the reference)."""
import os

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden", "golden_ref.npz")
REF_SRC = "/root/reference/proj"

# fp32 single-kernel results (env step, GAE, scalarise, Adam, hypernet fwd)
REL_F32 = 1e-5
# GEMM-fed results: the policy / critic / hypernet contractions run on the
# tcgen05 tensor cores with bf16 operands and fp32 accumulation (north star:
# "bf16 in, fp32 accumulate"). Stated bf16 tolerance, NORMWISE:
#   max|gpu - ref| <= REL_BF16 * max|ref|   (theta, losses, gradients)
REL_BF16 = 5e-3
# trajectories fed back through the bf16 policy (rollout obs / actions /
# values over T steps) and post-Adam weights
REL_CHAIN = 2e-2


def assert_normwise(a, b, rel, what=""):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    scale = max(float(np.abs(b).max()), 1e-30)
    e = float(np.abs(a - b).max()) / scale
    assert e <= rel, f"{what}: normwise rel err {e:.3g} > {rel:.3g}"


def golden():
    return np.load(GOLDEN)


def max_rel_err(a, b, floor):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    scale = np.maximum(np.maximum(np.abs(a), np.abs(b)), floor)
    return float(np.max(np.abs(a - b) / scale)) if a.size else 0.0


def assert_close(a, b, rel, floor=1e-6, what=""):
    e = max_rel_err(a, b, floor)
    assert e <= rel, f"{what}: max rel err {e:.3g} > {rel:.3g}"


def ref_available():
    return os.path.exists(os.path.join(ROOT, "oracle", "_ref", "libmorlax_ref.so"))


def bf16(x):
    """Round to bfloat16 (round-to-nearest-even), returned as float64: the
    operand rounding of the device's tensor-core GEMMs."""
    b = np.ascontiguousarray(x, np.float32).view(np.uint32).astype(np.uint64)
    b = ((b + 0x7FFF + ((b >> 16) & 1)) & 0xFFFF0000).astype(np.uint32)
    return b.view(np.float32).astype(np.float64)


def hyper_blocks(spec):
    """[feature | M (P x F) | b (P)] flat-layout blocks of a hypernet spec
    (hypernet.hpp:20-36), for per-block comparisons."""
    nf, P, F = spec.n_feature, spec.P, spec.F
    return {"feature": (0, nf), "M": (nf, nf + P * F), "b": (nf + P * F, nf + P * F + P)}


def update_errors(p, ref, p0, lr, blocks):
    """Compare two Adam trajectories from the same start p0 in update space:
    per block, the relative L2 error of the update (p - p0) against the
    reference update (ref - p0), and the sign agreement of the updates on the
    entries the reference moved by at least half a learning-rate step (Adam
    moves every weight by ~lr per step regardless of |g|, so only weights
    with a decided gradient sign are expected to agree)."""
    out = {}
    for name, (lo, hi) in blocks.items():
        d = np.asarray(p[lo:hi], np.float64) - p0[lo:hi]
        r = np.asarray(ref[lo:hi], np.float64) - p0[lo:hi]
        big = np.abs(r) >= 0.5 * lr
        out[name] = {"rel_l2": float(np.linalg.norm(d - r) / max(np.linalg.norm(r), 1e-30)),
                     "sign_agree": float(np.mean(np.sign(d[big]) == np.sign(r[big]))) if big.any() else 1.0,
                     "moved": int(big.sum())}
    return out


def assert_update_close(p, ref, p0, lr, blocks, rel_l2, sign_agree, what=""):
    errs = update_errors(p, ref, p0, lr, blocks)
    for name, e in errs.items():
        assert e["rel_l2"] <= rel_l2, f"{what} {name}: update rel L2 err {e['rel_l2']:.3g} > {rel_l2} ({errs})"
        assert e["sign_agree"] >= sign_agree, \
            f"{what} {name}: update sign agreement {e['sign_agree']:.4f} < {sign_agree} ({errs})"
    return errs
