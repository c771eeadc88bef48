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
