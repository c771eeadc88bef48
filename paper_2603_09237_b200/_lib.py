"""Loads the in-tree CUDA library (libmorlax_b200.so, sm_100a). Builds it with
nvcc (build.sh) when it is missing. There is no fallback: if the library
cannot be built or loaded the import fails loudly."""
from __future__ import annotations

import ctypes as C
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libmorlax_b200.so")
HEADER = os.path.join(os.path.dirname(HERE), "include", "morlax_b200.h")


def build(quiet: bool = True) -> str:
    r = subprocess.run(["bash", os.path.join(HERE, "build.sh")], capture_output=True, text=True)
    if r.returncode != 0:
        raise ImportError("building libmorlax_b200.so failed:\n" + r.stdout[-4000:] + r.stderr[-4000:])
    if not quiet:
        print(r.stdout)
    return LIB_PATH


def _stale() -> bool:
    if not os.path.exists(LIB_PATH):
        return True
    so = os.path.getmtime(LIB_PATH)
    src = os.path.join(HERE, "csrc")
    return any(os.path.getmtime(os.path.join(src, f)) > so for f in os.listdir(src)) or \
        os.path.getmtime(HEADER) > so


def _load():
    if not os.path.exists(LIB_PATH) or (os.environ.get("MORLAX_REBUILD") and _stale()):
        build()
    lib = C.CDLL(LIB_PATH, mode=C.RTLD_GLOBAL)
    lib.morlax_last_error.restype = C.c_char_p
    lib.morlax_last_error_kind.restype = C.c_char_p
    lib.morlax_env_clamp_count.restype = C.c_uint64
    lib.morlax_env_clamp_count.argtypes = [C.c_void_p]
    lib.morlax_env_destroy.argtypes = [C.c_void_p]
    lib.morlax_trainer_destroy.argtypes = [C.c_void_p]
    lib.morlax_loopback_destroy.argtypes = [C.c_void_p]
    lib.morlax_trainer_create_loopback.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_void_p]
    lib.morlax_hypernet_param_count.restype = C.c_int64
    lib.morlax_hypernet_target_count.restype = C.c_int64
    lib.morlax_trainer_kernel_launches.restype = C.c_int64
    lib.morlax_trainer_kernel_launches.argtypes = [C.c_void_p]
    lib.morlax_trainer_stream.restype = C.c_void_p
    lib.morlax_trainer_stream.argtypes = [C.c_void_p]
    lib.morlax_policy_destroy.argtypes = [C.c_void_p]
    lib.morlax_policy_set_params.argtypes = [C.c_void_p, C.c_void_p]
    lib.morlax_policy_forward.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
    lib.morlax_policy_forward_device.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
    lib.morlax_policy_flops.restype = C.c_double
    lib.morlax_policy_flops.argtypes = [C.c_void_p]
    lib.morlax_simplex_grid_size.restype = C.c_int64
    lib.morlax_dm_adam_test.argtypes = [C.c_int] * 3 + [C.c_void_p] * 5 + [C.c_float] * 3 + [C.c_void_p]
    for name in ("morlax_env_reset", "morlax_env_step", "morlax_env_current_obs",
                 "morlax_env_step_device", "morlax_trainer_iteration", "morlax_trainer_phase",
                 "morlax_trainer_sizes", "morlax_trainer_get_params", "morlax_trainer_set_params",
                 "morlax_trainer_get_grad", "morlax_trainer_get", "morlax_trainer_set",
                 "morlax_trainer_losses", "morlax_trainer_get_theta"):
        getattr(lib, name).argtypes = None  # variadic-safe: callers pass ctypes objects
    return lib


LIB = _load()


def exported_symbols() -> list:
    """Every function the C header declares (for the ABI test)."""
    import re
    with open(HEADER) as f:
        src = f.read()
    return sorted(set(re.findall(r"\b(morlax_[a-z0-9_]+)\s*\(", src)))
