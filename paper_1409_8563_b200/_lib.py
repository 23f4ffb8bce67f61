"""ctypes binding of include/parareal.h — argument marshalling only.

Every step of the hot path runs in libparareal.so (hand-written sm_100a
kernels + NCCL).  There is no CPU fallback: if the library is missing or the
device is not a B200 the calls raise.
"""
from __future__ import annotations

import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
# PR_LIB: an alternative build of the same library (e.g. the PRK_DEBUG index-checking build)
LIB_PATH = os.environ.get("PR_LIB") or os.path.join(HERE, "libparareal.so")

PR_OK, PR_EINVAL, PR_ENOMEM, PR_ECUDA, PR_ENCCL, PR_EDOMAIN, PR_ESTATE = range(7)
STATUS_NAMES = {0: "PR_OK", 1: "PR_EINVAL", 2: "PR_ENOMEM", 3: "PR_ECUDA", 4: "PR_ENCCL",
                5: "PR_EDOMAIN", 6: "PR_ESTATE"}
PR_NU_STAGE, PR_NU_STEP_START = 0, 1
PR_FLAG_G_IS_F = 1
PR_FLAG_PEER_HANDOFF = 2
PR_FLAG_G_HALF_MESH = 4
PR_NCCL_ID_BYTES = 128
OPS = {1: "G_PREFIX", 2: "G_INIT", 3: "DEFECT0", 4: "F", 5: "RECV", 6: "G", 7: "CORRECT",
       8: "SEND", 9: "END_ITER"}

# Every symbol include/parareal.h declares (checked by tests/test_abi.py).
EXPORTS = ["pr_create_grid", "pr_destroy_grid", "pr_fine", "pr_coarse", "pr_coarse_mesh", "pr_defect",
           "pr_fill_sine", "pr_correct", "pr_nccl_unique_id", "pr_comm_init", "pr_parareal",
           "pr_plan", "pr_last_timings", "pr_kernel_launches", "pr_stability_ratio",
           "pr_last_error", "pr_version", "pr_grid_info", "pr_last_monitors", "pr_local_group"]


class PrProblem(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int32), ("c", ctypes.c_double * 3), ("nu0", ctypes.c_double),
                ("omega", ctypes.c_double), ("T", ctypes.c_double), ("nu_mode", ctypes.c_int32)]


class PrPararealCfg(ctypes.Structure):
    _fields_ = [("n_slices", ctypes.c_int32), ("n_coarse_per_slice", ctypes.c_int32),
                ("n_fine_per_slice", ctypes.c_int32), ("K", ctypes.c_int32),
                ("flags", ctypes.c_int32), ("tol", ctypes.c_double)]


class PrOp(ctypes.Structure):
    _fields_ = [("op", ctypes.c_int32), ("k", ctypes.c_int32), ("slice", ctypes.c_int32),
                ("peer", ctypes.c_int32)]


class PrGridInfo(ctypes.Structure):
    _fields_ = [("fine_kernels_per_step", ctypes.c_int32), ("fine_bytes_per_point", ctypes.c_int32),
                ("coarse_bytes_per_point", ctypes.c_int32), ("sms", ctypes.c_int32),
                ("fine_variant", ctypes.c_int32)]


class PrError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS_NAMES.get(status, status)}: {msg}")
        self.status = status


_lib = None


def load() -> ctypes.CDLL:
    """Load libparareal.so (fails loudly if it was not built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: run `python -c 'import __graft_entry__ as g; g.build()'` "
                          "(nvcc, sm_100a).  There is no CPU fallback.")
    L = ctypes.CDLL(LIB_PATH)
    vp, i32, i64, dbl = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_double
    st = ctypes.c_int
    sig = {
        "pr_create_grid": (st, [ctypes.POINTER(PrProblem), i32, ctypes.POINTER(vp)]),
        "pr_destroy_grid": (st, [vp]),
        "pr_fine": (st, [vp, vp, vp, i64, i64, dbl, vp]),
        "pr_coarse": (st, [vp, vp, vp, i64, i64, dbl, vp]),
        "pr_coarse_mesh": (st, [vp, vp, vp, i64, i64, dbl, vp]),
        "pr_defect": (st, [vp, vp, vp, ctypes.POINTER(dbl), vp]),
        "pr_fill_sine": (st, [vp, vp, vp]),
        "pr_correct": (st, [vp, vp, vp, vp, vp, vp, ctypes.POINTER(dbl), vp]),
        "pr_nccl_unique_id": (st, [vp]),
        "pr_comm_init": (st, [vp, i32, i32, vp]),
        "pr_parareal": (st, [vp, ctypes.POINTER(PrPararealCfg), vp, vp, vp, ctypes.POINTER(dbl), vp]),
        "pr_plan": (st, [i32, i32, i32, i32, ctypes.POINTER(PrOp), i32, ctypes.POINTER(i32)]),
        "pr_last_timings": (st, [vp, ctypes.POINTER(dbl), i32]),
        "pr_kernel_launches": (i64, []),
        "pr_stability_ratio": (st, [ctypes.POINTER(PrProblem), dbl, i32, ctypes.POINTER(dbl)]),
        "pr_last_error": (ctypes.c_char_p, []),
        "pr_version": (ctypes.c_char_p, []),
        "pr_grid_info": (st, [vp, ctypes.POINTER(PrGridInfo)]),
        "pr_last_monitors": (st, [vp, ctypes.POINTER(dbl), i32, ctypes.POINTER(i32)]),
        "pr_local_group": (st, [ctypes.POINTER(vp), i32]),
    }
    for name, (res, args) in sig.items():
        f = getattr(L, name)
        f.restype, f.argtypes = res, args
    _lib = L
    return L


def check(status: int) -> None:
    if status != PR_OK:
        raise PrError(status, load().pr_last_error().decode())
