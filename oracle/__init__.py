"""CPU oracle for arXiv:1409.8563 — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` leg may import this package.  The
product path (``paper_1409_8563_b200``) never imports it and shares no code
with it.

``liboracle.so`` is built from ``oracle.c`` (plain C, fp64,
``-ffp-contract=off``) by :func:`build`; this module is argument marshalling
over ctypes plus numpy conveniences.  Every function cites the paper passage it
follows in ``oracle.c``.  Parity pins: see ``tests/test_oracle_*.py``.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

CFLAGS = ["-O2", "-std=c11", "-ffp-contract=off", "-fno-fast-math", "-fPIC",
          "-shared", "-fopenmp"]


def build(force: bool = False) -> str:
    """Compile oracle.c -> liboracle.so (gcc, plain C, no FMA contraction)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < max(
            os.path.getmtime(_SRC), os.path.getmtime(os.path.join(_HERE, "oracle.h"))):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", *CFLAGS, _SRC, "-o", tmp, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


class _Problem(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int32), ("c", ctypes.c_double * 3),
                ("nu0", ctypes.c_double), ("omega", ctypes.c_double),
                ("T", ctypes.c_double), ("nu_mode", ctypes.c_int32)]


@dataclass
class Problem:
    """Eq.(adv_diff_eq), nu(t) P:437, parameters P:447-448."""
    n: int
    c: tuple = (1.0, 1.0, 1.0)
    nu0: float = 0.1
    omega: float = 100.0
    T: float = 0.1
    nu_mode: int = 0  # 0 = stage times, 1 = step start (C1)

    def _c(self) -> _Problem:
        p = _Problem()
        p.n = self.n
        p.c[0], p.c[1], p.c[2] = (float(v) for v in self.c)
        p.nu0, p.omega, p.T, p.nu_mode = self.nu0, self.omega, self.T, self.nu_mode
        return p


_lib = None
_D = ctypes.POINTER(ctypes.c_double)


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        P = ctypes.POINTER(_Problem)
        i32, i64, dbl = ctypes.c_int32, ctypes.c_int64, ctypes.c_double
        sig = {
            "orc_nu": (dbl, [dbl, dbl, dbl]),
            "orc_amplitude": (dbl, [dbl, dbl, dbl]),
            "orc_initial": (None, [i32, _D]),
            "orc_exact": (None, [P, dbl, _D]),
            "orc_rhs_coarse": (None, [i32, _D, dbl, _D, _D]),
            "orc_rhs_fine": (None, [i32, _D, dbl, _D, _D]),
            "orc_coarse": (None, [P, _D, i64, i64, dbl]),
            "orc_fine": (None, [P, _D, i64, i64, dbl]),
            "orc_inf_norm": (dbl, [i32, _D]),
            "orc_inf_diff": (dbl, [i32, _D, _D]),
            "orc_defect": (dbl, [i32, _D, _D]),
            "orc_parareal": (ctypes.c_int, [P, i32, i32, i32, i32, _D, _D, _D, _D, i32]),
            "orc_threads": (ctypes.c_int, []),
            "orc_parareal_tol": (ctypes.c_int, [P, i32, i32, i32, i32, dbl, i32, _D, _D, _D, _D, _D,
                                                ctypes.POINTER(ctypes.c_int32), i32]),
            "orc_restrict": (None, [i32, _D, _D]),
            "orc_prolong": (None, [i32, _D, _D]),
            "orc_coarse_mesh": (None, [P, _D, i64, i64, dbl]),
        }
        for name, (res, args) in sig.items():
            f = getattr(L, name)
            f.restype, f.argtypes = res, args
        _lib = L
    return _lib


def _ptr(a: np.ndarray):
    assert a.dtype == np.float64 and a.flags.c_contiguous
    return a.ctypes.data_as(_D)


def _field(n: int) -> np.ndarray:
    return np.empty((n, n, n), dtype=np.float64)


def nu(nu0: float, omega: float, t: float) -> float:
    return lib().orc_nu(nu0, omega, t)


def amplitude(nu0: float, omega: float, t: float) -> float:
    return lib().orc_amplitude(nu0, omega, t)


def initial(n: int) -> np.ndarray:
    u = _field(n)
    lib().orc_initial(n, _ptr(u))
    return u


def exact(p: Problem, t: float) -> np.ndarray:
    u = _field(p.n)
    pc = p._c()
    lib().orc_exact(ctypes.byref(pc), t, _ptr(u))
    return u


def _cvec(c):
    arr = (ctypes.c_double * 3)(*[float(v) for v in c])
    return ctypes.cast(arr, _D), arr


def rhs_coarse(u: np.ndarray, c, nu_val: float) -> np.ndarray:
    u = np.ascontiguousarray(u, dtype=np.float64)
    out = np.empty_like(u)
    cp, _keep = _cvec(c)
    lib().orc_rhs_coarse(u.shape[0], cp, nu_val, _ptr(u), _ptr(out))
    return out


def rhs_fine(u: np.ndarray, c, nu_val: float) -> np.ndarray:
    u = np.ascontiguousarray(u, dtype=np.float64)
    out = np.empty_like(u)
    cp, _keep = _cvec(c)
    lib().orc_rhs_fine(u.shape[0], cp, nu_val, _ptr(u), _ptr(out))
    return out


def coarse(p: Problem, u: np.ndarray, step0: int, n_steps: int, dt: float) -> np.ndarray:
    """G over global steps [step0, step0+n_steps) (Alg.2); returns a new array."""
    v = np.array(u, dtype=np.float64, order="C", copy=True)
    pc = p._c()
    lib().orc_coarse(ctypes.byref(pc), _ptr(v), step0, n_steps, dt)
    return v


def restrict(u: np.ndarray) -> np.ndarray:
    """Injection onto the n/2 mesh (C24)."""
    u = np.ascontiguousarray(u, dtype=np.float64)
    n = u.shape[0]
    uc = _field(n // 2)
    lib().orc_restrict(n, _ptr(u), _ptr(uc))
    return uc


def prolong(uc: np.ndarray) -> np.ndarray:
    """Periodic trilinear prolongation from the n/2 mesh (C25)."""
    uc = np.ascontiguousarray(uc, dtype=np.float64)
    n = 2 * uc.shape[0]
    u = _field(n)
    lib().orc_prolong(n, _ptr(uc), _ptr(u))
    return u


def coarse_mesh(p: Problem, u: np.ndarray, step0: int, n_steps: int, dt: float) -> np.ndarray:
    """G_c = prolong o (Alg.2 on the n/2 mesh) o restrict (C26)."""
    v = np.array(u, dtype=np.float64, order="C", copy=True)
    pc = p._c()
    lib().orc_coarse_mesh(ctypes.byref(pc), _ptr(v), step0, n_steps, dt)
    return v


def fine(p: Problem, u: np.ndarray, step0: int, n_steps: int, dt: float) -> np.ndarray:
    """F over global steps [step0, step0+n_steps) (classical RK4)."""
    v = np.array(u, dtype=np.float64, order="C", copy=True)
    pc = p._c()
    lib().orc_fine(ctypes.byref(pc), _ptr(v), step0, n_steps, dt)
    return v


def inf_norm(u: np.ndarray) -> float:
    u = np.ascontiguousarray(u, dtype=np.float64)
    return lib().orc_inf_norm(u.shape[0], _ptr(u))


def defect(u: np.ndarray, ref: np.ndarray) -> float:
    u = np.ascontiguousarray(u, dtype=np.float64)
    ref = np.ascontiguousarray(ref, dtype=np.float64)
    return lib().orc_defect(u.shape[0], _ptr(u), _ptr(ref))


@dataclass
class PararealResult:
    u_T: np.ndarray
    defects: np.ndarray = field(default=None)


def parareal(p: Problem, n_slices: int, nc: int, nf: int, K: int,
             u0: np.ndarray | None = None, u_ref: np.ndarray | None = None,
             g_is_f: bool = False, g_half_mesh: bool = False) -> PararealResult:
    """Alg.1 for all ranks, executed serially in pipeline order."""
    u0 = initial(p.n) if u0 is None else np.ascontiguousarray(u0, dtype=np.float64)
    uT = _field(p.n)
    d = np.full(K + 1, np.nan)
    pc = p._c()
    rc = lib().orc_parareal(ctypes.byref(pc), n_slices, nc, nf, K, _ptr(u0),
                            _ptr(np.ascontiguousarray(u_ref)) if u_ref is not None else None,
                            _ptr(uT), _ptr(d), (1 if g_is_f else 0) | (4 if g_half_mesh else 0))
    if rc != 0:
        raise ValueError("orc_parareal: bad arguments")
    return PararealResult(uT, d if u_ref is not None else None)


@dataclass
class PararealTolResult:
    u_T: np.ndarray
    defects: np.ndarray
    changes: np.ndarray   # (world, K) relative iterate change per rank and iteration
    iters: np.ndarray     # iterations run per rank


def parareal_tol(p: Problem, n_slices: int, nc: int, nf: int, K: int, tol: float, world: int,
                 u0: np.ndarray | None = None, u_ref: np.ndarray | None = None,
                 g_half_mesh: bool = False) -> PararealTolResult:
    """Alg.1 with the convergence-controlled stop rule of DESIGN.md C23."""
    u0 = initial(p.n) if u0 is None else np.ascontiguousarray(u0, dtype=np.float64)
    uT = _field(p.n)
    d = np.full(K + 1, np.nan)
    ch = np.full(world * K, np.nan)
    it = (ctypes.c_int32 * world)()
    pc = p._c()
    rc = lib().orc_parareal_tol(ctypes.byref(pc), n_slices, nc, nf, K, tol, world, _ptr(u0),
                                _ptr(np.ascontiguousarray(u_ref)) if u_ref is not None else None,
                                _ptr(uT), _ptr(d), _ptr(ch), it, 4 if g_half_mesh else 0)
    if rc != 0:
        raise ValueError("orc_parareal_tol: bad arguments")
    return PararealTolResult(uT, d, ch.reshape(world, K), np.array(list(it)))


def serial_fine(p: Problem, n_steps_total: int, u0: np.ndarray | None = None) -> np.ndarray:
    """u_fine: F over [0, N_t) with dt = T/N_t (reading C7)."""
    u0 = initial(p.n) if u0 is None else u0
    return fine(p, u0, 0, n_steps_total, p.T / n_steps_total)


def threads() -> int:
    return lib().orc_threads()
