"""B200-native hot path of arXiv:1409.8563 (Parareal over fp64 stencils).

Thin Python binding over ``libparareal.so`` (C ABI: ``include/parareal.h``).
The functions keep the C names; tensors replace pointers.  Fields are
C-contiguous float64 arrays of shape (n, n, n) indexed (z, y, x): CUDA tensors
(device pointers, asynchronous on the current torch stream) or CPU tensors /
numpy arrays (host pointers, staged by the library, synchronous).

PyTorch is plumbing here (device memory, streams, process groups); every step
of the method runs in the library's kernels.  There is no CPU fallback.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass

from . import _lib
from ._lib import (PR_NU_STAGE, PR_NU_STEP_START, PR_FLAG_G_IS_F, PR_FLAG_PEER_HANDOFF,
                   PR_FLAG_G_HALF_MESH, PrError, OPS,
                   PR_NCCL_ID_BYTES)

__all__ = ["Problem", "PararealCfg", "Grid", "pr_create_grid", "pr_destroy_grid", "pr_fine",
           "pr_coarse", "pr_defect", "pr_fill_sine", "pr_correct", "pr_nccl_unique_id",
           "pr_comm_init", "pr_parareal", "pr_plan", "pr_last_timings", "pr_kernel_launches",
           "pr_stability_ratio", "pr_last_error", "pr_version", "pr_grid_info", "pr_last_monitors", "PrError", "PR_NU_STAGE",
           "PR_NU_STEP_START", "PR_FLAG_G_IS_F", "PR_FLAG_PEER_HANDOFF", "PR_FLAG_G_HALF_MESH",
           "pr_coarse_mesh", "comm_init_torch", "pr_local_group"]


@dataclass
class Problem:
    """Eq.(adv_diff_eq); nu(t) = nu0 + nu0/2 sin(omega t); T."""
    n: int
    c: tuple = (1.0, 1.0, 1.0)
    nu0: float = 0.1
    omega: float = 100.0
    T: float = 0.1
    nu_mode: int = PR_NU_STAGE

    def _c(self) -> _lib.PrProblem:
        p = _lib.PrProblem()
        p.n = int(self.n)
        for i in range(3):
            p.c[i] = float(self.c[i])
        p.nu0, p.omega, p.T, p.nu_mode = float(self.nu0), float(self.omega), float(self.T), int(self.nu_mode)
        return p


@dataclass
class PararealCfg:
    """N_p, N_c, N_f, K of P:211-214 (Alg.1)."""
    n_slices: int
    n_coarse_per_slice: int
    n_fine_per_slice: int
    K: int
    flags: int = 0
    tol: float = 0.0   # > 0: convergence-controlled stopping (C23)

    def _c(self) -> _lib.PrPararealCfg:
        c = _lib.PrPararealCfg()
        c.n_slices, c.n_coarse_per_slice, c.n_fine_per_slice = self.n_slices, self.n_coarse_per_slice, self.n_fine_per_slice
        c.K, c.flags, c.tol = self.K, self.flags, float(self.tol)
        return c


def _ptr(x):
    """Device or host address of a contiguous float64 field (torch or numpy)."""
    if x is None:
        return None
    if hasattr(x, "data_ptr"):  # torch.Tensor
        import torch
        if x.dtype != torch.float64 or not x.is_contiguous():
            raise TypeError("fields must be contiguous float64 tensors")
        return ctypes.c_void_p(x.data_ptr())
    import numpy as np
    if not isinstance(x, np.ndarray) or x.dtype != np.float64 or not x.flags.c_contiguous:
        raise TypeError("fields must be contiguous float64 arrays")
    return ctypes.c_void_p(x.ctypes.data)


def _stream(stream, *fields):
    if stream is not None:
        return ctypes.c_void_p(int(stream))
    for f in fields:
        if f is not None and hasattr(f, "is_cuda") and f.is_cuda:
            import torch
            return ctypes.c_void_p(torch.cuda.current_stream(f.device).cuda_stream)
    return ctypes.c_void_p(0)


def _size_check(grid, *fields):
    n3 = grid.problem.n ** 3
    for f in fields:
        if f is None:
            continue
        numel = f.numel() if hasattr(f, "numel") else f.size
        if numel != n3:
            raise ValueError(f"field has {numel} values, expected n^3 = {n3}")


class Grid:
    """Owns a pr_grid handle (scratch fields, nu tables, graphs, NCCL comm)."""

    def __init__(self, problem: Problem, device: int = 0):
        L = _lib.load()
        self.problem = problem
        self.device = device
        h = ctypes.c_void_p()
        pc = problem._c()
        _lib.check(L.pr_create_grid(ctypes.byref(pc), device, ctypes.byref(h)))
        self._h = h

    @property
    def handle(self):
        if self._h is None:
            raise PrError(_lib.PR_ESTATE, "grid destroyed")
        return self._h

    def destroy(self):
        if getattr(self, "_h", None) is not None:
            _lib.check(_lib.load().pr_destroy_grid(self._h))
            self._h = None

    def __del__(self):
        try:
            self.destroy()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.destroy()

    # same names as the C ABI --------------------------------------------
    def pr_fine(self, u_in, u_out, step0, n_steps, dt, stream=None):
        return pr_fine(self, u_in, u_out, step0, n_steps, dt, stream)

    def pr_coarse(self, u_in, u_out, step0, n_steps, dt, stream=None):
        return pr_coarse(self, u_in, u_out, step0, n_steps, dt, stream)

    def pr_coarse_mesh(self, u_in, u_out, step0, n_steps, dt, stream=None):
        return pr_coarse_mesh(self, u_in, u_out, step0, n_steps, dt, stream)

    def pr_defect(self, u, u_ref, stream=None):
        return pr_defect(self, u, u_ref, stream)

    def pr_fill_sine(self, u, stream=None):
        return pr_fill_sine(self, u, stream)

    def pr_correct(self, f, g_new, g_old, u_out, u_ref=None, stream=None):
        return pr_correct(self, f, g_new, g_old, u_out, u_ref, stream)

    def pr_parareal(self, cfg, u0, u_T=None, u_ref=None, stream=None):
        return pr_parareal(self, cfg, u0, u_T, u_ref, stream)

    def pr_comm_init(self, world, rank, unique_id: bytes):
        return pr_comm_init(self, world, rank, unique_id)

    def pr_last_timings(self):
        return pr_last_timings(self)


def pr_create_grid(problem: Problem, device: int = 0) -> Grid:
    return Grid(problem, device)


def pr_destroy_grid(grid: Grid) -> None:
    grid.destroy()


def pr_fine(grid, u_in, u_out, step0: int, n_steps: int, dt: float, stream=None) -> None:
    """F (classical RK4) over global steps [step0, step0+n_steps)."""
    _size_check(grid, u_in, u_out)
    _lib.check(_lib.load().pr_fine(grid.handle, _ptr(u_in), _ptr(u_out), int(step0), int(n_steps),
                                   float(dt), _stream(stream, u_in, u_out)))


def pr_coarse(grid, u_in, u_out, step0: int, n_steps: int, dt: float, stream=None) -> None:
    """G (forward Euler, Alg.2) over global steps [step0, step0+n_steps)."""
    _size_check(grid, u_in, u_out)
    _lib.check(_lib.load().pr_coarse(grid.handle, _ptr(u_in), _ptr(u_out), int(step0), int(n_steps),
                                     float(dt), _stream(stream, u_in, u_out)))


def pr_coarse_mesh(grid, u_in, u_out, step0: int, n_steps: int, dt: float, stream=None) -> None:
    """G_c: restriction, Alg.2 on the n/2 mesh, trilinear prolongation (NEXT-4)."""
    _size_check(grid, u_in, u_out)
    _lib.check(_lib.load().pr_coarse_mesh(grid.handle, _ptr(u_in), _ptr(u_out), int(step0),
                                          int(n_steps), float(dt), _stream(stream, u_in, u_out)))


def pr_defect(grid, u, u_ref, stream=None) -> float:
    """Eq.(defect) P:291 (synchronous)."""
    _size_check(grid, u, u_ref)
    d = ctypes.c_double()
    _lib.check(_lib.load().pr_defect(grid.handle, _ptr(u), _ptr(u_ref), ctypes.byref(d),
                                     _stream(stream, u, u_ref)))
    return d.value


def pr_fill_sine(grid, u, stream=None) -> None:
    """u0 = sin(2pi x) sin(2pi y) sin(2pi z)."""
    _size_check(grid, u)
    _lib.check(_lib.load().pr_fill_sine(grid.handle, _ptr(u), _stream(stream, u)))


def pr_correct(grid, f, g_new, g_old, u_out, u_ref=None, stream=None):
    """u_out = f + (g_new - g_old); returns the defect vs u_ref if given."""
    _size_check(grid, f, g_new, g_old, u_out, u_ref)
    d = ctypes.c_double()
    _lib.check(_lib.load().pr_correct(grid.handle, _ptr(f), _ptr(g_new), _ptr(g_old), _ptr(u_out),
                                      _ptr(u_ref), ctypes.byref(d) if u_ref is not None else None,
                                      _stream(stream, f)))
    return d.value if u_ref is not None else None


def pr_nccl_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(PR_NCCL_ID_BYTES)
    _lib.check(_lib.load().pr_nccl_unique_id(buf))
    return buf.raw


def pr_comm_init(grid, world: int, rank: int, unique_id: bytes) -> None:
    if len(unique_id) != PR_NCCL_ID_BYTES:
        raise ValueError("unique id must be 128 bytes")
    buf = ctypes.create_string_buffer(unique_id, PR_NCCL_ID_BYTES)
    _lib.check(_lib.load().pr_comm_init(grid.handle, int(world), int(rank), buf))


def pr_local_group(grids) -> None:
    """Link grids of this process as ranks 0..W-1 of one pipeline (no NCCL); each is
    then driven by its own thread calling pr_parareal (ctypes releases the GIL)."""
    arr = (ctypes.c_void_p * len(grids))(*[g.handle.value for g in grids])
    _lib.check(_lib.load().pr_local_group(arr, len(grids)))


def comm_init_torch(grid) -> None:
    """Bootstrap the library's NCCL communicator from the torch.distributed
    process group (rank 0 creates the id, broadcast_object_list shares it)."""
    import torch.distributed as dist
    world, rank = dist.get_world_size(), dist.get_rank()
    obj = [pr_nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    pr_comm_init(grid, world, rank, obj[0])


def pr_parareal(grid, cfg: PararealCfg, u0, u_T=None, u_ref=None, stream=None):
    """Alg.1 for this rank's slice group (synchronous).  Returns the
    defect history d^0..d^K on the last rank when u_ref is given, else None."""
    _size_check(grid, u0, u_T, u_ref)
    K = cfg.K
    d = (ctypes.c_double * (K + 1))()
    cc = cfg._c()
    _lib.check(_lib.load().pr_parareal(grid.handle, ctypes.byref(cc), _ptr(u0), _ptr(u_T),
                                       _ptr(u_ref), d if u_ref is not None else None,
                                       _stream(stream, u0, u_T, u_ref)))
    return [d[i] for i in range(K + 1)] if (u_ref is not None and u_T is not None) else None


def pr_plan(n_slices: int, K: int, world: int, rank: int) -> list[tuple]:
    """Alg.1 schedule of one rank: list of (op_name, k, slice, peer)."""
    L = _lib.load()
    cnt = ctypes.c_int32()
    _lib.check(L.pr_plan(n_slices, K, world, rank, None, 0, ctypes.byref(cnt)))
    ops = (_lib.PrOp * max(cnt.value, 1))()
    _lib.check(L.pr_plan(n_slices, K, world, rank, ops, cnt.value, ctypes.byref(cnt)))
    return [(OPS[o.op], o.k, o.slice, o.peer) for o in ops[:cnt.value]]


def pr_last_timings(grid) -> dict:
    out = (ctypes.c_double * 5)()
    _lib.check(_lib.load().pr_last_timings(grid.handle, out, 5))
    return dict(zip(["total_ms", "init_ms", "fine_ms", "wait_ms", "coarse_correct_ms"], list(out)))


def pr_grid_info(grid) -> dict:
    info = _lib.PrGridInfo()
    _lib.check(_lib.load().pr_grid_info(grid.handle, ctypes.byref(info)))
    return {f: getattr(info, f) for f, _ in _lib.PrGridInfo._fields_}


def pr_last_monitors(grid) -> tuple[list, int]:
    """(iterate-change monitor per iteration, iterations run) of the last pr_parareal."""
    cap = 4096
    buf = (ctypes.c_double * cap)()
    it = ctypes.c_int32()
    _lib.check(_lib.load().pr_last_monitors(grid.handle, buf, cap, ctypes.byref(it)))
    return [buf[k] for k in range(it.value)], it.value


def pr_kernel_launches() -> int:
    return int(_lib.load().pr_kernel_launches())


def pr_stability_ratio(problem: Problem, dt: float, fine: bool) -> float:
    r = ctypes.c_double()
    pc = problem._c()
    _lib.check(_lib.load().pr_stability_ratio(ctypes.byref(pc), float(dt), 1 if fine else 0, ctypes.byref(r)))
    return r.value


def pr_last_error() -> str:
    return _lib.load().pr_last_error().decode()


def pr_version() -> str:
    return _lib.load().pr_version().decode()
