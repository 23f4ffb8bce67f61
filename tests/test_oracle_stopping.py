"""Pins for the oracle's convergence-controlled stopping (C23; P:153,
P:301-302): tol <= 0 is exactly the fixed-K algorithm, one rank stops at the
first iteration whose iterate change is below tol and then equals the fixed-K
result for that K, and the monitor equals the difference of two fixed-K runs."""
import numpy as np
import pytest

from synthetic import random_field, PARITY_C


def setup(orc, n=8, Np=4, nf=6, nc=2, T=0.004, seed=21):
    p = orc.Problem(n, c=PARITY_C, T=T)
    u0 = random_field(n, seed)
    uf = orc.serial_fine(p, Np * nf, u0)
    return p, u0, uf


@pytest.mark.parametrize("world", [1, 2, 4])
def test_tol_zero_is_fixed_K(orc, world):
    p, u0, uf = setup(orc)
    a = orc.parareal(p, 4, 2, 6, 3, u0, uf)
    b = orc.parareal_tol(p, 4, 2, 6, 3, 0.0, world, u0, uf)
    assert np.array_equal(a.u_T, b.u_T) and np.array_equal(a.defects, b.defects)
    assert list(b.iters) == [3] * world


def test_single_rank_stops_at_first_small_change(orc):
    p, u0, uf = setup(orc)
    full = orc.parareal_tol(p, 4, 2, 6, 4, 0.0, 1, u0, uf)
    ch = full.changes[0]
    assert np.all(np.diff(ch) < 0)          # rapid convergence
    tol = 0.5 * (ch[1] + ch[2])             # between iterations 2 and 3
    r = orc.parareal_tol(p, 4, 2, 6, 4, tol, 1, u0, uf)
    assert r.iters[0] == 3
    ref = orc.parareal(p, 4, 2, 6, 3, u0, uf)
    assert np.array_equal(r.u_T, ref.u_T)
    assert np.array_equal(r.defects[:4], ref.defects) and np.isnan(r.defects[4])
    huge = orc.parareal_tol(p, 4, 2, 6, 4, 1e300, 1, u0, uf)
    assert huge.iters[0] == 1 and np.array_equal(huge.u_T, orc.parareal(p, 4, 2, 6, 1, u0, uf).u_T)


def test_monitor_is_iterate_difference(orc):
    """With one slice per rank the last rank's monitor is
    ||u^{k+1}_{Np} - u^k_{Np}|| / ||u^{k+1}_{Np}||, computed from fixed-K runs."""
    p, u0, uf = setup(orc)
    r = orc.parareal_tol(p, 4, 2, 6, 3, 0.0, 4, u0, uf)
    prev = orc.parareal(p, 4, 2, 6, 0, u0).u_T
    for k in range(3):
        cur = orc.parareal(p, 4, 2, 6, k + 1, u0).u_T
        exp = np.max(np.abs(cur - prev)) / np.max(np.abs(cur))
        assert r.changes[3, k] == pytest.approx(exp, rel=1e-14, abs=0)
        prev = cur


def test_pipeline_stop_order(orc):
    """A rank never stops before its predecessor; the final defect is of the
    order of the tolerance."""
    p, u0, uf = setup(orc, Np=8, nf=4, nc=1, T=0.004)
    tol = 1e-6
    r = orc.parareal_tol(p, 8, 1, 4, 8, tol, 8, u0, uf)
    assert np.all(np.diff(r.iters) >= 0) and r.iters[-1] <= 8
    last = r.iters[-1]
    assert r.defects[last] < 1e3 * tol
