"""Pins of the oracle's spatially coarsened G (C24-C26):
restriction by injection, periodic trilinear prolongation, and their composition
with Alg.2 on the n/2 mesh.  Each pin is a property the definitions fix, not the
oracle's own code retyped:

* restriction of the paper's initial value is the initial value of the n/2 mesh;
* R o P = identity (bitwise: even fine points carry the coarse values);
* P reproduces constants and, away from the periodic seam, linear functions
  (bitwise: integer data, power-of-two weights);
* P of a Fourier mode is the closed form e^{i th x/2} (1 or cos(th/2) per axis);
* G_c on the sine initial value equals the exact per-mode Euler recurrence on
  the n/2 mesh (tests/modal_ref.py), prolongated by that closed form.
"""
import numpy as np
import pytest

import oracle
from synthetic import random_field
from modal_ref import ModalSolver, sine_modes


@pytest.mark.parametrize("n", [8, 16, 32])
def test_restrict_initial_value(n):
    assert np.max(np.abs(oracle.restrict(oracle.initial(n)) - oracle.initial(n // 2))) <= 1e-15


@pytest.mark.parametrize("m", [4, 6, 8])
def test_restrict_prolong_identity_and_constants(m):
    v = random_field(m, 5)
    assert np.array_equal(oracle.restrict(oracle.prolong(v)), v)
    c = np.full((m, m, m), 0.375)
    assert np.array_equal(oracle.prolong(c), np.full((2 * m,) * 3, 0.375))


@pytest.mark.parametrize("axis", [0, 1, 2])
def test_prolong_linear_exact_off_seam(axis):
    """Data linear along one axis (arrays are (z, y, x)): odd fine points are the
    midpoints; at the last odd point the partner is the periodic image, index 0."""
    m = 6
    shape = [1, 1, 1]
    shape[axis] = m
    vc = np.broadcast_to(np.arange(m, dtype=np.float64).reshape(shape) * 3.0 + 1.0, (m, m, m)).copy()
    u = oracle.prolong(vc)
    X = np.arange(2 * m)
    line = np.where(X % 2 == 0, 3.0 * (X // 2) + 1.0, 3.0 * (X // 2) + 2.5)  # midpoints
    line[-1] = ((3.0 * (m - 1) + 1.0) + 1.0) / 2  # seam: mean of coarse m-1 and 0
    full = [1, 1, 1]
    full[axis] = 2 * m
    assert np.array_equal(u, np.broadcast_to(line.reshape(full), u.shape))


def _prolonged_mode(n, th_c):
    """Closed form of P applied to the coarse wave e^{i th_c I} (I = coarse index):
    at fine index x the value e^{i th_c x/2}, times cos(th_c/2) when x is odd."""
    x = np.arange(n)
    return np.exp(1j * th_c * x / 2) * np.where(x % 2 == 1, np.cos(th_c / 2), 1.0)


def test_prolong_fourier_mode_closed_form():
    n, m = 16, 8
    th = 2 * np.pi * 3 / m
    zc = np.arange(m)
    vc = np.real(np.exp(1j * th * zc))[:, None, None] * np.ones((m, m, m))  # wave along z
    u = oracle.prolong(np.ascontiguousarray(vc))
    exact = np.real(_prolonged_mode(n, th))[:, None, None] * np.ones((n, n, n))
    assert np.max(np.abs(u - exact)) <= 1e-15


@pytest.mark.parametrize("c", [(1.0, 1.0, 1.0), (-1.0, 0.5, 0.0)])
def test_coarse_mesh_vs_modal(c):
    n, m = 32, 16
    p = oracle.Problem(n, c=c)
    Dt, step0, steps = 2e-4, 5, 40
    got = oracle.coarse_mesh(p, oracle.initial(n), step0, steps, Dt)
    th, coef = sine_modes(m)
    z = ModalSolver(m, c=c, thetas=th).coarse(coef, step0, steps, Dt)
    exact = np.zeros((n, n, n))
    for t, a in zip(th, z):
        wx, wy, wz = (_prolonged_mode(n, t[d]) for d in range(3))
        exact += np.real(a * wz[:, None, None] * wy[None, :, None] * wx[None, None, :])
    assert np.max(np.abs(got - exact)) / np.max(np.abs(exact)) <= 1e-13


def test_parareal_with_coarse_mesh_exactness():
    """K = N_p: Parareal reproduces the serial fine solution whatever G is,
    here with G_c; K = 0 is the serial G_c sweep."""
    n, Np, nc, nf = 8, 4, 4, 8
    p = oracle.Problem(n, T=0.002)
    u0 = random_field(n, 9)
    uf = oracle.serial_fine(p, Np * nf, u0)
    res = oracle.parareal(p, Np, nc, nf, Np, u0, uf, g_half_mesh=True)
    assert np.max(np.abs(res.u_T - uf)) <= 1e-14 * np.max(np.abs(uf))
    res0 = oracle.parareal(p, Np, nc, nf, 0, u0, uf, g_half_mesh=True)
    v = u0
    for s in range(Np):
        v = oracle.coarse_mesh(p, v, s * nc, nc, p.T / (Np * nc))
    assert np.array_equal(res0.u_T, v)
    # the coarse-mesh G is a different G: its iterates differ from the default ones
    assert not np.array_equal(oracle.parareal(p, Np, nc, nf, 1, u0, uf).u_T,
                              oracle.parareal(p, Np, nc, nf, 1, u0, uf, g_half_mesh=True).u_T)
