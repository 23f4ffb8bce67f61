"""Pins for the oracle's spatial operators and single steps (CPU only).

Each test checks the oracle against something other than itself: closed-form
Fourier symbols, hand-computed spikes, polynomial
exactness, conservation/linearity/equivariance, and a dense 8^3 brute force
built from the printed weights as Kronecker sums of 1D circulant matrices.
"""
import numpy as np
import pytest

from modal_ref import Symbols
from synthetic import random_field, PARITY_C

C = PARITY_C


def mode_field(n, m, kind):
    """cos or sin of theta . (i, j, k), theta = 2 pi m / n, shape (z, y, x)."""
    idx = np.arange(n)
    ph = (2 * np.pi * m[2] / n) * idx[:, None, None] + (2 * np.pi * m[1] / n) * idx[None, :, None] \
        + (2 * np.pi * m[0] / n) * idx[None, None, :]
    return np.cos(ph) if kind == "cos" else np.sin(ph), ph


@pytest.mark.parametrize("n", [8, 12, 16])
@pytest.mark.parametrize("m", [(1, 0, 0), (0, 2, 0), (1, 1, 3), (3, -2, 1)])
def test_rhs_symbols(orc, n, m):
    """L e^{i th.j} = lambda(th) e^{i th.j}: real/imag parts on cos/sin modes."""
    nu = 0.15
    th = np.array([2 * np.pi * v / n for v in m])
    sym = Symbols(n, C, th[None, :])
    for name, fn, lam in (("coarse", orc.rhs_coarse, sym.lam_G(nu)[0]),
                          ("fine", orc.rhs_fine, sym.lam_F(nu)[0])):
        ucos, ph = mode_field(n, m, "cos")
        usin, _ = mode_field(n, m, "sin")
        # cos = Re e^{i ph}; L cos = Re(lam e^{i ph}) = Re(lam) cos - Im(lam) sin
        exp_cos = lam.real * np.cos(ph) - lam.imag * np.sin(ph)
        exp_sin = lam.real * np.sin(ph) + lam.imag * np.cos(ph)
        scale = abs(lam) + 1.0
        assert np.max(np.abs(fn(ucos, C, nu) - exp_cos)) <= 1e-12 * scale, name
        assert np.max(np.abs(fn(usin, C, nu) - exp_sin)) <= 1e-12 * scale, name


def test_coarse_spike_hand_values(orc):
    """c=0, unit spike: rhs(centre) = -6 nu/dx^2, faces nu/dx^2."""
    n = 8
    u = np.zeros((n, n, n)); u[3, 4, 5] = 1.0
    r = orc.rhs_coarse(u, (0.0, 0.0, 0.0), 1.0)
    inv = n * n  # 1/dx^2
    assert r[3, 4, 5] == -6.0 * inv
    for dz, dy, dx in [(1, 0, 0), (-1, 0, 0), (0, 1, 0), (0, -1, 0), (0, 0, 1), (0, 0, -1)]:
        assert r[3 + dz, 4 + dy, 5 + dx] == inv
    assert np.count_nonzero(r) == 7


def test_euler_step_hand_values(orc):
    """one Euler step, nu=1, c=0: centre 1 - 6 nu Dt/dx^2, faces nu Dt/dx^2.
    With n=8 (dx^2 = 1/64) and Dt = 0.1/64 this is the 0.4 / 0.1 example."""
    n = 8
    u = np.zeros((n, n, n)); u[0, 0, 0] = 1.0
    p = orc.Problem(n, c=(0.0, 0.0, 0.0), nu0=1.0, omega=0.0)
    v = orc.coarse(p, u, 0, 1, 0.1 / 64)
    assert abs(v[0, 0, 0] - 0.4) < 1e-15
    # periodic wrap: the face neighbours of (0,0,0) include index n-1
    for pos in [(1, 0, 0), (n - 1, 0, 0), (0, 1, 0), (0, n - 1, 0), (0, 0, 1), (0, 0, n - 1)]:
        assert abs(v[pos] - 0.1) < 1e-15


@pytest.mark.parametrize("sign", [1.0, -1.0])
def test_upwind_branch(orc, sign):
    """Alg.2: c_x > 0 -> backward difference, else forward."""
    n = 8
    u = np.zeros((n, n, n)); u[2, 2, 4] = 1.0
    r = orc.rhs_coarse(u, (sign, 0.0, 0.0), 0.0)
    if sign > 0:   # rhs_i = -c (u_i - u_{i-1})/dx : nonzero at i=4 (-c/dx) and i=5 (+c/dx)
        assert r[2, 2, 4] == -sign * n and r[2, 2, 5] == sign * n and r[2, 2, 3] == 0
    else:          # rhs_i = -c (u_{i+1} - u_i)/dx : nonzero at i=4 (+c/dx) and i=3 (-c/dx)
        assert r[2, 2, 4] == sign * n and r[2, 2, 3] == -sign * n and r[2, 2, 5] == 0
    # c = 0: both branches give zero (C4)
    assert np.all(orc.rhs_coarse(u, (0.0, 0.0, 0.0), 0.0) == 0)


def test_lap4_quadratic_exact(orc):
    """Fourth-order second derivative is exact on quadratics:
    u = (i dx)^2 along x, interior points away from the periodic wrap."""
    n = 16
    dx = 1.0 / n
    x = np.arange(n) * dx
    u = np.broadcast_to((x ** 2)[None, None, :], (n, n, n)).copy()
    r = orc.rhs_fine(u, (0.0, 0.0, 0.0), 1.0)
    assert np.max(np.abs(r[:, :, 2:n - 2] - 2.0)) < 1e-9
    # D1 is exact on cubics: u = x^3, nu = 0, c = (1,0,0) -> rhs = -3x^2
    u3 = np.broadcast_to((x ** 3)[None, None, :], (n, n, n)).copy()
    r3 = orc.rhs_fine(u3, (1.0, 0.0, 0.0), 0.0)
    assert np.max(np.abs(r3[:, :, 2:n - 2] + 3 * x[2:n - 2] ** 2)) < 1e-11


@pytest.mark.parametrize("which", ["coarse", "fine"])
def test_rhs_properties(orc, which):
    """Mean conservation, linearity, periodic shift equivariance."""
    fn = orc.rhs_coarse if which == "coarse" else orc.rhs_fine
    n = 12
    u, v = random_field(n, 0), random_field(n, 1)
    nu = 0.1
    ru = fn(u, C, nu)
    scale = np.max(np.abs(ru))
    assert abs(ru.mean()) <= 1e-13 * scale
    lin = fn(2.0 * u - 0.5 * v, C, nu) - (2.0 * ru - 0.5 * fn(v, C, nu))
    assert np.max(np.abs(lin)) <= 1e-13 * scale
    for axis in range(3):
        sh = fn(np.roll(u, 3, axis=axis), C, nu)
        assert np.array_equal(sh, np.roll(ru, 3, axis=axis))


def circulant(n, weights):
    """Dense n x n periodic operator: (M u)_i = sum_o w_o u_{i+o}."""
    M = np.zeros((n, n))
    for off, w in weights.items():
        for i in range(n):
            M[i, (i + off) % n] += w
    return M


def dense_ops(n, c, fine):
    """Kronecker-sum 3D operators from the printed 1D weights; field index
    q = (z n + y) n + x, so x is the fastest (rightmost) Kronecker factor."""
    dx = 1.0 / n
    I = np.eye(n)
    if fine:
        lap1 = circulant(n, {-2: -1, -1: 16, 0: -30, 1: 16, 2: -1}) / (12 * dx * dx)
        adv1 = [circulant(n, {-2: 1, -1: -8, 1: 8, 2: -1}) / (12 * dx) for _ in range(3)]
    else:
        lap1 = circulant(n, {-1: 1, 0: -2, 1: 1}) / (dx * dx)
        adv1 = [circulant(n, {0: 1, -1: -1}) / dx if c[a] > 0 else circulant(n, {1: 1, 0: -1}) / dx
                for a in range(3)]

    def k3(Az, Ay, Ax):
        return np.kron(Az, np.kron(Ay, Ax))

    L = k3(I, I, lap1) + k3(I, lap1, I) + k3(lap1, I, I)
    B = c[0] * k3(I, I, adv1[0]) + c[1] * k3(I, adv1[1], I) + c[2] * k3(adv1[2], I, I)
    return L, B


@pytest.mark.parametrize("fine", [False, True])
def test_rhs_dense_bruteforce_8(orc, fine):
    n = 8
    L, B = dense_ops(n, C, fine)
    u = random_field(n, 2)
    nu = 0.13
    ref = (nu * (L @ u.ravel()) - B @ u.ravel()).reshape(n, n, n)
    got = (orc.rhs_fine if fine else orc.rhs_coarse)(u, C, nu)
    assert np.max(np.abs(got - ref)) <= 1e-13 * np.max(np.abs(ref))


def test_propagators_dense_bruteforce_8(orc):
    """G = Euler (Alg.2) and F = classical RK4 by dense mat-vecs."""
    n = 8
    Lg, Bg = dense_ops(n, C, False)
    Lf, Bf = dense_ops(n, C, True)
    for nu_mode in (0, 1):
        p = orc.Problem(n, c=C, nu0=0.1, omega=100.0, nu_mode=nu_mode)
        u = random_field(n, 3).ravel()
        dt, Dt = 1e-4, 4e-4
        # G over global steps [5, 12)
        g = u.copy()
        for j in range(5, 12):
            nuj = 0.1 + 0.05 * np.sin(100.0 * j * Dt)
            g = g + Dt * (nuj * (Lg @ g) - Bg @ g)
        got = orc.coarse(p, u.reshape(n, n, n), 5, 7, Dt).ravel()
        assert np.max(np.abs(got - g)) <= 1e-13 * np.max(np.abs(g))
        # F over global steps [3, 9)
        f = u.copy()

        def rhs(y, t):
            nut = 0.1 + 0.05 * np.sin(100.0 * t)
            return nut * (Lf @ y) - Bf @ y
        for j in range(3, 9):
            t1, t2, t4 = j * dt, (j + 0.5) * dt, (j + 1.0) * dt
            if nu_mode == 1:
                t2 = t4 = t1
            k1 = rhs(f, t1)
            k2 = rhs(f + dt / 2 * k1, t2)
            k3 = rhs(f + dt / 2 * k2, t2)
            k4 = rhs(f + dt * k3, t4)
            f = f + dt / 6 * (k1 + 2 * k2 + 2 * k3 + k4)
        got = orc.fine(p, u.reshape(n, n, n), 3, 6, dt).ravel()
        assert np.max(np.abs(got - f)) <= 1e-13 * np.max(np.abs(f))


def test_nu_profile_and_amplitude(orc):
    """P:437 nu(t); a(t) (exp restored per C18) vs a tiny-step RK4
    integration of a' = -12 pi^2 nu(t) a to 1e-10."""
    assert orc.nu(0.1, 100.0, 0.0) == 0.1
    assert abs(orc.nu(0.1, 100.0, np.pi / 200) - 0.15) < 1e-15
    assert orc.nu(0.1, 0.0, 0.7) == 0.1
    for omega in (0.0, 100.0):
        a, t, h = 1.0, 0.0, 1e-5

        def f(t, a):
            return -12 * np.pi ** 2 * (0.1 + 0.05 * np.sin(omega * t)) * a
        for _ in range(10000):
            k1 = f(t, a); k2 = f(t + h / 2, a + h / 2 * k1)
            k3 = f(t + h / 2, a + h / 2 * k2); k4 = f(t + h, a + h * k3)
            a += h / 6 * (k1 + 2 * k2 + 2 * k3 + k4); t += h
        assert abs(orc.amplitude(0.1, omega, 0.1) - a) <= 1e-10 * a
    assert orc.amplitude(0.1, 100.0, 0.0) == 1.0


def test_initial_and_exact(orc):
    """P:418-420 and P:444-446; SPEC S:253-282 examples."""
    n = 16
    u0 = orc.initial(n)
    assert np.all(u0[:, :, 0] == 0.0)                      # sin(0) = 0
    assert abs(u0[n // 4, n // 4, n // 4] - 1.0) < 1e-15   # sin(pi/2)^3
    assert abs(orc.inf_norm(u0) - 1.0) < 1e-15
    p = orc.Problem(n)
    assert np.max(np.abs(orc.exact(p, 0.0) - u0)) < 1e-15
    # c = (1,1,1), t = 1: a full period shift -> a(1) u0
    assert np.max(np.abs(orc.exact(p, 1.0) - orc.amplitude(0.1, 100.0, 1.0) * u0)) < 1e-12
    # nu0 -> 0, c = (1,0,0), t = 1/4: pure advection by a quarter period
    p2 = orc.Problem(n, c=(1.0, 0.0, 0.0), nu0=0.0)
    assert np.max(np.abs(orc.exact(p2, 0.25) - np.roll(u0, n // 4, axis=2))) < 1e-12


def test_inf_norm_and_defect(orc):
    n = 8
    u = np.zeros((n, n, n)); u[1, 2, 3] = -7.5
    assert orc.inf_norm(u) == 7.5
    ref = random_field(n, 4)
    assert orc.defect(ref, ref) == 0.0
    assert abs(orc.defect(1.5 * ref, ref) - 0.5) < 1e-15
    u[0, 0, 0] = np.nan
    assert np.isnan(orc.inf_norm(u))
