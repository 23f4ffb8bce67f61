"""Pins for the oracle's propagators F, G and its Parareal emulation (CPU only).

Pinned by: the exact per-mode discrete recurrence (tests/modal_ref.py), the
paper's printed accuracy numbers (tests/golden/paper_accuracy.json; P:456,
P:458), the semi-discrete exact solution (temporal order), the closed-form
solution (spatial order), Parareal finite-step exactness, the
degenerate G = F case, the error bound of P:296, and a dense 8^3
brute-force Parareal written from Eq.(parareal).
"""
import json
import os

import numpy as np
import pytest

import modal_ref as M
from synthetic import CONFIGS, random_field, PARITY_C
from test_oracle_operators import dense_ops

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def cfg1_problem(orc, nu_mode=0, omega=100.0):
    c = CONFIGS["cfg1"]
    return c, orc.Problem(c.n, c=c.c, nu0=c.nu0, omega=omega, T=c.T, nu_mode=nu_mode)


@pytest.fixture(scope="module")
def cfg1_runs(orc):
    """Oracle serial fine + Parareal for cfg1 (32^3, 4 slices, K=2), both nu modes."""
    out = {}
    for nu_mode in (0, 1):
        c, p = cfg1_problem(orc, nu_mode)
        u0 = orc.initial(c.n)
        uf = orc.serial_fine(p, c.Nt, u0)
        res = orc.parareal(p, c.slices, c.nc, c.nf, c.K, u0, uf)
        out[nu_mode] = (c, p, u0, uf, res)
    return out


def modal_fields(c, nu_mode, omega=100.0):
    thetas, coef = M.sine_modes(c.n)
    ms = M.ModalSolver(c.n, c.c, c.nu0, omega, nu_mode, thetas)
    zf = ms.fine(coef, 0, c.Nt, c.T / c.Nt)
    zT, hist = ms.parareal(coef, c.slices, c.nc, c.nf, c.K, c.T)
    uf = M.synthesize(c.n, thetas, zf)
    return uf, M.synthesize(c.n, thetas, zT), [M.synthesize(c.n, thetas, h) for h in hist]


@pytest.mark.parametrize("nu_mode", [0, 1])
def test_cfg1_vs_modal_recurrence(orc, cfg1_runs, nu_mode):
    c, p, u0, uf, res = cfg1_runs[nu_mode]
    thetas, coef = M.sine_modes(c.n)
    assert np.max(np.abs(u0 - M.synthesize(c.n, thetas, coef))) < 1e-15
    uf_m, uT_m, hist = modal_fields(c, nu_mode)
    scale = np.max(np.abs(uf_m))
    assert np.max(np.abs(uf - uf_m)) <= 1e-13 * scale
    assert np.max(np.abs(res.u_T - uT_m)) <= 1e-13 * scale
    d_modal = [np.max(np.abs(h - uf_m)) / scale for h in hist]
    assert np.max(np.abs(res.defects - np.array(d_modal))) <= 1e-13
    # rapid, monotone convergence
    assert res.defects[0] > res.defects[1] > res.defects[2] > 0


def test_paper_printed_accuracy(orc):
    """P:456 / P:458 at the paper's 128^3, dt = T/2^15, Dt = T/2^11, evaluated
    with the exact discrete modal recurrence (validated against the oracle at
    32^3 above and at 8^3 by brute force).  Printed values have 2 significant
    digits; the reading C1 = step_start is the only one that reproduces 4.8e-6."""
    g = json.load(open(os.path.join(GOLDEN, "paper_accuracy.json")))
    n, T = 128, 0.1
    thetas, coef = M.sine_modes(n)

    def eps(omega, nu_mode, fine):
        ms = M.ModalSolver(n, (1.0, 1.0, 1.0), 0.1, omega, nu_mode, thetas)
        z = ms.fine(coef, 0, 2 ** 15, T / 2 ** 15) if fine else ms.coarse(coef, 0, 2 ** 11, T / 2 ** 11)
        u = M.synthesize(n, thetas, z)
        ex = M.exact_solution(n, (1.0, 1.0, 1.0), 0.1, omega, T)
        return np.max(np.abs(u - ex)) / np.max(np.abs(ex))

    def sig2(x):
        return float(f"{x:.1e}")

    assert sig2(eps(0.0, 1, True)) == g["eps_fine_omega0"]["value"]
    assert sig2(eps(0.0, 0, True)) == g["eps_fine_omega0"]["value"]
    assert sig2(eps(100.0, 1, True)) == g["eps_fine_omega100"]["value"]
    assert sig2(eps(100.0, 0, True)) != g["eps_fine_omega100"]["value"]  # C1
    assert sig2(eps(0.0, 0, False)) == g["eps_coarse"]["value"]
    assert sig2(eps(100.0, 0, False)) == g["eps_coarse"]["value"]


@pytest.mark.parametrize("nu_mode,expected", [(0, 4.0), (1, 1.0)])
def test_fine_temporal_order(orc, nu_mode, expected):
    """Oracle F vs the semi-discrete exact solution at n=8: RK4 with stage-time
    nu is 4th order; nu frozen at the step start is 1st order when omega != 0."""
    n, T = 8, 0.02
    p = orc.Problem(n, nu_mode=nu_mode, T=T)
    thetas, coef = M.sine_modes(n)
    ms = M.ModalSolver(n, (1.0, 1.0, 1.0), 0.1, 100.0, nu_mode, thetas)
    ex = M.synthesize(n, thetas, ms.semidiscrete_exact(coef, T))
    errs = []
    for N in (16, 32, 64):
        u = orc.fine(p, orc.initial(n), 0, N, T / N)
        errs.append(np.max(np.abs(u - ex)))
    orders = np.log2(np.array(errs[:-1]) / np.array(errs[1:]))
    assert np.all(np.abs(orders - expected) < 0.3), orders


def test_coarse_temporal_order(orc):
    n, T = 8, 0.02
    p = orc.Problem(n, T=T)
    thetas, coef = M.sine_modes(n)
    ms = M.ModalSolver(n, (1.0, 1.0, 1.0), 0.1, 100.0, 0, thetas)
    ex = M.synthesize(n, thetas, ms.semidiscrete_exact(coef, T, fine=False))
    errs = [np.max(np.abs(orc.coarse(p, orc.initial(n), 0, N, T / N) - ex)) for N in (32, 64, 128)]
    orders = np.log2(np.array(errs[:-1]) / np.array(errs[1:]))
    assert np.all(np.abs(orders - 1.0) < 0.15), orders


def test_fine_spatial_order(orc):
    """Against the closed form: error ratio 16 per grid doubling (4th order)."""
    T, errs = 0.002, []
    for n in (16, 32):
        p = orc.Problem(n, omega=0.0, T=T)
        u = orc.fine(p, orc.initial(n), 0, 8, T / 8)
        ex = M.exact_solution(n, (1.0, 1.0, 1.0), 0.1, 0.0, T)
        errs.append(np.max(np.abs(u - ex)) / np.max(np.abs(ex)))
    assert 3.7 <= np.log2(errs[0] / errs[1]) <= 4.3


def test_coarse_spatial_order(orc):
    """Upwind (1st order) dominates the coarse spatial error."""
    T, errs = 0.002, []
    for n in (16, 32):
        p = orc.Problem(n, omega=0.0, T=T)
        u = orc.coarse(p, orc.initial(n), 0, 64, T / 64)
        ex = M.exact_solution(n, (1.0, 1.0, 1.0), 0.1, 0.0, T)
        errs.append(np.max(np.abs(u - ex)) / np.max(np.abs(ex)))
    assert 0.8 <= np.log2(errs[0] / errs[1]) <= 1.3


def test_slicewise_fine_equals_serial(orc):
    """C6/C7: F over N_p slices with global step indices == one F call, bitwise."""
    n = 8
    p = orc.Problem(n, c=PARITY_C)
    u0 = random_field(n, 5)
    a = orc.fine(p, u0, 0, 40, 1e-4)
    b = u0
    for m in range(4):
        b = orc.fine(p, b, 10 * m, 10, 1e-4)
    assert np.array_equal(a, b)


@pytest.mark.parametrize("Np", [1, 2, 3, 4])
def test_parareal_exactness(orc, Np):
    """K = N_p reproduces the serial fine solution; bitwise with C5+C6."""
    n = 8
    p = orc.Problem(n, c=PARITY_C, T=0.004)
    u0 = random_field(n, 6)
    nf, nc = 8, 2
    uf = orc.serial_fine(p, Np * nf, u0)
    res = orc.parareal(p, Np, nc, nf, Np, u0, uf)
    assert np.array_equal(res.u_T, uf)
    assert res.defects[Np] == 0.0


def test_parareal_g_equals_f(orc):
    """Degenerate G = F: d^1 = 0."""
    n = 8
    p = orc.Problem(n, c=PARITY_C, T=0.004)
    u0 = random_field(n, 7)
    uf = orc.serial_fine(p, 4 * 6, u0)
    res = orc.parareal(p, 4, 2, 6, 2, u0, uf, g_is_f=True)
    assert res.defects[1] == 0.0 and res.defects[2] == 0.0


def test_parareal_k0_is_coarse(orc):
    n = 8
    p = orc.Problem(n, c=PARITY_C, T=0.004)
    u0 = random_field(n, 8)
    res = orc.parareal(p, 3, 2, 6, 0, u0)
    assert np.array_equal(res.u_T, orc.coarse(p, u0, 0, 6, 0.004 / 6))


def test_parareal_dense_bruteforce_8(orc):
    """Eq.(parareal) P:142 written with dense operators at 8^3 (independent of
    the oracle's loops and of its rank-by-rank Alg.1 layout)."""
    n, Np, nc, nf, K, T = 8, 4, 3, 12, 2, 0.006
    c = PARITY_C
    Lg, Bg = dense_ops(n, c, False)
    Lf, Bf = dense_ops(n, c, True)
    nuf = lambda t: 0.1 + 0.05 * np.sin(100.0 * t)
    Dt, dt = T / (Np * nc), T / (Np * nf)

    def G(u, m):
        for j in range(m * nc, (m + 1) * nc):
            u = u + Dt * (nuf(j * Dt) * (Lg @ u) - Bg @ u)
        return u

    def F(u, m):
        f = lambda y, t: nuf(t) * (Lf @ y) - Bf @ y
        for j in range(m * nf, (m + 1) * nf):
            k1 = f(u, j * dt); k2 = f(u + dt / 2 * k1, (j + .5) * dt)
            k3 = f(u + dt / 2 * k2, (j + .5) * dt); k4 = f(u + dt * k3, (j + 1) * dt)
            u = u + dt / 6 * (k1 + 2 * k2 + 2 * k3 + k4)
        return u

    u0 = random_field(n, 9).ravel()
    U = [u0]
    for m in range(Np):
        U.append(G(U[m], m))
    for _ in range(K):
        V = [u0]
        for m in range(Np):
            V.append(G(V[m], m) + F(U[m], m) - G(U[m], m))
        U = V
    p = orc.Problem(n, c=c, T=T)
    res = orc.parareal(p, Np, nc, nf, K, u0.reshape(n, n, n))
    assert np.max(np.abs(res.u_T.ravel() - U[Np])) <= 1e-13 * np.max(np.abs(U[Np]))


def test_error_bound(orc, cfg1_runs):
    """eps_parareal <= d^k ||u_fine|| / ||u_exact|| + eps_fine."""
    c, p, u0, uf, res = cfg1_runs[0]
    ex = M.exact_solution(c.n, c.c, c.nu0, 100.0, c.T)
    nex = np.max(np.abs(ex))
    eps_fine = np.max(np.abs(uf - ex)) / nex
    eps_par = np.max(np.abs(res.u_T - ex)) / nex
    assert eps_par <= res.defects[-1] * np.max(np.abs(uf)) / nex + eps_fine + 1e-15
