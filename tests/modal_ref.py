"""Exact discrete Fourier-mode reference (test infrastructure; independent of
both the C oracle and the CUDA path).

Every operator on the hot path is linear, periodic and constant-coefficient in
space, so the discrete Fourier modes e^{i theta . j} (theta_a = 2 pi m_a / n)
are eigenvectors of all of them.  The eigenvalues (symbols) below follow from
applying each printed stencil to e^{i theta j}:

  7-point Laplacian (Alg.2):    sum_a (2 cos th_a - 2) / dx^2
  upwind, c_a > 0 (Alg.2):  (1 - e^{-i th_a}) / dx
  upwind, c_a <= 0:        (e^{+i th_a} - 1) / dx
  4th-order Laplacian (C3):            sum_a (-2 cos 2th_a + 32 cos th_a - 30) / (12 dx^2)
  4th-order first derivative (C3):     i (8 sin th_a - sin 2 th_a) / (6 dx)

lambda_G(nu) = nu * Lap2 - sum_a c_a Up_a,  lambda_F(nu) = nu * Lap4 - sum_a c_a D1_a.
A forward-Euler step multiplies a mode by 1 + Dt lambda_G(nu_j); a classical RK4
step applies the four stages to the scalar.  Parareal (Eq.(parareal) P:142,
Alg.1) is then the same recurrence on complex scalars, per mode.

The semi-discrete exact solution (exact in time, discrete in space) is
z(t) = exp(Lap * int_0^t nu - B t) z(0), because nu(t) only scales the
commuting part Lap; it pins the temporal order of accuracy.
"""
from __future__ import annotations

import numpy as np


class Symbols:
    def __init__(self, n: int, c, thetas: np.ndarray):
        """thetas: (..., 3) array of per-axis angles (x, y, z)."""
        self.n = n
        self.dx = 1.0 / n
        th = np.asarray(thetas, dtype=np.float64)
        dx = self.dx
        c = [float(v) for v in c]
        self.lap2 = np.sum((2.0 * np.cos(th) - 2.0) / dx ** 2, axis=-1).astype(complex)
        self.lap4 = np.sum((-2.0 * np.cos(2 * th) + 32.0 * np.cos(th) - 30.0)
                           / (12.0 * dx ** 2), axis=-1).astype(complex)
        up = np.zeros(th.shape[:-1], dtype=complex)
        d1 = np.zeros(th.shape[:-1], dtype=complex)
        for a in range(3):
            t = th[..., a]
            if c[a] > 0:
                up += c[a] * (1.0 - np.exp(-1j * t)) / dx
            else:
                up += c[a] * (np.exp(1j * t) - 1.0) / dx
            d1 += c[a] * 1j * (8.0 * np.sin(t) - np.sin(2 * t)) / (6.0 * dx)
        self.bG = up
        self.bF = d1

    def lam_G(self, nu):
        return nu * self.lap2 - self.bG

    def lam_F(self, nu):
        return nu * self.lap4 - self.bF


def nu_of(nu0, omega, t):
    return nu0 + (nu0 / 2.0) * np.sin(omega * t)


def nu_integral(nu0, omega, t):
    if omega == 0.0:
        return nu0 * t
    return nu0 * t + nu0 / (2.0 * omega) * (1.0 - np.cos(omega * t))


class ModalSolver:
    """Per-mode exact discrete propagators for a fixed problem."""

    def __init__(self, n, c=(1.0, 1.0, 1.0), nu0=0.1, omega=100.0, nu_mode=0,
                 thetas=None):
        self.n, self.c, self.nu0, self.omega, self.nu_mode = n, c, nu0, omega, nu_mode
        if thetas is None:
            thetas = sine_modes(n)[0]
        self.thetas = np.asarray(thetas)
        self.sym = Symbols(n, c, self.thetas)

    def nu(self, t):
        return nu_of(self.nu0, self.omega, t)

    def coarse(self, z, step0, n_steps, dt):
        z = np.array(z, dtype=complex, copy=True)
        for j in range(step0, step0 + n_steps):
            z = z + dt * (self.sym.lam_G(self.nu(j * dt)) * z)
        return z

    def fine(self, z, step0, n_steps, dt):
        z = np.array(z, dtype=complex, copy=True)
        for j in range(step0, step0 + n_steps):
            if self.nu_mode == 1:
                l1 = l2 = l4 = self.sym.lam_F(self.nu(j * dt))
            else:
                l1 = self.sym.lam_F(self.nu(j * dt))
                l2 = self.sym.lam_F(self.nu((j + 0.5) * dt))
                l4 = self.sym.lam_F(self.nu((j + 1.0) * dt))
            k1 = l1 * z
            k2 = l2 * (z + dt / 2 * k1)
            k3 = l2 * (z + dt / 2 * k2)
            k4 = l4 * (z + dt * k3)
            z = z + dt / 6 * (k1 + 2 * k2 + 2 * k3 + k4)
        return z

    def semidiscrete_exact(self, z, t, fine=True):
        lap = self.sym.lap4 if fine else self.sym.lap2
        b = self.sym.bF if fine else self.sym.bG
        return z * np.exp(lap * nu_integral(self.nu0, self.omega, t) - b * t)

    def parareal(self, z0, n_slices, nc, nf, K, T, g_is_f=False):
        """Alg.1 on complex mode amplitudes; returns (z_T^K, [z_T^0..z_T^K])."""
        Dt, dt = T / (n_slices * nc), T / (n_slices * nf)

        def G(z, m):
            return self.fine(z, m * nf, nf, dt) if g_is_f else self.coarse(z, m * nc, nc, Dt)

        def F(z, m):
            return self.fine(z, m * nf, nf, dt)

        # initial guess: serial coarse sweep (u^0_{n+1} = G(u^0_n))
        U = [np.array(z0, dtype=complex)]
        for m in range(n_slices):
            U.append(G(U[-1], m))
        Gold = [U[m + 1] for m in range(n_slices)]
        hist = [U[-1]]
        for _ in range(K):
            Fk = [F(U[m], m) for m in range(n_slices)]
            V = [np.array(z0, dtype=complex)]
            for m in range(n_slices):
                g = G(V[m], m)
                V.append(Fk[m] + (g - Gold[m]))
                Gold[m] = g
            U = V
            hist.append(U[-1])
        return U[-1], hist


def sine_modes(n):
    """The paper's u0 = sin(2pi x) sin(2pi y) sin(2pi z) is
    sum over s in {+-1}^3 of (i/8) s_x s_y s_z e^{i theta s.j}, theta = 2pi/n.
    Returns (thetas (8,3), coefficients (8,))."""
    th = 2.0 * np.pi / n
    thetas, coef = [], []
    for sx in (1, -1):
        for sy in (1, -1):
            for sz in (1, -1):
                thetas.append((sx * th, sy * th, sz * th))
                # 1/(2i)^3 = i/8 ; sin(a) = (e^{ia} - e^{-ia}) / (2i)
                coef.append((1j / 8.0) * sx * sy * sz)
    return np.array(thetas), np.array(coef, dtype=complex)


def synthesize(n, thetas, amps):
    """Real field Re sum_m amps[m] e^{i theta_m . (i, j, k)} on the n^3 grid,
    shape (z, y, x).  Separable evaluation: each mode is a product of 1D waves."""
    idx = np.arange(n)
    out = np.zeros((n, n, n))
    for th, a in zip(thetas, amps):
        ex = np.exp(1j * th[0] * idx)
        ey = np.exp(1j * th[1] * idx)
        ez = np.exp(1j * th[2] * idx)
        out += np.real(a * ez[:, None, None] * ey[None, :, None] * ex[None, None, :])
    return out


def synthesize_torch(n, thetas, amps, device):
    """synthesize() evaluated with torch on `device` (large n: 512^3 in seconds).
    Same formula, fp64; a checker, not part of the CUDA path."""
    import torch
    idx = torch.arange(n, dtype=torch.float64, device=device)
    out = torch.zeros((n, n, n), dtype=torch.float64, device=device)
    for th, a in zip(thetas, amps):
        ex = torch.exp(1j * float(th[0]) * idx)
        ey = torch.exp(1j * float(th[1]) * idx)
        ez = torch.exp(1j * float(th[2]) * idx)
        out += torch.real(complex(a) * ez[:, None, None] * ey[None, :, None] * ex[None, None, :])
    return out


def exact_solution(n, c, nu0, omega, t):
    """Closed form u = a(t) u0(x - c t) (exp restored per C18)."""
    a = np.exp(-12.0 * np.pi ** 2 * nu_integral(nu0, omega, t))
    x = np.arange(n) / n
    sx = np.sin(2 * np.pi * (x - c[0] * t))
    sy = np.sin(2 * np.pi * (x - c[1] * t))
    sz = np.sin(2 * np.pi * (x - c[2] * t))
    return a * sz[:, None, None] * sy[None, :, None] * sx[None, None, :]


def fft_thetas(n):
    m = np.fft.fftfreq(n, d=1.0 / n)  # integer wavenumbers
    th = 2 * np.pi * m / n
    TZ, TY, TX = np.meshgrid(th, th, th, indexing="ij")
    return np.stack([TX, TY, TZ], axis=-1)  # (z, y, x, 3) with x-angle first


def fft_apply(u, factor):
    """Apply per-wavenumber multiplier (array shaped like fftn(u)) to a real field."""
    return np.real(np.fft.ifftn(np.fft.fftn(u) * factor))
