"""The paper's own configuration on the GPU (BASELINE configs[1]):
128^3, dt = T/2^15, Dt = T/2^11, 8 slices, K = 3 on one GPU (slice group 8).

Pinned by the exact discrete modal recurrence (tests/modal_ref.py) at a size
the CPU oracle cannot run to T, and by the paper's printed accuracy numbers
(tests/golden/paper_accuracy.json)."""
import json
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import modal_ref as M
import paper_1409_8563_b200 as pr

pytestmark = pytest.mark.gpu
GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


@pytest.mark.parametrize("omega,nu_mode,key", [(0.0, 1, "eps_fine_omega0"), (100.0, 1, "eps_fine_omega100")])
def test_paper_eps_fine_on_gpu(omega, nu_mode, key):
    g_ = json.load(open(os.path.join(GOLDEN, "paper_accuracy.json")))
    n, T = 128, 0.1
    with pr.Grid(pr.Problem(n, omega=omega, nu_mode=nu_mode)) as g:
        u = torch.empty((n, n, n), dtype=torch.float64, device="cuda")
        pr.pr_fill_sine(g, u)
        pr.pr_fine(g, u, u, 0, 2 ** 15, T / 2 ** 15)
        ex = M.exact_solution(n, (1.0, 1.0, 1.0), 0.1, omega, T)
        eps = float(np.max(np.abs(u.cpu().numpy() - ex)) / np.max(np.abs(ex)))
        assert float(f"{eps:.1e}") == g_[key]["value"]
        # and the exact discrete solution (modal recurrence) to 1e-12 normwise
        th, coef = M.sine_modes(n)
        ms = M.ModalSolver(n, (1.0, 1.0, 1.0), 0.1, omega, nu_mode, th)
        um = M.synthesize(n, th, ms.fine(coef, 0, 2 ** 15, T / 2 ** 15))
        assert np.max(np.abs(u.cpu().numpy() - um)) / np.max(np.abs(um)) <= 1e-12


def test_paper_eps_coarse_on_gpu():
    g_ = json.load(open(os.path.join(GOLDEN, "paper_accuracy.json")))
    n, T = 128, 0.1
    with pr.Grid(pr.Problem(n)) as g:
        u = torch.empty((n, n, n), dtype=torch.float64, device="cuda")
        pr.pr_fill_sine(g, u)
        pr.pr_coarse(g, u, u, 0, 2 ** 11, T / 2 ** 11)
        ex = M.exact_solution(n, (1.0, 1.0, 1.0), 0.1, 100.0, T)
        eps = float(np.max(np.abs(u.cpu().numpy() - ex)) / np.max(np.abs(ex)))
        assert float(f"{eps:.1e}") == g_["eps_coarse"]["value"]


@pytest.mark.parametrize("nu_mode", [0, 1])
def test_cfg2_parareal_defects_vs_modal(nu_mode):
    """d^0..d^3 of the paper's Parareal configuration vs the exact modal
    recurrence: |d_gpu - d_modal| <= 1e-10 (C14); d^3 << eps_fine."""
    n, T, Np, K, Nt, NC = 128, 0.1, 8, 3, 2 ** 15, 2 ** 11
    th, coef = M.sine_modes(n)
    ms = M.ModalSolver(n, (1.0, 1.0, 1.0), 0.1, 100.0, nu_mode, th)
    zf = ms.fine(coef, 0, Nt, T / Nt)
    _, hist = ms.parareal(coef, Np, NC // Np, Nt // Np, K, T)
    uf_m = M.synthesize(n, th, zf)
    d_m = [np.max(np.abs(M.synthesize(n, th, h) - uf_m)) / np.max(np.abs(uf_m)) for h in hist]
    with pr.Grid(pr.Problem(n, nu_mode=nu_mode)) as g:
        u0 = torch.empty((n, n, n), dtype=torch.float64, device="cuda")
        pr.pr_fill_sine(g, u0)
        uf = torch.empty_like(u0)
        pr.pr_fine(g, u0, uf, 0, Nt, T / Nt)
        uT = torch.empty_like(u0)
        d = pr.pr_parareal(g, pr.PararealCfg(Np, NC // Np, Nt // Np, K), u0, uT, uf)
    assert np.max(np.abs(np.array(d) - np.array(d_m))) <= 1e-10, (d, d_m)
    assert d[0] > d[1] > d[2] > d[3]
    if nu_mode == 1:
        assert d[3] < 4.8e-6 / 10


@pytest.mark.parametrize("omega", [0.0, 100.0])
@pytest.mark.parametrize("Np", [32, 128])
def test_fig3_many_slices_vs_modal(Np, omega):
    """Fig. 3: at the paper's discretization with N_p = 32 and 128
    slices (one slice group on this GPU) d^k matches the exact modal recurrence
    to 1e-10, convergence is rapid, and d^3 is far below eps_fine ~ 4.8e-6 for
    omega = 100."""
    n, T, Nt, NC, K = 128, 0.1, 2 ** 15, 2 ** 11, 3
    th, coef = M.sine_modes(n)
    ms = M.ModalSolver(n, (1.0, 1.0, 1.0), 0.1, omega, 0, th)
    zf = ms.fine(coef, 0, Nt, T / Nt)
    _, hist = ms.parareal(coef, Np, NC // Np, Nt // Np, K, T)
    uf_m = M.synthesize(n, th, zf)
    d_m = [np.max(np.abs(M.synthesize(n, th, h) - uf_m)) / np.max(np.abs(uf_m)) for h in hist]
    with pr.Grid(pr.Problem(n, omega=omega)) as g:
        u0 = torch.empty((n, n, n), dtype=torch.float64, device="cuda")
        pr.pr_fill_sine(g, u0)
        uf = torch.empty_like(u0)
        pr.pr_fine(g, u0, uf, 0, Nt, T / Nt)
        uT = torch.empty_like(u0)
        d = pr.pr_parareal(g, pr.PararealCfg(Np, NC // Np, Nt // Np, K), u0, uT, uf)
    assert np.max(np.abs(np.array(d) - np.array(d_m))) <= 1e-10, (d, d_m)
    assert d[0] > d[1] > d[2] > d[3]
    if omega == 100.0:
        assert d[3] < 4.8e-6 / 10
