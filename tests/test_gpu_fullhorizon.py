"""Full-horizon Parareal at BASELINE's large sizes on one GPU:
cfg3 (256^3, T = 0.1, N_t = 2^17, N_C = 2^13) and cfg4 (512^3, T = 0.1/32,
N_t = 2^14, N_C = 2^10), N_p = 8 slices as one slice group, K = 3, in the
launch configuration bench.py times (fused two-kernel F, persistent G).

The CPU oracle cannot run these to T, so the pin is the exact discrete modal
recurrence of the same Alg.1 run (tests/modal_ref.py: per-Fourier-mode scalar
recurrences of the printed stencils, independent of the oracle and of the CUDA
path): |d^k_gpu - d^k_modal| <= 1e-10 (C14) and u_T within 1e-12 normwise
(C13).  The modal d^k are also held to SURVEY Appendix A's printed 8-digit
values (golden/modal_pins.json), so a regression in modal_ref itself shows."""
import json
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import modal_ref as M
import paper_1409_8563_b200 as pr
from synthetic import CONFIGS

pytestmark = pytest.mark.gpu
GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


@pytest.mark.parametrize("name", ["cfg3", "cfg4"])
def test_full_horizon_parareal_vs_modal(name):
    cfg = CONFIGS[name]
    pins = json.load(open(os.path.join(GOLDEN, "modal_pins.json")))[name]
    n, Np, K = cfg.n, 8, 3
    th, coef = M.sine_modes(n)
    ms = M.ModalSolver(n, cfg.c, cfg.nu0, cfg.omega, cfg.nu_mode, th)
    zf = ms.fine(coef, 0, cfg.Nt, cfg.T / cfg.Nt)
    zT, hist = ms.parareal(coef, Np, cfg.NC // Np, cfg.Nt // Np, K, cfg.T)
    dev = torch.device("cuda", 0)
    uf_m = M.synthesize_torch(n, th, zf, dev)
    Mx = float(uf_m.abs().max())
    d_m = [float((M.synthesize_torch(n, th, h, dev) - uf_m).abs().max()) / Mx for h in hist]
    uT_m = M.synthesize_torch(n, th, zT, dev)
    # the modal reference reproduces SURVEY Appendix A's printed digits (8 significant;
    # the survey's runs used slice-local step times, which moves the smallest d^k by
    # ~2e-14 absolute: hence the 1e-13 floor, still 1000x inside C14's 1e-10)
    for got, want in zip(d_m, pins["defects"]):
        if want >= 1e-14:
            assert abs(got - want) <= 6e-8 * want + 1e-13, (d_m, pins["defects"])
    del uf_m
    torch.cuda.empty_cache()
    with pr.Grid(pr.Problem(n, c=cfg.c, nu0=cfg.nu0, omega=cfg.omega, T=cfg.T, nu_mode=cfg.nu_mode)) as g:
        u0 = torch.empty((n, n, n), dtype=torch.float64, device=dev)
        pr.pr_fill_sine(g, u0)
        uf = torch.empty_like(u0)
        pr.pr_fine(g, u0, uf, 0, cfg.Nt, cfg.T / cfg.Nt)
        uT = torch.empty_like(u0)
        d = pr.pr_parareal(g, pr.PararealCfg(Np, cfg.NC // Np, cfg.Nt // Np, K), u0, uT, uf)
        torch.cuda.synchronize()
    err = float((uT - uT_m).abs().max() / uT_m.abs().max())
    assert err <= 1e-12, err
    assert np.max(np.abs(np.array(d) - np.array(d_m))) <= 1e-10, (d, d_m)
    assert abs(float(uf.abs().max()) - pins["max_u_fine"]) <= 1e-12
