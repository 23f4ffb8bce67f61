"""Reproduce the paper's convergence study (Fig. 3) on one GPU:
d^k versus k for N_p = 8, 32, 128 time slices and omega = 0, 100 at the
paper's discretization (128^3, N_t = 2^15, N_C = 2^11, T = 0.1), the slices of
each run as one slice group on the GPU, next to the exact modal recurrence.

    python tools/fig3.py [K] [out.txt]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import modal_ref as M  # noqa: E402
import paper_1409_8563_b200 as pr  # noqa: E402

n, T, Nt, NC = 128, 0.1, 2 ** 15, 2 ** 11


def modal_defects(omega, Np, K):
    th, coef = M.sine_modes(n)
    ms = M.ModalSolver(n, (1.0, 1.0, 1.0), 0.1, omega, 0, th)
    zf = ms.fine(coef, 0, Nt, T / Nt)
    _, hist = ms.parareal(coef, Np, NC // Np, Nt // Np, K, T)
    uf = M.synthesize(n, th, zf)
    return [float(np.max(np.abs(M.synthesize(n, th, h) - uf)) / np.max(np.abs(uf))) for h in hist]


def main():
    K = int(sys.argv[1]) if len(sys.argv) > 1 else 4
    out = sys.argv[2] if len(sys.argv) > 2 else None
    lines = ["# Fig. 3 (P:478-492): relative defect d^k (Eq.(defect)) vs iteration k, 128^3, "
             "N_t = 2^15, N_C = 2^11, T = 0.1, nu0 = 0.1, c = (1,1,1), stage-time nu (C1)",
             "# GPU: pr_parareal on one B200 (all N_p slices as one slice group); modal: exact "
             "per-mode recurrence (tests/modal_ref.py)",
             f"{'omega':>6} {'N_p':>4} {'k':>2} {'d^k GPU':>14} {'d^k modal':>14} {'|diff|':>10}"]
    for omega in (0.0, 100.0):
        with pr.Grid(pr.Problem(n, omega=omega)) as g:
            u0 = torch.empty((n, n, n), dtype=torch.float64, device="cuda")
            pr.pr_fill_sine(g, u0)
            uf = torch.empty_like(u0)
            pr.pr_fine(g, u0, uf, 0, Nt, T / Nt)
            uT = torch.empty_like(u0)
            for Np in (8, 32, 128):
                d = pr.pr_parareal(g, pr.PararealCfg(Np, NC // Np, Nt // Np, K), u0, uT, uf)
                dm = modal_defects(omega, Np, K)
                for k in range(K + 1):
                    lines.append(f"{omega:6.0f} {Np:4d} {k:2d} {d[k]:14.6e} {dm[k]:14.6e} "
                                 f"{abs(d[k] - dm[k]):10.1e}")
                    print(lines[-1], flush=True)
    txt = "\n".join(lines) + "\n"
    if out:
        open(out, "w").write(txt)


if __name__ == "__main__":
    main()
