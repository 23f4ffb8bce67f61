"""Small run of every kernel for compute-sanitizer (racecheck / memcheck / synccheck).

    compute-sanitizer --tool racecheck python tools/sanitize_run.py
Covers: fused F (n=32, 64), four-stage F (n=32 forced, n=40 ragged), coarse (odd/even),
correction + defect, fill_sine, Parareal with 4 slices."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import paper_1409_8563_b200 as pr  # noqa: E402


def run(n, f2):
    os.environ["PR_F2"] = "1" if f2 else "0"
    g = pr.Grid(pr.Problem(n, c=(1.0, -0.5, 0.25), T=0.002), 0)
    u = torch.empty((n, n, n), dtype=torch.float64, device="cuda")
    pr.pr_fill_sine(g, u)
    v = torch.empty_like(u)
    w = torch.empty_like(u)
    pr.pr_fine(g, u, v, 0, 3, 1e-5)
    pr.pr_fine(g, v, v, 3, 2, 1e-5)
    pr.pr_coarse(g, u, w, 0, 3, 4e-5)
    pr.pr_coarse(g, w, w, 3, 2, 4e-5)
    pr.pr_correct(g, v, w, u, v, u)
    d = pr.pr_parareal(g, pr.PararealCfg(4, 2, 4, 2), u, w, v)
    torch.cuda.synchronize()
    g.destroy()
    return d


for n, f2 in ((32, True), (64, True), (32, False), (40, False)):
    print(n, f2, run(n, f2), flush=True)
print("sanitize_run ok")
