"""Run every kernel family once on small and mid-size grids (seam and TMA tiles,
ragged four-stage tiles, G on the n/2 mesh, slice groups) and print one digest of
all outputs.  With PR_LIB pointing at the PRK_DEBUG build every in-kernel index
check is armed (a violation traps); tests/test_gpu_debug.py compares the digest
with the release build's."""
import hashlib
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import paper_1409_8563_b200 as pr  # noqa: E402

h = hashlib.sha256()
for n, f2 in ((32, "1"), (64, "1"), (128, "1"), (40, "0"), (32, "0")):
    os.environ["PR_F2"] = f2
    g = pr.Grid(pr.Problem(n, c=(1.0, -0.5, 0.25), T=0.002), 0)
    u = torch.empty((n, n, n), dtype=torch.float64, device="cuda")
    pr.pr_fill_sine(g, u)
    v = torch.empty_like(u)
    pr.pr_fine(g, u, v, 3, 21, 1e-5)
    h.update(v.cpu().numpy().tobytes())
    pr.pr_coarse(g, u, v, 5, 37, 1e-5)
    h.update(v.cpu().numpy().tobytes())
    if n % 4 == 0:
        pr.pr_coarse_mesh(g, u, v, 5, 9, 1e-5)
        h.update(v.cpu().numpy().tobytes())
    uf = torch.empty_like(u)
    pr.pr_fine(g, u, uf, 0, 64, 0.002 / 64)
    d = pr.pr_parareal(g, pr.PararealCfg(4, 4, 16, 2), u, v, uf)
    h.update(v.cpu().numpy().tobytes())
    h.update(repr(d).encode())
    torch.cuda.synchronize()
    g.destroy()
print("digest", h.hexdigest(), flush=True)
