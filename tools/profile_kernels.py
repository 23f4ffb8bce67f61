"""Launch each hot-path kernel a few times at one grid size, for ncu.

    python tools/profile_kernels.py [n]
Order: pr_fine 3 steps (S1..S4 x 3, direct launches), pr_coarse 3 steps,
pr_correct with fused defect, pr_defect.  Kernel sequence for ncu -s/-c:
fill_sine, set_pos, [S1 S2 S3 S4] x 3, set_pos, [coarse] x 3 (+ copy), ...
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import paper_1409_8563_b200 as pr  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
g = pr.Grid(pr.Problem(n), 0)
u = torch.empty((n, n, n), dtype=torch.float64, device="cuda")
pr.pr_fill_sine(g, u)
v = torch.empty_like(u)
w = torch.empty_like(u)
pr.pr_fine(g, u, v, 0, 3, 0.1 / 2 ** 17)
pr.pr_coarse(g, u, w, 0, 3, 0.1 / 2 ** 13)
d = pr.pr_correct(g, v, w, u, v, u)
d2 = pr.pr_defect(g, v, u)
torch.cuda.synchronize()
print("ok", n, d, d2, pr.pr_kernel_launches())
g.destroy()
