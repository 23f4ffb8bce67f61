"""A/B: time pr_fine with a given libparareal.so (path in argv[1]) and PR_FTILE variants."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1409_8563_b200._lib as L
L.LIB_PATH = os.path.abspath(sys.argv[1])
import torch
import paper_1409_8563_b200 as pr
n = 256
for v in sys.argv[2:]:
    os.environ["PR_FTILE"] = v
    g = pr.Grid(pr.Problem(n), 0)
    u = torch.empty((n, n, n), dtype=torch.float64, device="cuda"); pr.pr_fill_sine(g, u)
    w = torch.empty_like(u)
    pr.pr_fine(g, u, w, 0, 32, 1e-6); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); pr.pr_fine(g, u, w, 0, 64, 1e-6); e1.record(); torch.cuda.synchronize()
    print(sys.argv[1], v, e0.elapsed_time(e1) / 64, flush=True)
    g.destroy()
