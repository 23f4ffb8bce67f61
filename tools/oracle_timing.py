"""CPU oracle timing on the host cores of the GPU box (SURVEY 8(d) "Oracle timing"):
per-step tau_f (RK4) and tau_c (Euler) at 32^3 .. 512^3, with 1 OpenMP thread and
with all of them, next to the GPU per-step times for the GPU/CPU ratio.

    python tools/oracle_timing.py [out.txt]
The oracle is test infrastructure; this tool only times it (as bench.py's
cpu_baseline does).  GPU columns come from the product path (pr_fine/pr_coarse)."""
import os
import platform
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

SIZES = [(32, 64, 64), (128, 8, 16), (256, 2, 4), (512, 1, 1)]  # n, fine steps, coarse steps


def cpu_model():
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True).stdout
        keep = [l for l in out.splitlines() if l.split(":")[0].strip() in
                ("Model name", "Socket(s)", "Core(s) per socket", "Thread(s) per core", "CPU(s)")]
        return "; ".join(" ".join(l.split()) for l in keep)
    except OSError:
        return platform.processor()


def time_oracle(threads, n, nf, nc):
    """Runs in a subprocess so OMP_NUM_THREADS takes effect."""
    code = f"""
import time, oracle
p = oracle.Problem({n})
u = oracle.initial({n})
oracle.fine(p, u, 0, 1, 1e-7)
t0 = time.perf_counter(); oracle.fine(p, u, 0, {nf}, 1e-7); tf = (time.perf_counter() - t0) / {nf}
t0 = time.perf_counter(); oracle.coarse(p, u, 0, {nc}, 1e-6); tc = (time.perf_counter() - t0) / {nc}
print(tf, tc, oracle.threads())
"""
    env = dict(os.environ, OMP_NUM_THREADS=str(threads), PYTHONPATH=ROOT)
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env,
                         cwd=ROOT, timeout=1800).stdout.split()
    return float(out[0]), float(out[1]), int(out[2])


def time_gpu(n):
    import torch
    import paper_1409_8563_b200 as pr
    g = pr.Grid(pr.Problem(n), 0)
    u = torch.empty((n, n, n), dtype=torch.float64, device="cuda")
    pr.pr_fill_sine(g, u)
    v = torch.empty_like(u)
    steps = max(16, 4096 * 32 ** 3 // n ** 3)
    res = []
    for fn, dt in ((pr.pr_fine, 1e-7), (pr.pr_coarse, 1e-6)):
        fn(g, u, v, 0, 16, dt)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn(g, u, v, 0, steps, dt)
        e1.record()
        torch.cuda.synchronize()
        res.append(e0.elapsed_time(e1) / steps / 1e3)
    g.destroy()
    return res


def main():
    out = sys.argv[1] if len(sys.argv) > 1 else None
    allt = os.cpu_count() or 1
    lines = [f"# host: {cpu_model()}; nproc={allt}",
             "# oracle/oracle.c (-O2 -ffp-contract=off -fopenmp), seconds per step; GPU: pr_fine / pr_coarse",
             f"{'n':>5} {'tau_f 1 thr':>12} {'tau_f all':>12} {'tau_c 1 thr':>12} {'tau_c all':>12} "
             f"{'tau_f GPU':>12} {'tau_c GPU':>12} {'F CPU(all)/GPU':>15}"]
    for n, nf, nc in SIZES:
        f1, c1, _ = time_oracle(1, n, nf, nc)
        fa, ca, th = time_oracle(allt, n, nf, nc)
        fg, cg = time_gpu(n)
        lines.append(f"{n:>5} {f1:12.4e} {fa:12.4e} {c1:12.4e} {ca:12.4e} {fg:12.4e} {cg:12.4e} {fa / fg:15.0f}")
        print(lines[-1], flush=True)
    lines.append(f"# all = {th} OpenMP threads; the paper's GPU/CPU ratio per step is about 4.5 (P:527), "
                 "K20X vs one 8-core Xeon node, as context only")
    txt = "\n".join(lines) + "\n"
    print(txt)
    if out:
        open(out, "w").write(txt)


if __name__ == "__main__":
    main()
