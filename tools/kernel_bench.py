"""Time the fused stencil kernels per tile variant / z-chunking (tuning aid).

    python tools/kernel_bench.py [n] [variants...]
Prints per-step device times (CUDA events, warm, L2 flushed implicitly by
fields > L2 at 256^3; median of BENCH_REPS repetitions, default 5) and
algorithmic GB/s; checks variants agree bitwise."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import paper_1409_8563_b200 as pr  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
variants = [v for v in sys.argv[2:]] or ["0", "1", "2", "3"]
chunks = os.environ.get("BENCH_CHUNKS", "").split(",") if os.environ.get("BENCH_CHUNKS") else [None]
REPS = int(os.environ.get("BENCH_REPS", "5"))
ref = None
u0 = None
for ch in chunks:
    for v in variants:
        # "f2_N" = fused two-kernel RK4 step, variant N; "0".."3" = four-stage tile variants;
        # "cN" = default F with persistent coarse variant N; "cold" = the lockstep coarse kernel
        if v.startswith("c"):
            os.environ["PR_F2"] = "1"
            os.environ["PR_FTILE"] = "14"
            os.environ["PR_TILE"] = "0"
            os.environ["PR_C2"] = "0" if v == "cold" else "1"
            os.environ["PR_CTILE"] = "0" if v == "cold" else v[1:]
        else:
            os.environ.pop("PR_C2", None)
            os.environ["PR_F2"] = "1" if v.startswith("f2") else "0"
            os.environ["PR_FTILE"] = v[3:] if v.startswith("f2_") else "14"
            os.environ["PR_TILE"] = "0" if v.startswith("f2") else str(v)
        if ch is None:
            os.environ.pop("PR_CHUNKS_Z", None)
        else:
            os.environ["PR_CHUNKS_Z"] = ch
        try:
            g = pr.Grid(pr.Problem(n), 0)
        except pr.PrError as e:
            print(f"n={n} variant={v}: {e}", flush=True)
            continue
        if u0 is None:
            u0 = torch.empty((n, n, n), dtype=torch.float64, device="cuda")
            pr.pr_fill_sine(g, u0)
        u = torch.empty_like(u0)
        dt, Dt = 0.1 / 2 ** 17 * (256 / n) ** 2, 0.1 / 2 ** 13 * (256 / n) ** 2
        pr.pr_fine(g, u0, u, 0, 32, dt)
        pr.pr_coarse(g, u0, u, 0, 64, Dt)
        torch.cuda.synchronize()
        NF, NC = 64, 256
        w = torch.empty_like(u0)
        tfs, tcs = [], []
        for _ in range(REPS):  # median of REPS timings (run-to-run spread is a few %)
            e = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
            e[0].record()
            pr.pr_fine(g, u0, u, 0, NF, dt)
            e[1].record()
            e[2].record()
            pr.pr_coarse(g, u0, w, 0, NC, Dt)
            e[3].record()
            torch.cuda.synchronize()
            tfs.append(e[0].elapsed_time(e[1]) / NF)
            tcs.append(e[2].elapsed_time(e[3]) / NC)
        tf, tc = sorted(tfs)[REPS // 2], sorted(tcs)[REPS // 2]
        same = None
        if ref is None:
            ref = (u.clone(), w.clone())
        else:
            same = bool(torch.equal(ref[0], u) and torch.equal(ref[1], w))
        print(f"n={n} variant={v} chunks={ch}: fine {tf:.4f} ms/step ({128 * n**3 / tf / 1e6:.0f} GB/s), "
              f"coarse {tc:.4f} ms/step ({16 * n**3 / tc / 1e6:.0f} GB/s), tau_c/tau_f={tc / tf:.3f}, "
              f"bitwise-equal-to-first={same}", flush=True)
        g.destroy()
