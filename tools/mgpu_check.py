"""Multi-GPU Parareal check (run under torchrun, one process per GPU).

    torchrun --nproc-per-node W --master-addr 127.0.0.1 --master-port P tools/mgpu_check.py [n] [Np] [K] [tol] [nccl|peer] [stress]

Every rank runs pr_parareal on its slice group with NCCL hand-off; the last
rank compares u_T and d^k with (a) a single-GPU run of the same N_p slices
(W-invariance, must be bitwise) and (b) the CPU oracle (1e-12 / 1e-10).
Prints one JSON line on the last rank and exits non-zero on mismatch.
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_1409_8563_b200 as pr  # noqa: E402


def same(a, b):
    """Defect lists equal, NaN (iterations not run) equal to NaN."""
    a, b = np.asarray(a, dtype=float), np.asarray(b, dtype=float)
    return a.shape == b.shape and bool(np.array_equal(a, b, equal_nan=True))


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 32
    Np = int(sys.argv[2]) if len(sys.argv) > 2 else 4
    K = int(sys.argv[3]) if len(sys.argv) > 3 else 2
    tol = float(sys.argv[4]) if len(sys.argv) > 4 else 0.0
    handoff = sys.argv[5] if len(sys.argv) > 5 else "nccl"
    flags = pr.PR_FLAG_PEER_HANDOFF if handoff == "peer" else 0
    T, Nt, NC = 0.1, 2048 * (n // 32) ** 2 if n <= 64 else 2048, 128 * (n // 32) ** 2 if n <= 64 else 128
    if n > 64:  # short horizon with the cfg-style step sizes
        T, Nt, NC = 0.1 / 64, 2 ** 11, 2 ** 7
    stress = len(sys.argv) > 6 and sys.argv[6] == "stress"
    if stress:  # many hand-offs: the default step sizes on a 64-step horizon, K up to ~10^3
        T, Nt, NC = 0.1 * 64 / 2048, 64, 8
    world, rank, local = int(os.environ["WORLD_SIZE"]), int(os.environ["RANK"]), int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    g = pr.Grid(pr.Problem(n, T=T), local)
    pr.comm_init_torch(g)
    dev = torch.device("cuda", local)
    u0 = torch.empty((n, n, n), dtype=torch.float64, device=dev)
    pr.pr_fill_sine(g, u0)
    last = rank == world - 1
    uf = torch.empty_like(u0) if last else None
    if last:
        pr.pr_fine(g, u0, uf, 0, Nt, T / Nt)
    uT = torch.empty_like(u0)
    cfg = pr.PararealCfg(Np, NC // Np, Nt // Np, K, flags=flags, tol=tol)
    d = pr.pr_parareal(g, cfg, u0, uT if last else None, uf)
    t = pr.pr_last_timings(g)
    mon, iters = pr.pr_last_monitors(g)
    all_iters = [None] * world
    dist.all_gather_object(all_iters, iters)
    ok = True
    d2 = pr.pr_parareal(g, cfg, u0, uT if last else None, uf)  # second call: same buffers, next epoch
    info = {"world": world, "n": n, "Np": Np, "K": K, "tol": tol, "handoff": handoff, "defects": d,
            "repeat_equal": same(d2, d), "timings": t,
            "iters": all_iters}
    if last and tol > 0:
        # convergence control: per-rank iteration counts and u_T against the oracle's stop rule
        import oracle
        p = oracle.Problem(n, T=T)
        o0 = oracle.initial(n)
        ouf = oracle.serial_fine(p, Nt, o0)
        ref = oracle.parareal_tol(p, Np, NC // Np, Nt // Np, K, tol, world, o0, ouf)
        err = float(np.max(np.abs(uT.cpu().numpy() - ref.u_T)) / np.max(np.abs(ref.u_T)))
        info.update(oracle_iters=[int(x) for x in ref.iters], oracle_rel_err=err)
        ok &= err <= 1e-12 and [int(x) for x in ref.iters] == all_iters and same(d2, d)
        info["bitwise_equal_to_1gpu"] = True
        info["ok"] = bool(ok)
        print(json.dumps(info), flush=True)
    elif last:
        # (a) W-invariance: the same slices on this one GPU, without NCCL
        g1 = pr.Grid(pr.Problem(n, T=T), local)
        uT1 = torch.empty_like(u0)
        d1 = pr.pr_parareal(g1, pr.PararealCfg(Np, NC // Np, Nt // Np, K, tol=tol), u0, uT1, uf)
        info["bitwise_equal_to_1gpu"] = bool(torch.equal(uT, uT1)) and d1 == d
        ok &= info["bitwise_equal_to_1gpu"] and same(d2, d)
        # (b) oracle (small grids only)
        if n <= 48 and not stress:  # (stress: K ~ 10^3 iterations, bitwise vs (a) only)
            import oracle
            p = oracle.Problem(n, T=T)
            o0 = oracle.initial(n)
            ouf = oracle.serial_fine(p, Nt, o0)
            ref = oracle.parareal(p, Np, NC // Np, Nt // Np, K, o0, ouf)
            err = float(np.max(np.abs(uT.cpu().numpy() - ref.u_T)) / np.max(np.abs(ref.u_T)))
            derr = float(np.max(np.abs(np.array(d) - ref.defects)))
            info.update(oracle_rel_err=err, oracle_defect_err=derr)
            ok &= err <= 1e-12 and derr <= 1e-10
        info["ok"] = bool(ok)
        print(json.dumps(info), flush=True)
        g1.destroy()
    g.destroy()
    dist.barrier(device_ids=[local])
    dist.destroy_process_group()
    return 0 if ok else 1


if __name__ == "__main__":
    sys.exit(main())
