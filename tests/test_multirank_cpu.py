"""World-size-2 (and 4, 8) CPU test of the multi-rank host logic over torch.distributed
gloo: every rank executes the schedule the C library emits (pr_plan) with the
oracle's F and G and real point-to-point send/recv; the last rank's u_T and
defect history must equal the oracle's serial Alg.1 emulation bitwise (the
hand-off is a byte copy and every rank does the same arithmetic)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def execute_plan(plan, rank, W, Np, nc, nf, p, orc, u0, u_ref, tol=0.0):
    """Python mirror of pr_parareal's executor: same buffer roles, same order,
    including convergence-controlled stopping (C23: the iterate-change
    monitor over own slices, the stop flag appended to the hand-off message)."""
    s, j0 = Np // W, rank * (Np // W)
    Dt, dt = p.T / (Np * nc), p.T / (Np * nf)
    G = lambda u, m: orc.coarse(p, u, m * nc, nc, Dt)
    F = lambda u, m: orc.fine(p, u, m * nf, nf, dt)
    start, f, out, gold, used = [None] * s, [None] * s, [None] * s, [None] * s, [None] * s
    v, recvb, gnew, defects = u0, None, None, []
    K = sum(1 for q in plan if q[0] == "END_ITER")
    pred_stopped, recvd, stopped, iters = rank == 0, False, False, 0
    dmax = umax = 0.0
    for op, k, sl, peer in plan:
        if stopped:
            break
        l = sl - j0
        if op == "G_PREFIX":
            v = G(v, sl)
        elif op == "G_INIT":
            start[l] = v
            gold[l] = G(start[l], sl)
            v = gold[l]
        elif op == "DEFECT0":
            defects.append(orc.defect(gold[s - 1], u_ref))
        elif op == "F":
            f[l] = F(start[l], sl)
        elif op == "RECV":
            recvd = False
            if not pred_stopped:
                t = torch.empty(u0.size + (1 if tol > 0 else 0), dtype=torch.float64)
                dist.recv(t, src=peer)
                arr = t.numpy()
                recvb = arr[:u0.size].reshape(u0.shape).copy()
                recvd = True
                if tol > 0 and arr[-1] != 0.0:
                    pred_stopped = True
        elif op == "G":
            if sl == 0:
                used[l] = u0
            elif l == 0:
                used[l] = recvb if recvd else start[0]
            else:
                used[l] = out[l - 1]
            gnew = G(used[l], sl)
        elif op == "CORRECT":
            prev = gold[l] if k == 0 else (start[l + 1] if l < s - 1 else out[s - 1])
            new = f[l] + (gnew - gold[l])
            if l == 0:
                dmax = umax = 0.0
            dmax = max(dmax, float(np.max(np.abs(new - prev))))
            umax = max(umax, float(np.max(np.abs(new))))
            out[l] = new
            gold[l] = gnew
            if sl == Np - 1:
                defects.append(orc.defect(out[l], u_ref))
            if l == s - 1:
                iters = k + 1
                ch = dmax / umax if umax > 0 else dmax
                stop_now = k == K - 1 or (tol > 0 and pred_stopped and ch <= tol)
                if stop_now:
                    stopped = True
                    if rank < W - 1:  # the last message carries the stop flag
                        msg = np.append(out[s - 1].ravel(), 1.0) if tol > 0 else out[s - 1]
                        dist.send(torch.from_numpy(np.ascontiguousarray(msg)), dst=rank + 1)
                elif rank < W - 1:
                    pending = np.append(out[s - 1].ravel(), 0.0) if tol > 0 else out[s - 1]
        elif op == "SEND":
            dist.send(torch.from_numpy(np.ascontiguousarray(pending)), dst=peer)
        elif op == "END_ITER":
            start = list(used)
    return (out[s - 1] if K > 0 else gold[s - 1]), defects, iters


def worker(rank, W, port, Np, K, q, tol=0.0):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=W)
    try:
        import oracle
        import paper_1409_8563_b200 as pr
        from synthetic import random_field, PARITY_C
        n, nc, nf = 8, 2, 6
        p = oracle.Problem(n, c=PARITY_C, T=0.003)
        u0 = random_field(n, 11)
        u_ref = oracle.serial_fine(p, Np * nf, u0)
        plan = pr.pr_plan(Np, K, W, rank)
        uT, defects, iters = execute_plan(plan, rank, W, Np, nc, nf, p, oracle, u0, u_ref, tol)
        all_iters = [None] * W
        dist.all_gather_object(all_iters, iters)
        if rank == W - 1:
            if tol > 0:
                ref = oracle.parareal_tol(p, Np, nc, nf, K, tol, W, u0, u_ref)
                ok_d = bool(np.array_equal(np.array(defects), ref.defects[:len(defects)]))
                q.put((bool(np.array_equal(uT, ref.u_T)), ok_d and list(ref.iters) == all_iters,
                       (defects, all_iters, list(ref.iters))))
            else:
                ref = oracle.parareal(p, Np, nc, nf, K, u0, u_ref)
                q.put((bool(np.array_equal(uT, ref.u_T)),
                       bool(np.array_equal(np.array(defects), ref.defects)), defects))
        dist.barrier()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("W,Np,K,tol", [(2, 2, 1, 0.0), (2, 2, 2, 0.0), (2, 4, 2, 0.0), (2, 4, 3, 0.0),
                                        (4, 4, 2, 0.0), (2, 4, 4, 3e-3), (2, 4, 4, 1e-6), (4, 4, 4, 1e-6),
                                        (8, 8, 3, 0.0)])  # the bench's 8-GPU schedule
def test_pipelined_plan_matches_serial_alg1(W, Np, K, tol, orc):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=worker, args=(r, W, port, Np, K, q, tol)) for r in range(W)]
    for pp in procs:
        pp.start()
    res = q.get(timeout=300)
    for pp in procs:
        pp.join(timeout=120)
        assert pp.exitcode == 0
    same_u, same_d, d = res
    assert same_u, "u_T differs from the serial Alg.1 emulation"
    assert same_d, d
    if K >= Np and tol == 0.0:
        assert d[Np] == 0.0  # finite-step exactness
