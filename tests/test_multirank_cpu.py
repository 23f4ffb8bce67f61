"""World-size-2 (and 4) CPU test of the multi-rank host logic over torch.distributed
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


def execute_plan(plan, rank, W, Np, nc, nf, p, orc, u0, u_ref):
    """Python mirror of pr_parareal's executor: same buffer roles, same order."""
    s, j0 = Np // W, rank * (Np // W)
    Dt, dt = p.T / (Np * nc), p.T / (Np * nf)
    G = lambda u, m: orc.coarse(p, u, m * nc, nc, Dt)
    F = lambda u, m: orc.fine(p, u, m * nf, nf, dt)
    start, f, out, gold, used = [None] * s, [None] * s, [None] * s, [None] * s, [None] * s
    v, recvb, gnew, defects = u0, None, None, []
    for op, k, sl, peer in plan:
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
            t = torch.empty(u0.shape, dtype=torch.float64)
            dist.recv(t, src=peer)
            recvb = t.numpy()
        elif op == "G":
            used[l] = u0 if sl == 0 else (recvb if l == 0 else out[l - 1])
            gnew = G(used[l], sl)
        elif op == "CORRECT":
            out[l] = f[l] + (gnew - gold[l])
            gold[l] = gnew
            if sl == Np - 1:
                defects.append(orc.defect(out[l], u_ref))
        elif op == "SEND":
            dist.send(torch.from_numpy(np.ascontiguousarray(out[l])), dst=peer)
        elif op == "END_ITER":
            start = list(used)
    K = sum(1 for q in plan if q[0] == "END_ITER")
    return (out[s - 1] if K > 0 else gold[s - 1]), defects


def worker(rank, W, port, Np, K, q):
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
        uT, defects = execute_plan(plan, rank, W, Np, nc, nf, p, oracle, u0, u_ref)
        if rank == W - 1:
            ref = oracle.parareal(p, Np, nc, nf, K, u0, u_ref)
            q.put((bool(np.array_equal(uT, ref.u_T)),
                   bool(np.array_equal(np.array(defects), ref.defects)), defects))
        dist.barrier()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("W,Np,K", [(2, 2, 1), (2, 2, 2), (2, 4, 2), (2, 4, 3), (4, 4, 2)])
def test_pipelined_plan_matches_serial_alg1(W, Np, K, orc):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=worker, args=(r, W, port, Np, K, q)) for r in range(W)]
    for pp in procs:
        pp.start()
    res = q.get(timeout=300)
    for pp in procs:
        pp.join(timeout=120)
        assert pp.exitcode == 0
    same_u, same_d, d = res
    assert same_u, "u_T differs from the serial Alg.1 emulation"
    assert same_d, d
    if K >= Np:
        assert d[Np] == 0.0  # finite-step exactness
