"""Multi-rank Parareal on ONE GPU: W ranks as grids of one process linked by
pr_local_group, each driven by its own host thread (ctypes releases the GIL).

This exercises every rank-dependent step of Alg.1 that a 1-GPU box
can run: the redundant coarse prefix of ranks r > 0 (R4), the
hand-off in the paper's pipelined order (R7) with the peer-store
data path (the correction kernel writes u^{k+1} into the successor's receive
buffer), the alternating receive buffers and the buffer rotation of END_ITER,
the successor's release of its receive buffer, the stop-flag propagation of
convergence control (C23), and the slice groups of N_p > W.  Ordering is by
CUDA events announced between the ranks' host threads, so no stream or kernel
ever waits on another rank's unannounced value (ranks that spin on each other
as separate processes on one GPU are unsafe on this pool).

Pins: u_T and d^k bitwise equal to the 1-rank slice-group run of the same N_p
slices (W-invariance: the hand-off is a byte copy), and within 1e-12 / 1e-10
of the oracle (Alg.1 serialised, oracle.parareal / parareal_tol)."""
import threading

import numpy as np
import pytest

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import oracle
import paper_1409_8563_b200 as pr

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True)
def _handoff_timeout(monkeypatch):
    """A protocol error shows up as PR_ENCCL within a minute, not as a hang."""
    monkeypatch.setenv("PR_NCCL_TIMEOUT_S", "60")


def horizon(n):
    """cfg1-style step counts (the paper's Euler CFL ~0.73 at every n)."""
    if n <= 64:
        return 0.1, 2048 * (n // 32) ** 2, 128 * (n // 32) ** 2
    return 0.1 / 64, 2 ** 11, 2 ** 7


def run_group(n, Np, K, W, tol=0.0, flags=0, calls=2, nf=None, nc=None, T=None, devices=None):
    """All W ranks of one pr_local_group (on cuda:0, or rank r on devices[r]); returns the
    last rank's (u_T, defects) per call, per-rank iteration counts and the serial fine u_ref."""
    T0, Nt, NC = horizon(n)
    if T is not None:
        T0 = T
    if nf is not None:
        Nt, NC = nf * Np, nc * Np
    devices = devices or [0] * W
    grids = [pr.Grid(pr.Problem(n, T=T0), devices[r]) for r in range(W)]
    pr.pr_local_group(grids)
    u0 = torch.empty((n, n, n), dtype=torch.float64, device="cuda:0")
    with pr.Grid(pr.Problem(n, T=T0), 0) as g0:
        pr.pr_fill_sine(g0, u0)
        uf = torch.empty_like(u0)
        pr.pr_fine(g0, u0, uf, 0, Nt, T0 / Nt)
    torch.cuda.synchronize()
    # every rank's own copy of u0 on its device; the last rank's u_ref there too
    u0s = [u0.to(f"cuda:{d}") for d in devices]
    ufl = uf.to(f"cuda:{devices[-1]}")
    cfg = pr.PararealCfg(Np, NC // Np, Nt // Np, K, flags=flags, tol=tol)
    outs = [[None] * calls for _ in range(W)]
    iters = [[None] * calls for _ in range(W)]
    errs = [None] * W
    streams = [torch.cuda.Stream(device=f"cuda:{d}") for d in devices]

    def worker(r):
        try:
            last = r == W - 1
            for c in range(calls):
                uT = torch.empty_like(u0s[r]) if last else None
                d = pr.pr_parareal(grids[r], cfg, u0s[r], uT, ufl if last else None,
                                   stream=streams[r].cuda_stream)
                iters[r][c] = pr.pr_last_monitors(grids[r])[1]
                outs[r][c] = (uT, d)
        except Exception as e:  # reported by the main thread
            errs[r] = e

    th = [threading.Thread(target=worker, args=(r,), daemon=True) for r in range(W)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=240)
    assert not any(t.is_alive() for t in th), ("a rank hung", errs)
    assert not any(errs), errs
    torch.cuda.synchronize()
    # 1-rank reference: the same N_p slices as one slice group
    with pr.Grid(pr.Problem(n, T=T0), 0) as g1:
        uT1 = torch.empty_like(u0)
        d1 = pr.pr_parareal(g1, cfg, u0, uT1, uf)
        it1 = pr.pr_last_monitors(g1)[1]
    for g in grids:
        g.destroy()
    res = [(uT.to("cuda:0"), d) for uT, d in outs[W - 1]]
    return res, [iters[r][0] for r in range(W)], (uT1, d1, it1), uf, (T0, Nt, NC)


def same(a, b):
    a, b = np.asarray(a, dtype=float), np.asarray(b, dtype=float)
    return a.shape == b.shape and bool(np.array_equal(a, b, equal_nan=True))


CASES = [  # W, n, N_p, K
    (2, 32, 2, 2), (2, 32, 4, 2), (2, 40, 4, 3), (4, 32, 4, 3), (4, 32, 8, 3), (8, 32, 8, 3),
    (8, 32, 16, 2), (3, 32, 6, 2), (2, 128, 2, 1), (4, 64, 8, 2), (4, 32, 4, 0),
]


@pytest.mark.parametrize("W,n,Np,K", CASES)
def test_local_ranks_match_single_rank_and_oracle(W, n, Np, K):
    """Two calls per rank group (the second reuses every buffer at the next
    sequence epoch): bitwise the 1-rank slice-group run; the oracle at small n."""
    res, _, (uT1, d1, _), _, (T, Nt, NC) = run_group(n, Np, K, W)
    for uT, d in res:
        assert torch.equal(uT, uT1) and same(d, d1), (W, n, Np, K)
    if n <= 48:
        p = oracle.Problem(n, T=T)
        o0 = oracle.initial(n)
        ouf = oracle.serial_fine(p, Nt, o0)
        ref = oracle.parareal(p, Np, NC // Np, Nt // Np, K, o0, ouf)
        uT, d = res[0]
        err = float(np.max(np.abs(uT.cpu().numpy() - ref.u_T)) / np.max(np.abs(ref.u_T)))
        assert err <= 1e-12, err
        assert np.max(np.abs(np.array(d) - ref.defects)) <= 1e-10


@pytest.mark.parametrize("W,Np,K,tol", [(2, 4, 4, 3e-3), (4, 4, 4, 3e-3), (4, 8, 6, 1e-4), (8, 8, 8, 3e-3)])
def test_local_ranks_convergence_control(W, Np, K, tol):
    """Stopping rule C23 across ranks: per-rank iteration counts and u_T equal
    the oracle's pipelined stop rule (orc_parareal_tol with the same world)."""
    n = 32
    res, iters, _, _, (T, Nt, NC) = run_group(n, Np, K, W, tol=tol)
    p = oracle.Problem(n, T=T)
    o0 = oracle.initial(n)
    ouf = oracle.serial_fine(p, Nt, o0)
    ref = oracle.parareal_tol(p, Np, NC // Np, Nt // Np, K, tol, W, o0, ouf)
    assert [int(x) for x in ref.iters] == iters
    for uT, d in res:
        err = float(np.max(np.abs(uT.cpu().numpy() - ref.u_T)) / np.max(np.abs(ref.u_T)))
        assert err <= 1e-12, err
    assert same(res[0][1], res[1][1])


def test_local_ranks_half_mesh_g():
    """G on the n/2 mesh (NEXT-4) across 4 ranks: bitwise the 1-rank run."""
    res, _, (uT1, d1, _), _, _ = run_group(32, 4, 2, 4, flags=pr.PR_FLAG_G_HALF_MESH)
    for uT, d in res:
        assert torch.equal(uT, uT1) and same(d, d1)


def test_local_handoff_stress():
    """8 ranks x K = 256 iterations = 1792 hand-offs through the alternating
    receive buffers: bitwise the 1-rank run, and (K >= N_p, C5 + C6) bitwise the
    serial fine solution."""
    n, W, Np, K = 32, 8, 8, 256
    res, _, (uT1, d1, _), uf, _ = run_group(n, Np, K, W, nf=4, nc=1, T=8 * 4 * 2e-4, calls=1)
    uT, d = res[0]
    assert torch.equal(uT, uT1) and same(d, d1)
    assert torch.equal(uT, uf)
    assert d[-1] == 0.0


def _lone_rank(W, run_rank, monkeypatch):
    monkeypatch.setenv("PR_NCCL_TIMEOUT_S", "2")
    n = 32
    grids = [pr.Grid(pr.Problem(n), 0) for _ in range(W)]
    pr.pr_local_group(grids)
    u0 = torch.empty((n, n, n), dtype=torch.float64, device="cuda")
    pr.pr_fill_sine(grids[0], u0)
    last = run_rank == W - 1
    with pytest.raises(pr.PrError) as ei:
        pr.pr_parareal(grids[run_rank], pr.PararealCfg(W, 4, 16, 2), u0,
                       torch.empty_like(u0) if last else None, None)
    for g in grids:
        g.destroy()
    return ei.value


def test_stuck_predecessor_fails_with_rank_and_iteration(monkeypatch):
    """A successor whose predecessor never delivers returns PR_ENCCL after the
    hand-off timeout, naming its rank and iteration (SURVEY 8(b) errors)."""
    e = _lone_rank(2, 1, monkeypatch)
    assert e.status == pr._lib.PR_ENCCL
    assert "rank 1, iteration 0" in str(e) and "rank 0" in str(e), str(e)


def test_stuck_successor_fails_with_rank_and_iteration(monkeypatch):
    """A predecessor whose successor never starts its call cannot hand off."""
    e = _lone_rank(2, 0, monkeypatch)
    assert e.status == pr._lib.PR_ENCCL
    assert "rank 0, iteration 0" in str(e) and "rank 1" in str(e), str(e)


@pytest.mark.parametrize("per_gpu", [1, 2])
def test_local_group_across_gpus(per_gpu):
    """One process driving ranks on several GPUs (rank r on device r % G): the
    correction kernel stores the hand-off into the next GPU's memory through a peer
    mapping (cudaDeviceEnablePeerAccess); with 2 ranks per GPU the 8-rank executor
    of an 8-GPU run is exercised on a 4-GPU box.  Bitwise the 1-rank run; oracle."""
    G = torch.cuda.device_count()
    if G < 2:
        pytest.skip("needs 2 GPUs")
    W = G * per_gpu
    res, _, (uT1, d1, _), _, (T, Nt, NC) = run_group(32, W, 3, W, devices=[r % G for r in range(W)])
    for uT, d in res:
        assert torch.equal(uT, uT1) and same(d, d1)
    p = oracle.Problem(32, T=T)
    o0 = oracle.initial(32)
    ref = oracle.parareal(p, W, NC // W, Nt // W, 3, o0, oracle.serial_fine(p, Nt, o0))
    err = float(np.max(np.abs(res[0][0].cpu().numpy() - ref.u_T)) / np.max(np.abs(ref.u_T)))
    assert err <= 1e-12, err


def test_local_group_argument_errors():
    """pr_local_group rejects an empty group and a grid listed twice (PR_EINVAL)."""
    g = pr.Grid(pr.Problem(32), 0)
    with pytest.raises(pr.PrError) as ei:
        pr.pr_local_group([g, g])
    assert ei.value.status == pr._lib.PR_EINVAL
    with pytest.raises(pr.PrError) as ei:
        pr.pr_local_group([])
    assert ei.value.status == pr._lib.PR_EINVAL
    g.destroy()


def test_local_group_rank_count_must_divide_slices():
    """N_p must be a multiple of the group size, as with NCCL ranks (PR_EINVAL)."""
    grids = [pr.Grid(pr.Problem(32), 0) for _ in range(3)]
    pr.pr_local_group(grids)
    u0 = torch.empty((32, 32, 32), dtype=torch.float64, device="cuda")
    pr.pr_fill_sine(grids[0], u0)
    with pytest.raises(pr.PrError) as ei:
        pr.pr_parareal(grids[0], pr.PararealCfg(4, 4, 16, 1), u0, None, None)
    assert ei.value.status == pr._lib.PR_EINVAL
    for g in grids:
        g.destroy()


@pytest.mark.parametrize("W", [2, 4, 8])
def test_local_liveness_sweep(W):
    """SURVEY T5 on one GPU: every (N_p, K) with N_p in {W, 2W} and K in {0, 1, 2, 5, 8}
    (K > N_p included) completes without a hang, bitwise equal to the 1-rank run."""
    n = 8
    for Np in (W, 2 * W):
        for K in (0, 1, 2, 5, 8):
            res, _, (uT1, d1, _), _, _ = run_group(n, Np, K, W, nf=2, nc=1, T=Np * 2 * 1e-3, calls=1)
            uT, d = res[0]
            assert torch.equal(uT, uT1) and same(d, d1), (W, Np, K)
