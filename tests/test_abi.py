"""C-ABI checks that run without a GPU: the library loads, exports every
symbol include/parareal.h declares, and its host-only logic (the Alg.1
schedule, the stability ratio, error reporting) behaves as documented."""
import ctypes
import os
import re

import pytest

import paper_1409_8563_b200 as pr
from paper_1409_8563_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "parareal.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(pr_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    L = _lib.load()
    decl = declared_symbols()
    assert len(decl) >= 14
    for name in decl:
        assert hasattr(L, name), name
    assert sorted(decl) == sorted(_lib.EXPORTS)


def test_version_and_no_gpu_error():
    assert "sm_100a" in pr.pr_version()
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(pr.PrError) as e:
        pr.Grid(pr.Problem(32))
    assert e.value.status in (_lib.PR_ECUDA, _lib.PR_EINVAL)


def test_create_grid_rejects_bad_problems():
    for bad in (pr.Problem(7), pr.Problem(2), pr.Problem(32, nu0=-1.0), pr.Problem(32, T=0.0),
                pr.Problem(32, nu_mode=5)):
        with pytest.raises(pr.PrError) as e:
            pr.Grid(bad)
        assert e.value.status == _lib.PR_EINVAL


def plan_counts(plan):
    out = {}
    for op, *_ in plan:
        out[op] = out.get(op, 0) + 1
    return out


@pytest.mark.parametrize("Np,W", [(1, 1), (4, 1), (4, 2), (4, 4), (8, 8), (8, 2)])
@pytest.mark.parametrize("K", [0, 1, 3])
def test_plan_structure(Np, W, K):
    """Alg.1 per rank: p+1 coarse sweeps at init (C9), then per
    iteration F on every own slice, one receive (not rank 0), G + correction per
    slice, one send (not the last rank)."""
    s = Np // W
    for r in range(W):
        plan = pr.pr_plan(Np, K, W, r)
        c = plan_counts(plan)
        assert c.get("G_PREFIX", 0) == r * s
        assert c.get("G_INIT", 0) == s
        assert c.get("G_PREFIX", 0) + c["G_INIT"] == (r + 1) * s   # last rank: N_p sweeps
        assert c.get("F", 0) == K * s and c.get("G", 0) == K * s and c.get("CORRECT", 0) == K * s
        assert c.get("RECV", 0) == (K if r > 0 else 0)
        assert c.get("SEND", 0) == (K if r < W - 1 else 0)
        assert c.get("DEFECT0", 0) == (1 if r == W - 1 else 0)
        # order inside an iteration: all F, then (recv), G, correct, ..., (send), end
        for k in range(K):
            it = [p for p in plan if p[1] == k]
            names = [p[0] for p in it]
            assert names[:s] == ["F"] * s
            assert names[-1] == "END_ITER"
            if r > 0:
                assert names[s] == "RECV" and it[s][3] == r - 1 and it[s][2] == r * s
            if r < W - 1:
                assert names[-2] == "SEND" and it[-2][3] == r + 1 and it[-2][2] == r * s + s - 1


def test_plan_sends_match_receives():
    """Every send of rank r in iteration k has the matching receive on r+1
    (pipelined order, no deadlock: the dependency chain only points forward)."""
    Np, K, W = 8, 3, 4
    sends = [(r, k) for r in range(W) for (op, k, sl, peer) in pr.pr_plan(Np, K, W, r) if op == "SEND"]
    recvs = [(peer, k) for r in range(W) for (op, k, sl, peer) in pr.pr_plan(Np, K, W, r) if op == "RECV"]
    assert sorted(sends) == sorted(recvs)


def test_plan_rejects_bad_sizes():
    for args in ((0, 1, 1, 0), (4, -1, 1, 0), (4, 1, 3, 0), (4, 1, 2, 2), (4, 1, 0, 0)):
        with pytest.raises(pr.PrError) as e:
            pr.pr_plan(*args)
        assert e.value.status == _lib.PR_EINVAL


def test_stability_ratio():
    """Euler limit dt (6 nu_max/dx^2 + sum|c|/dx) (positivity bound).
    The paper's 128^3 coarse step T/2^11 sits at ~0.74 of it; T/2^11 at 256^3
    exceeds it (the reason cfg3 uses 2^13 coarse steps)."""
    r128 = pr.pr_stability_ratio(pr.Problem(128), 0.1 / 2 ** 11, fine=False)
    assert abs(r128 - 0.1 / 2 ** 11 * (6 * 0.15 * 128 ** 2 + 3 * 128)) < 1e-12
    assert 0.7 < r128 < 0.8
    assert pr.pr_stability_ratio(pr.Problem(256), 0.1 / 2 ** 11, fine=False) > 1.0
    assert pr.pr_stability_ratio(pr.Problem(256), 0.1 / 2 ** 13, fine=False) < 1.0
    rf = pr.pr_stability_ratio(pr.Problem(128), 0.1 / 2 ** 15, fine=True)
    assert 0.0 < rf < 0.1


def test_kernel_launch_counter_starts_at_zero_without_gpu():
    assert pr.pr_kernel_launches() >= 0
