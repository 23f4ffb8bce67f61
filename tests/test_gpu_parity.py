"""GPU parity: the CUDA path (through the C ABI) vs the CPU oracle on the same
seeded inputs.  Tolerance (north_star; C13/C14): normwise
max|gpu - oracle| / max|oracle| <= 1e-12 on fields, |d_gpu - d_oracle| <= 1e-10
on defects.  Sizes span several tiles (32 x 16 in x, y; z chunks) and ragged
tails (n = 40, 48), non-powers of two (12), tiny grids whose tile wraps the
domain several times (n = 4, 8), and the full BASELINE sizes on a few steps."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import oracle
import paper_1409_8563_b200 as pr
from synthetic import random_field, PARITY_C

pytestmark = pytest.mark.gpu
TOL = 1e-12


def rel(a, b):
    a = a.cpu().numpy() if hasattr(a, "cpu") else a
    return float(np.max(np.abs(a - b)) / np.max(np.abs(b)))


def dev(x):
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


_grids = {}


def grid(n, c=PARITY_C, nu0=0.1, omega=100.0, T=0.1, nu_mode=0):
    key = (n, tuple(c), nu0, omega, T, nu_mode)
    if key not in _grids:
        _grids[key] = pr.Grid(pr.Problem(n, c=c, nu0=nu0, omega=omega, T=T, nu_mode=nu_mode))
    return _grids[key]


def oproblem(n, c=PARITY_C, nu0=0.1, omega=100.0, T=0.1, nu_mode=0):
    return oracle.Problem(n, c=c, nu0=nu0, omega=omega, T=T, nu_mode=nu_mode)


@pytest.mark.parametrize("n", [4, 8, 12, 32, 40, 48, 64, 96])
@pytest.mark.parametrize("nu_mode", [0, 1])
def test_fine_steps(n, nu_mode):
    u0 = random_field(n, 0)
    g = grid(n, nu_mode=nu_mode)
    dt = 2e-4 * (32 / n) ** 2
    for step0, steps in ((0, 1), (7, 3), (100, 21)):  # 21 > one 16-step graph + remainder
        out = torch.empty((n, n, n), dtype=torch.float64, device="cuda")
        pr.pr_fine(g, dev(u0), out, step0, steps, dt)
        ref = oracle.fine(oproblem(n, nu_mode=nu_mode), u0, step0, steps, dt)
        assert rel(out, ref) <= TOL, (n, step0, steps)


@pytest.mark.parametrize("n", [4, 8, 12, 32, 40, 48, 64])
def test_coarse_steps(n):
    u0 = random_field(n, 1)
    g = grid(n)
    Dt = 5e-4 * (32 / n) ** 2
    for step0, steps in ((0, 1), (3, 2), (5, 7), (9, 40), (0, 33)):
        out = torch.empty((n, n, n), dtype=torch.float64, device="cuda")
        pr.pr_coarse(g, dev(u0), out, step0, steps, Dt)
        ref = oracle.coarse(oproblem(n), u0, step0, steps, Dt)
        assert rel(out, ref) <= TOL, (n, step0, steps)


@pytest.mark.parametrize("which", ["fine", "coarse"])
@pytest.mark.parametrize("steps", [0, 1, 2, 5, 34])
def test_in_place_and_zero_steps(which, steps):
    n = 32
    u0 = random_field(n, 2)
    g = grid(n)
    dt = 1e-4
    fn = pr.pr_fine if which == "fine" else pr.pr_coarse
    ofn = oracle.fine if which == "fine" else oracle.coarse
    u = dev(u0)
    fn(g, u, u, 11, steps, dt)
    ref = ofn(oproblem(n), u0, 11, steps, dt)
    if steps == 0:
        assert np.array_equal(u.cpu().numpy(), u0)
    else:
        assert rel(u, ref) <= TOL


@pytest.mark.parametrize("c", [(1.0, 1.0, 1.0), (-1.0, -0.5, 0.0), (0.0, 0.0, 0.0), (0.3, -2.0, 1.5)])
def test_velocity_signs(c):
    """Both upwind branches and c_a = 0 (strict > test, C4)."""
    n = 32
    u0 = random_field(n, 3)
    g = grid(n, c=c)
    for which, fn, ofn, dt in (("f", pr.pr_fine, oracle.fine, 1e-4), ("g", pr.pr_coarse, oracle.coarse, 4e-4)):
        out = torch.empty_like(dev(u0))
        fn(g, dev(u0), out, 0, 5, dt)
        assert rel(out, ofn(oproblem(n, c=c), u0, 0, 5, dt)) <= TOL, which


def test_host_pointers():
    """pr_fine / pr_coarse / pr_defect accept host buffers (staged internally)."""
    n = 32
    u0 = random_field(n, 4)
    g = grid(n)
    out = np.empty_like(u0)
    pr.pr_fine(g, u0, out, 3, 4, 1e-4)
    assert rel(out, oracle.fine(oproblem(n), u0, 3, 4, 1e-4)) <= TOL
    pr.pr_coarse(g, u0, out, 3, 5, 4e-4)
    assert rel(out, oracle.coarse(oproblem(n), u0, 3, 5, 4e-4)) <= TOL
    v = random_field(n, 5)
    assert abs(pr.pr_defect(g, v, u0) - oracle.defect(v, u0)) <= 1e-15


def test_fill_sine_defect_correct():
    n = 48
    g = grid(n)
    u = torch.empty((n, n, n), dtype=torch.float64, device="cuda")
    pr.pr_fill_sine(g, u)
    assert rel(u, oracle.initial(n)) <= 1e-15
    a, b, c, r = (random_field(n, s) for s in (6, 7, 8, 9))
    out = torch.empty_like(u)
    d = pr.pr_correct(g, dev(a), dev(b), dev(c), out, dev(r))
    exp = a + (b - c)
    assert np.array_equal(out.cpu().numpy(), exp)  # elementwise, C5 order: bitwise
    assert d == oracle.defect(exp, r)
    assert pr.pr_defect(g, dev(a), dev(r)) == oracle.defect(a, r)
    bad = dev(a)
    bad[3, 4, 5] = float("nan")
    assert np.isnan(pr.pr_defect(g, bad, dev(r)))
    with pytest.raises(pr.PrError) as e:
        pr.pr_defect(g, dev(a), torch.zeros_like(u))
    assert e.value.status == 5  # PR_EDOMAIN


def test_errors():
    g = grid(32)
    u = torch.zeros((32, 32, 32), dtype=torch.float64, device="cuda")
    with pytest.raises(pr.PrError):
        pr.pr_fine(g, u, u, 0, -1, 1e-4)
    with pytest.raises(pr.PrError):
        pr.pr_fine(g, u, u, 0, 1, 0.0)
    big = torch.zeros(2 * 32 ** 3, dtype=torch.float64, device="cuda")
    with pytest.raises(pr.PrError):  # overlapping but not identical
        pr.pr_coarse(g, big[:32 ** 3], big[8:8 + 32 ** 3], 0, 1, 1e-4)
    for bad in (pr.PararealCfg(0, 2, 2, 1), pr.PararealCfg(2, 0, 2, 1), pr.PararealCfg(2, 2, 2, -1)):
        with pytest.raises(pr.PrError) as e:
            pr.pr_parareal(g, bad, u, u)
        assert e.value.status == 1  # PR_EINVAL


# ----------------------------------------------------------------- Parareal
def cfg1_oracle(nu_mode):
    n, Nt, NC, Np, K = 32, 2048, 128, 4, 2
    p = oracle.Problem(n, nu_mode=nu_mode)
    u0 = oracle.initial(n)
    uf = oracle.serial_fine(p, Nt, u0)
    res = oracle.parareal(p, Np, NC // Np, Nt // Np, K, u0, uf)
    return p, u0, uf, res


@pytest.fixture(scope="module")
def cfg1_ref():
    return {m: cfg1_oracle(m) for m in (0, 1)}


@pytest.mark.parametrize("nu_mode", [0, 1])
def test_parareal_cfg1(cfg1_ref, nu_mode):
    """BASELINE configs[0]: 32^3, 4 slices, K=2 on one GPU (slice group s = 4)."""
    p, u0, uf, res = cfg1_ref[nu_mode]
    g = grid(32, c=(1.0, 1.0, 1.0), nu_mode=nu_mode)
    uf_g = torch.empty((32, 32, 32), dtype=torch.float64, device="cuda")
    pr.pr_fine(g, dev(u0), uf_g, 0, 2048, 0.1 / 2048)
    assert rel(uf_g, uf) <= TOL
    uT = torch.empty_like(uf_g)
    d = pr.pr_parareal(g, pr.PararealCfg(4, 32, 512, 2), dev(u0), uT, dev(uf))
    assert rel(uT, res.u_T) <= TOL
    assert np.max(np.abs(np.array(d) - res.defects)) <= 1e-10
    # host buffers through the same call (the e2e path)
    uT_h = np.empty_like(u0)
    d_h = pr.pr_parareal(g, pr.PararealCfg(4, 32, 512, 2), u0, uT_h, uf)
    assert np.array_equal(uT_h, uT.cpu().numpy()) and d_h == d


def test_parareal_exactness_and_degenerate():
    """K = N_p: u_T equals the GPU serial fine run bitwise (C5 + C6); G = F: d^1 = 0."""
    n, Np, nc, nf = 32, 4, 8, 32
    g = grid(n, T=0.01)
    u0 = dev(random_field(n, 12))
    uf = torch.empty_like(u0)
    pr.pr_fine(g, u0, uf, 0, Np * nf, 0.01 / (Np * nf))
    uT = torch.empty_like(u0)
    d = pr.pr_parareal(g, pr.PararealCfg(Np, nc, nf, Np), u0, uT, uf)
    assert torch.equal(uT, uf) and d[Np] == 0.0
    d = pr.pr_parareal(g, pr.PararealCfg(Np, nc, nf, 2, flags=pr.PR_FLAG_G_IS_F), u0, uT, uf)
    assert d[1] == 0.0 and d[2] == 0.0
    # K = 0: the coarse initial guess
    d = pr.pr_parareal(g, pr.PararealCfg(Np, nc, nf, 0), u0, uT, uf)
    ug = torch.empty_like(u0)
    pr.pr_coarse(g, u0, ug, 0, Np * nc, 0.01 / (Np * nc))
    assert torch.equal(uT, ug)


def test_parareal_small_random_vs_oracle():
    n, Np, nc, nf, K = 12, 3, 3, 10, 2
    p = oracle.Problem(n, c=PARITY_C, T=0.004)
    u0 = random_field(n, 13)
    uf = oracle.serial_fine(p, Np * nf, u0)
    ref = oracle.parareal(p, Np, nc, nf, K, u0, uf)
    g = grid(n, T=0.004)
    uT = torch.empty((n, n, n), dtype=torch.float64, device="cuda")
    d = pr.pr_parareal(g, pr.PararealCfg(Np, nc, nf, K), dev(u0), uT, dev(uf))
    assert rel(uT, ref.u_T) <= TOL
    assert np.max(np.abs(np.array(d) - ref.defects)) <= 1e-10


# ---------------------------------------------------------- full BASELINE sizes
@pytest.mark.parametrize("f2", ["1", "0"])
@pytest.mark.parametrize("n", [32, 64])
def test_fine_paths_agree(n, f2, monkeypatch):
    """Both F implementations (fused two-kernel step for tile-aligned n, four
    stage passes otherwise) against the oracle, odd/even step counts, in place."""
    monkeypatch.setenv("PR_F2", f2)
    g = pr.Grid(pr.Problem(n, c=PARITY_C))
    u0 = random_field(n, 30)
    p = oproblem(n)
    dt = 2e-4 * (32 / n) ** 2
    for step0, steps in ((0, 1), (3, 2), (5, 17), (2, 33), (1, 16)):
        out = torch.empty((n, n, n), dtype=torch.float64, device="cuda")
        pr.pr_fine(g, dev(u0), out, step0, steps, dt)
        assert rel(out, oracle.fine(p, u0, step0, steps, dt)) <= TOL, (step0, steps)
        u = dev(u0)
        pr.pr_fine(g, u, u, step0, steps, dt)
        assert torch.equal(u, out)
    g.destroy()


@pytest.mark.parametrize("n", [256])
def test_default_designs_bitwise_at_256(n, monkeypatch):
    """At the bench's size the two default designs (14 below 256^3, 23 from 256^3) and the
    four-stage path give the same bits over a few RK4 steps."""
    u0 = dev(random_field(n, 37))
    outs = []
    for f2, v in (("0", None), ("1", "14"), ("1", "23")):
        monkeypatch.setenv("PR_F2", f2)
        if v is None:
            monkeypatch.delenv("PR_FTILE", raising=False)
        else:
            monkeypatch.setenv("PR_FTILE", v)
        g = pr.Grid(pr.Problem(n, c=PARITY_C))
        out = torch.empty_like(u0)
        pr.pr_fine(g, u0, out, 3, 5, 1e-4 * (128 / n) ** 2)
        outs.append(out)
        g.destroy()
    assert torch.equal(outs[0], outs[1]) and torch.equal(outs[0], outs[2])


def test_default_fine_design_per_size(monkeypatch):
    """pr_grid_info names the two-kernel F design in use: the tensor-memory stage hand-off
    (23) from 256^3 up, the shared-memory one (14) below, PR_FTILE overriding both, 0 on the
    four-pass path (n not a multiple of 32)."""
    monkeypatch.delenv("PR_FTILE", raising=False)
    for n, want in ((128, 14), (256, 23), (40, 0)):
        g = pr.Grid(pr.Problem(n, c=PARITY_C))
        assert pr.pr_grid_info(g)["fine_variant"] == want, n
        g.destroy()
    monkeypatch.setenv("PR_FTILE", "14")
    g = pr.Grid(pr.Problem(256, c=PARITY_C))
    assert pr.pr_grid_info(g)["fine_variant"] == 14
    g.destroy()


@pytest.mark.parametrize("variant", [str(v) for v in list(range(10, 26)) + [29, 31, 32, 33, 34, 35, 36, 37, 38, 39, 40, 41, 42, 43, 44, 45]])
def test_fused_variants_bitwise(variant, monkeypatch):
    """Every persistent fused tile variant (PR_FTILE) gives the four-stage
    path's bits: same folded weights, same operation order per point.  n = 128
    has tiles on and away from the periodic seams (cp.async and TMA fills)."""
    n = 128
    u0 = dev(random_field(n, 31))
    outs = []
    for f2, v in (("0", None), ("1", variant)):
        monkeypatch.setenv("PR_F2", f2)
        if v is None:  # the four-stage path (no fused variant involved)
            monkeypatch.delenv("PR_FTILE", raising=False)
        else:
            monkeypatch.setenv("PR_FTILE", v)
        try:
            g = pr.Grid(pr.Problem(n, c=PARITY_C))
        except pr.PrError as e:  # a tuning variant not built (PRK_VARIANTS) or not fitting
            pytest.skip(str(e))
        out = torch.empty_like(u0)
        pr.pr_fine(g, u0, out, 3, 21, 1e-4)
        outs.append(out)
        g.destroy()
    assert torch.equal(outs[0], outs[1])


@pytest.mark.parametrize("variant", ["14", "23"])
@pytest.mark.parametrize("n", [128, 256])
def test_weights_as_parameters_bitwise(n, variant, monkeypatch):
    """Direct launches with the stage weights as kernel parameters (PR_WPARAM=1) give
    the bits of the CUDA-graph path (the default) that reads the weights
    from the device nu table (PR_WPARAM=0): fine_weights13 rounds every operation
    separately on host and device.  Odd and even step counts, in place and not."""
    u0 = dev(random_field(n, 61))
    outs = []
    for wp in ("0", "1"):
        monkeypatch.setenv("PR_FTILE", variant)
        monkeypatch.setenv("PR_WPARAM", wp)
        g = pr.Grid(pr.Problem(n, c=PARITY_C))
        res = []
        for step0, steps in ((5, 17), (100, 2)):
            out = torch.empty_like(u0)
            pr.pr_fine(g, u0, out, step0, steps, 1e-4 * (128 / n) ** 2)
            res.append(out)
        u = u0.clone()
        pr.pr_fine(g, u, u, 7, 3, 1e-4 * (128 / n) ** 2)
        res.append(u)
        outs.append(res)
        g.destroy()
    for a, b in zip(*outs):
        assert torch.equal(a, b)


@pytest.mark.parametrize("n", [128, 256])
def test_full_size_steps_vs_oracle(n):
    """Launch configuration bench.py times, a few steps, all n^3 outputs."""
    u0 = random_field(n, 20)
    g = grid(n, c=(1.0, 1.0, 1.0))
    p = oproblem(n, c=(1.0, 1.0, 1.0))
    dt, Dt = 0.1 / 2 ** 17 * (256 / n) ** 2, 0.1 / 2 ** 13 * (256 / n) ** 2
    out = torch.empty((n, n, n), dtype=torch.float64, device="cuda")
    pr.pr_fine(g, dev(u0), out, 1000, 2, dt)
    assert rel(out, oracle.fine(p, u0, 1000, 2, dt)) <= TOL
    pr.pr_coarse(g, dev(u0), out, 500, 3, Dt)
    assert rel(out, oracle.coarse(p, u0, 500, 3, Dt)) <= TOL


def test_cfg4_512_steps_vs_oracle():
    """cfg4 (512^3, 1 GiB per field; T = 0.1/32, N_t = 2^14, N_C = 2^10) in the
    launch configuration bench.py --config cfg4 times: one fine and one coarse step at a late
    step index, every output point against the oracle (≈ 3 s of 16-thread oracle work)."""
    n, T = 512, 0.1 / 32
    u0 = random_field(n, 21)
    g = pr.Grid(pr.Problem(n, c=(1.0, 1.0, 1.0), T=T))
    p = oproblem(n, c=(1.0, 1.0, 1.0), T=T)
    dt, Dt = T / 2 ** 14, T / 2 ** 10
    out = torch.empty((n, n, n), dtype=torch.float64, device="cuda")
    pr.pr_fine(g, dev(u0), out, 2 ** 14 - 1, 1, dt)
    assert rel(out, oracle.fine(p, u0, 2 ** 14 - 1, 1, dt)) <= TOL
    pr.pr_coarse(g, dev(u0), out, 2 ** 10 - 1, 1, Dt)
    assert rel(out, oracle.coarse(p, u0, 2 ** 10 - 1, 1, Dt)) <= TOL
    g.destroy()


@pytest.mark.parametrize("f2", ["1", "0"])
@pytest.mark.parametrize("n", [32, 64, 128])
def test_run_twice_bitwise(n, f2, monkeypatch):
    """Determinism (the race check available here: compute-sanitizer is closed on
    this pool): repeated F, G and Parareal runs give bitwise identical fields."""
    monkeypatch.setenv("PR_F2", f2)
    g = pr.Grid(pr.Problem(n, c=PARITY_C, T=0.001))
    u0 = dev(random_field(n, 40))
    outs = []
    for _ in range(3):
        f = torch.empty_like(u0)
        c = torch.empty_like(u0)
        pr.pr_fine(g, u0, f, 0, 19, 1e-6)
        pr.pr_coarse(g, u0, c, 0, 7, 4e-6)
        uT = torch.empty_like(u0)
        d = pr.pr_parareal(g, pr.PararealCfg(4, 2, 4, 2), u0, uT, f)
        outs.append((f, c, uT, d))
    for f, c, uT, d in outs[1:]:
        assert torch.equal(f, outs[0][0]) and torch.equal(c, outs[0][1])
        assert torch.equal(uT, outs[0][2]) and d == outs[0][3]
    g.destroy()


@pytest.mark.parametrize("pick", [1, 2])
def test_parareal_convergence_control(pick):
    """Convergence-controlled stopping (C23) on one GPU (slice group of
    4): same iteration count, monitors and u_T as the oracle's stop rule."""
    n, Np, nc, nf, K = 32, 4, 4, 16, 4
    p = oracle.Problem(n, c=PARITY_C, T=0.004)
    u0 = random_field(n, 50)
    uf = oracle.serial_fine(p, Np * nf, u0)
    full = oracle.parareal_tol(p, Np, nc, nf, K, 0.0, 1, u0, uf)
    ch = full.changes[0]
    tol = float(np.sqrt(ch[pick - 1] * ch[pick]))  # between two iterations, far from both
    ref = oracle.parareal_tol(p, Np, nc, nf, K, tol, 1, u0, uf)
    assert ref.iters[0] == pick + 1
    g = grid(n, T=0.004)
    uT = torch.empty((n, n, n), dtype=torch.float64, device="cuda")
    d = pr.pr_parareal(g, pr.PararealCfg(Np, nc, nf, K, tol=tol), dev(u0), uT, dev(uf))
    mon, iters = pr.pr_last_monitors(g)
    assert iters == pick + 1
    assert rel(uT, ref.u_T) <= TOL
    assert np.max(np.abs(np.array(mon) - ref.changes[0][:iters])) <= 1e-10
    assert np.allclose(np.array(d)[:iters + 1], ref.defects[:iters + 1], rtol=0, atol=1e-10)
    assert all(np.isnan(x) for x in d[iters + 1:])
    # without tol: K iterations and the same monitors as the oracle
    pr.pr_parareal(g, pr.PararealCfg(Np, nc, nf, K), dev(u0), uT, dev(uf))
    mon, iters = pr.pr_last_monitors(g)
    assert iters == K and np.max(np.abs(np.array(mon) - ch)) <= 1e-10


# ------------------------------------------- spatially coarsened G (NEXT-4)
@pytest.mark.parametrize("n", [8, 32, 40, 64, 128])
def test_coarse_mesh_steps(n):
    """pr_coarse_mesh (restriction, Alg.2 on the n/2 mesh, prolongation) vs the
    oracle's G_c, out of place and in place, odd and even step counts."""
    u0 = random_field(n, 50)
    g = grid(n)
    Dt = 5e-4 * (32 / n) ** 2
    for step0, steps in ((0, 1), (3, 2), (9, 37)):
        out = torch.empty((n, n, n), dtype=torch.float64, device="cuda")
        pr.pr_coarse_mesh(g, dev(u0), out, step0, steps, Dt)
        ref = oracle.coarse_mesh(oproblem(n), u0, step0, steps, Dt)
        assert rel(out, ref) <= TOL, (n, step0, steps)
        u = dev(u0)
        pr.pr_coarse_mesh(g, u, u, step0, steps, Dt)
        assert torch.equal(u, out)
    with pytest.raises(pr.PrError):
        pr.pr_coarse_mesh(grid(10), dev(random_field(10, 1)), torch.empty((10,) * 3, dtype=torch.float64,
                                                                           device="cuda"), 0, 1, Dt)


@pytest.mark.parametrize("K", [0, 2, 4])
def test_parareal_coarse_mesh_vs_oracle(K):
    """Alg.1 with G = G_c (PR_FLAG_G_HALF_MESH) against the oracle; K = N_p is exact."""
    n, Np, nc, nf = 32, 4, 8, 32
    p = oproblem(n, T=0.01)
    u0 = random_field(n, 51)
    uf = oracle.serial_fine(p, Np * nf, u0)
    ref = oracle.parareal(p, Np, nc, nf, K, u0, uf, g_half_mesh=True)
    g = grid(n, T=0.01)
    uT = torch.empty((n, n, n), dtype=torch.float64, device="cuda")
    d = pr.pr_parareal(g, pr.PararealCfg(Np, nc, nf, K, flags=pr.PR_FLAG_G_HALF_MESH), dev(u0), uT,
                       dev(uf))
    assert rel(uT, ref.u_T) <= TOL
    assert np.max(np.abs(np.array(d) - ref.defects)) <= 1e-10


@pytest.mark.parametrize("variant", ["0", "1", "2"])
@pytest.mark.parametrize("n", [32, 64, 128])
def test_coarse_kernels_bitwise(n, variant, monkeypatch):
    """The persistent TMA-fed G kernel (PR_CTILE variants) gives the lockstep
    stencil_kernel<K_COARSE>'s bits (same per-point operation order)."""
    u0 = dev(random_field(n, 52))
    outs = []
    for c2 in ("0", "1"):
        monkeypatch.setenv("PR_C2", c2)
        monkeypatch.setenv("PR_CTILE", variant)
        try:
            g = pr.Grid(pr.Problem(n, c=PARITY_C))
        except pr.PrError as e:  # a tuning variant not built (PRK_VARIANTS)
            pytest.skip(str(e))
        out = torch.empty_like(u0)
        pr.pr_coarse(g, u0, out, 5, 37, 4e-4 * (32 / n) ** 2)
        outs.append(out)
        g.destroy()
    assert torch.equal(outs[0], outs[1])


@pytest.mark.parametrize("n,Np,K", [(32, 4, 2), (64, 8, 3)])
def test_concurrent_slices_bitwise(n, Np, K, monkeypatch):
    """F over the slices of a group on concurrent streams (PR_CONC=1, one child grid per
    slice) gives the sequential run's bits, defects included (NEXT-2)."""
    u0 = dev(random_field(n, 53))
    res = []
    for conc in ("0", "1"):
        monkeypatch.setenv("PR_CONC", conc)
        g = pr.Grid(pr.Problem(n, c=PARITY_C, T=0.004))
        uf = torch.empty_like(u0)
        pr.pr_fine(g, u0, uf, 0, Np * 16, 0.004 / (Np * 16))
        uT = torch.empty_like(u0)
        d = pr.pr_parareal(g, pr.PararealCfg(Np, 4, 16, K), u0, uT, uf)
        res.append((uT, d))
        g.destroy()
    assert torch.equal(res[0][0], res[1][0]) and res[0][1] == res[1][1]


def test_nu_table_growth_keeps_graphs_consistent():
    """after a short pr_fine has cached CUDA graphs, a call long enough to
    outgrow the fine nu table (> 2^18 steps) reallocates it; every graph that captured
    the old table must be dropped (fused graphs included).  The long run must give the
    bits of the same run on a fresh grid."""
    n, steps, dt = 32, 270000, 2e-7
    u0 = dev(random_field(n, 71))
    g = pr.Grid(pr.Problem(n, c=PARITY_C))
    out = torch.empty_like(u0)
    pr.pr_fine(g, u0, out, 0, 64, dt)       # caches graphs on `out` with the first table
    pr.pr_fine(g, u0, out, 0, steps, dt)    # table grows past 1 << 20 doubles
    with pr.Grid(pr.Problem(n, c=PARITY_C)) as g2:
        ref = torch.empty_like(u0)
        pr.pr_fine(g2, u0, ref, 0, steps, dt)
    torch.cuda.synchronize()
    assert torch.equal(out, ref)
    g.destroy()


@pytest.mark.parametrize("nu0,omega", [(0.0, 0.0), (0.15, 0.0), (0.1, 100.0)])
@pytest.mark.parametrize("n", [12, 32, 128])
def test_nu_range_fine_and_coarse(n, nu0, omega):
    """SURVEY T2's nu range: pure advection (nu = 0), a constant nu = 0.15 and the paper's
    oscillating nu(t); the fused (n = 32, 128) and four-pass (n = 12) F paths and G
    against the oracle, 1e-12 normwise."""
    u0 = random_field(n, 81)
    g = grid(n, nu0=nu0, omega=omega)
    dt, Dt = 1e-4 * (32 / n) ** 2, 4e-4 * (32 / n) ** 2
    out = torch.empty((n, n, n), dtype=torch.float64, device="cuda")
    pr.pr_fine(g, dev(u0), out, 3, 19, dt)
    assert rel(out, oracle.fine(oproblem(n, nu0=nu0, omega=omega), u0, 3, 19, dt)) <= TOL
    pr.pr_coarse(g, dev(u0), out, 3, 7, Dt)
    assert rel(out, oracle.coarse(oproblem(n, nu0=nu0, omega=omega), u0, 3, 7, Dt)) <= TOL
