"""Pins for the speedup model used in bench reports (paper_1409_8563_b200/perfmodel.py)
against Table 1 (tests/golden/table1.json) and its algebraic identities."""
import json
import os

import numpy as np
import pytest

from paper_1409_8563_b200 import perfmodel as pm

T1 = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "table1.json")))


@pytest.mark.parametrize("backend", ["cpu", "gpu"])
def test_eq_speedup_reproduces_table1(backend):
    """One tau_c/tau_f, back-solved from the N_p = 8 row's E_bound, reproduces
    the S_bound / E_bound columns of every other row (to the printed rounding
    plus the spread of the single-node ratio) — only the pipelined Eq.(speedup)
     does; the north_star non-pipelined form does not."""
    K, q = T1["K"], T1["nc_over_nf"]
    rows = T1[backend]["rows"]
    n8 = [r for r in rows if r[0] == 8][0]
    r = pm.backsolve_ratio(n8[3] / 100 * 8, 8, K, q)
    assert 0.14 < r < 0.2
    for Np, Sb, Sm, Eb, Em in rows:
        S = pm.speedup_bound(Np, K, 1, 16, r, 1.0)
        assert abs(S - Sb) <= 0.05 * Sb + 0.05, (Np, S, Sb)
        assert abs(100 * pm.efficiency(S, Np) - Eb) <= 2.0, (Np, S, Eb)
    # the non-pipelined variant misses the large-N_p rows badly
    S128 = pm.speedup_bound_northstar(128, K, 1, 16, r, 1.0)
    assert S128 < 0.6 * [x for x in rows if x[0] == 128][0][1]


def test_cost_identities():
    rng = np.random.default_rng(0)
    for _ in range(1000):
        Np, K = int(rng.integers(1, 257)), int(rng.integers(1, 9))
        nc, nf = int(rng.integers(1, 64)), int(rng.integers(64, 4096))
        tc, tf = float(rng.uniform(1e-4, 1.0)), float(rng.uniform(1e-4, 1.0))
        Cf = pm.cost_serial(Np, nf, tf)
        Cp = pm.cost_parareal(Np, K, nc, tc, nf, tf)
        S = pm.speedup_bound(Np, K, nc, nf, tc, tf)
        assert abs(S - Cf / Cp) <= 1e-12 * S
        b1, b2 = pm.corollary_bounds(Np, K, nc, nf, tc, tf)
        assert S <= b1 * (1 + 1e-12) and S <= b2 * (1 + 1e-12)
        assert abs(pm.gamma_bound(Np, S) * S - Np) <= 1e-9 * Np  # Eq.(gamma_expected)
    # SPEC examples
    assert pm.cost_serial(4, 10, 0.5) == 20
    assert pm.cost_parareal(4, 3, 2, 1.0, 8, 1.0) == 38
    assert pm.speedup_bound(8, 2, 1, 16, 0.0, 1.0) == 4.0
