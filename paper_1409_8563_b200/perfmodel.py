"""Cost, speedup and efficiency model of Sec. 2.2.1-2.2.2 (host-side report
helper; no part of the compute path).

  C_f = N_t tau_f = N_p N_f tau_f                                 Eq.(cost_serial)
  C_p = (N_p + K) N_c tau_c + K N_f tau_f                         Eq.(cost_parareal)
  S_bound = C_f / C_p
          = 1 / ((1 + K/N_p) (N_c/N_f) (tau_c/tau_f) + K/N_p)     Eq.(speedup)
  S_bound <= N_p / K  and  S_bound <= (N_f/N_c)(tau_f/tau_c)
  E = S / N_p                                                     Eq.(efficiency)
  gamma_bound = N_p / S_bound                                     Eq.(gamma_expected)

north_star also quotes N/((1+K) N c_G/c_F + K) with c_G = N_c tau_c and
c_F = N_f tau_f: the non-pipelined variant (every iteration re-runs all N
coarse slices).  It is reported beside Eq.(speedup) (reading C21).
"""
from __future__ import annotations


def cost_serial(n_p: int, n_f: int, tau_f: float) -> float:
    return n_p * n_f * tau_f


def cost_parareal(n_p: int, K: int, n_c: int, tau_c: float, n_f: int, tau_f: float) -> float:
    return (n_p + K) * n_c * tau_c + K * n_f * tau_f


def speedup_bound(n_p: int, K: int, n_c: int, n_f: int, tau_c: float, tau_f: float) -> float:
    return 1.0 / ((1.0 + K / n_p) * (n_c / n_f) * (tau_c / tau_f) + K / n_p)


def speedup_bound_northstar(n_p: int, K: int, n_c: int, n_f: int, tau_c: float, tau_f: float) -> float:
    cg_cf = (n_c * tau_c) / (n_f * tau_f)
    return n_p / ((1.0 + K) * n_p * cg_cf + K)


def corollary_bounds(n_p: int, K: int, n_c: int, n_f: int, tau_c: float, tau_f: float):
    return n_p / K if K else float("inf"), (n_f / n_c) * (tau_f / tau_c)


def efficiency(speedup: float, n_p: int) -> float:
    return speedup / n_p


def gamma_bound(n_p: int, s_bound: float) -> float:
    return n_p / s_bound


def backsolve_ratio(S: float, n_p: int, K: int, n_c_over_n_f: float) -> float:
    """tau_c/tau_f that makes Eq.(speedup) equal S (used to read Table 1)."""
    return (1.0 / S - K / n_p) / ((1.0 + K / n_p) * n_c_over_n_f)
