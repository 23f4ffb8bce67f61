"""Seeded synthetic inputs shared by the oracle tests, the GPU parity tests and
bench.py.  This module holds NO arithmetic of the method (no stencils, no time
stepping, no initial condition): only seeded random fields and the numeric
parameters of the configurations (DESIGN.md §4 "Input recipe").

Configurations restate BASELINE.json's configs with the step counts of
SURVEY.md §8(d) (coarse steps scaled with n^2 to keep the paper's Euler CFL
number of ~0.73; fine/coarse step ratio 16 as in the paper).
"""
from __future__ import annotations

from dataclasses import dataclass, asdict, replace

import numpy as np


def random_field(n: int, seed: int, shape=None) -> np.ndarray:
    """Uniform [-1, 1) fp64 field of shape (n, n, n) (z, y, x), numpy PCG64."""
    rng = np.random.Generator(np.random.PCG64(seed))
    shape = (n, n, n) if shape is None else shape
    return rng.uniform(-1.0, 1.0, size=shape).astype(np.float64)


# Velocity used by kernel-parity tests: both upwind branches, distinct axes.
PARITY_C = (1.0, -0.5, 0.25)


@dataclass(frozen=True)
class Config:
    name: str
    n: int
    T: float
    Nt: int          # total fine steps  (delta t = T / Nt)
    NC: int          # total coarse steps (Delta t = T / NC)
    slices: int      # N_p
    K: int
    c: tuple = (1.0, 1.0, 1.0)
    nu0: float = 0.1
    omega: float = 100.0
    nu_mode: int = 0             # 0 = stage times, 1 = step start (C1)

    @property
    def nf(self) -> int:
        return self.Nt // self.slices

    @property
    def nc(self) -> int:
        return self.NC // self.slices

    def with_(self, **kw) -> "Config":
        return replace(self, **kw)

    def as_dict(self) -> dict:
        return asdict(self)


CONFIGS = {
    # BASELINE configs[0]: 32^3, 4 slices, K=2, CPU oracle finishes in seconds.
    "cfg1": Config("cfg1", 32, 0.1, 2048, 128, 4, 2),
    # configs[1]: the paper's discretisation, 8 slices, K=1..3.
    "cfg2": Config("cfg2", 128, 0.1, 2 ** 15, 2 ** 11, 8, 3),
    # configs[2]: 256^3 paper-shaped, N_p = W in {1,2,4,8}, K = min(3, N_p).
    "cfg3": Config("cfg3", 256, 0.1, 2 ** 17, 2 ** 13, 8, 3),
    # configs[3]: 512^3, T = 0.1/32 keeps dt, Dt at the 512^3 CFL-safe sizes.
    "cfg4": Config("cfg4", 512, 0.1 / 32, 2 ** 14, 2 ** 10, 8, 3),
    # configs[4]: ratio sweep at 256^3 (Nt in 2^15..2^18 over NC = 2^13).
    "cfg5": Config("cfg5", 256, 0.1, 2 ** 17, 2 ** 13, 8, 3),
    # bench workload: cfg3 shortened 16x in T with the same dt and Dt.
    "cfg3s": Config("cfg3s", 256, 0.1 / 16, 2 ** 13, 2 ** 9, 8, 3),
    # profiling variant: cfg3's dt and Dt, 512x shorter (launch lists under ncu).
    "cfg3p": Config("cfg3p", 256, 0.1 / 512, 2 ** 8, 2 ** 4, 8, 3),
}
