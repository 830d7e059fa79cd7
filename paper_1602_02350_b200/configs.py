"""The five BASELINE.json configurations and their synthetic data.

X = G diag(sigma) V^T with G iid N(0,1) (n x d), V Haar (QR of an iid N(0,1)
d x d matrix, V = Q diag(sign diag R)), optional |Student-t(3)| row scaling,
w* ~ N(0, I/d), y = X w* + tau N(0,1).  fp32 configs round X and y to fp32 and
the oracle consumes exactly those values promoted to fp64.

The generator is ``skridge.DataMatrix.generate`` (device, Philox4x32-10
streams 1..5, skr_data_generate).  The CPU side (tests, goldens, bench.py's
reference arm) regenerates the same instance with ``oracle.synth_instance``,
a host restatement of the device generator: identical integer streams, fp64
values within a few ulps, fp32 values identical except for rare rounding ties.
Row i of the instance does not depend on n, so a row-subsampled instance is
the first n rows of the full one.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass(frozen=True)
class Config:
    name: str
    dtype: str          # "f64" | "f32"
    n: int
    d: int
    seed: int
    spectrum: int       # 0: 1/j, 1: r^j, 2: j^-p, 3: 1/j (j<=50), 0.02/j beyond
    spectrum_param: float
    t_scale: bool
    tau: float
    lam: float
    k: int
    q: int
    epochs: int

    def sigma(self, d: int | None = None) -> np.ndarray:
        j = np.arange(1, (d or self.d) + 1, dtype=np.float64)
        if self.spectrum == 0:
            return 1.0 / j
        if self.spectrum == 1:
            return self.spectrum_param ** j
        if self.spectrum == 2:
            return j ** (-self.spectrum_param)
        return np.where(j <= 50, 1.0 / j, 0.02 / j)

    def scaled(self, n: int) -> "Config":
        """Same config at n rows (row-subsampled parity instances)."""
        return Config(**{**self.__dict__, "n": n})


CONFIGS = {
    "c1": Config("c1", "f64", 8192, 256, 0, 0, 0.0, False, 0.1, 1e-3, 16, 3, 20),
    "c2": Config("c2", "f64", 65536, 1024, 1, 1, 0.97, False, 0.05, 1e-5, 64, 4, 30),
    "c3": Config("c3", "f32", 1 << 20, 2048, 2, 2, 1.5, False, 0.1, 1e-6, 128, 3, 20),
    "c4": Config("c4", "f32", 1 << 22, 4096, 3, 3, 0.0, True, 0.1, 1e-6, 256, 3, 60),
    "c5": Config("c5", "f32", 1 << 24, 1024, 4, 1, 0.99, False, 0.2, 1e-6, 64, 2, 20),
}


def step_size(max_row_sq: float) -> float:
    """BASELINE c1 rule: eta = 1 / (4 max_i ||x~_i||^2) over the data rows of X~."""
    return 1.0 / (4.0 * max_row_sq)


def eta_for(cfg: Config, max_row_sq: float, beta_hat: float) -> float:
    """Step size per config.  c1 (and c2, where BASELINE is silent) use the c1 rule.
    For c3-c5 (eta unspecified) the c1 rule diverges — with lambda = 1e-6 the
    regulariser components lambda (n+d) ||b_j||^2 dominate the smoothness
    (beta_hat ~ 1.4e3 vs max data row ~ 1.7e2 at c3; the reference itself blows up
    from 0.0126 to 104 in 4 epochs) — so the rule is capped by the mean smoothness:
    eta = 1 / (4 max(max_row, beta_hat)) (the scale of the reference's own grid
    2^j / beta_hat, bench.cpp:96-100)."""
    if cfg.name in ("c1", "c2"):
        return step_size(max_row_sq)
    return 1.0 / (4.0 * max(max_row_sq, beta_hat))
