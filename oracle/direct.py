"""Direct O(N^2) summation  (oracle; test infrastructure).

u_i = sum_j K(x_i - y_j) rho_j   (Eq. 1.1; Laplace Eq. 3.1,
PAPER.md:465-467).  Coincident source/target pairs (distance exactly 0) are
omitted, as the paper does for the self-interaction (PAPER.md:524-536,
1192-1195).  Plain fp64 numpy, chunked over targets.
"""
from __future__ import annotations

import numpy as np


def laplace3d(sources, charges, targets=None, chunk: int = 2048) -> np.ndarray:
    """sum_{j: y_j != x_i} rho_j / |x_i - y_j|."""
    y = np.asarray(sources, dtype=np.float64)
    q = np.asarray(charges, dtype=np.float64)
    x = y if targets is None else np.asarray(targets, dtype=np.float64)
    out = np.empty(x.shape[0])
    for a in range(0, x.shape[0], chunk):
        d = x[a:a + chunk, None, :] - y[None, :, :]
        r = np.sqrt(np.einsum("ijk,ijk->ij", d, d))
        with np.errstate(divide="ignore"):
            inv = np.where(r > 0.0, 1.0 / r, 0.0)
        out[a:a + chunk] = inv @ q
    return out


def yukawa3d(sources, charges, lam: float, targets=None, chunk: int = 2048) -> np.ndarray:
    """sum_{j: y_j != x_i} rho_j exp(-lam |x_i - y_j|)/|x_i - y_j|  (Eq. 1.1 with the
    Yukawa kernel of Sec. 4.6)."""
    y = np.asarray(sources, dtype=np.float64)
    q = np.asarray(charges, dtype=np.float64)
    x = y if targets is None else np.asarray(targets, dtype=np.float64)
    out = np.empty(x.shape[0])
    for a in range(0, x.shape[0], chunk):
        d = x[a:a + chunk, None, :] - y[None, :, :]
        r = np.sqrt(np.einsum("ijk,ijk->ij", d, d))
        with np.errstate(divide="ignore", invalid="ignore"):
            k = np.where(r > 0.0, np.exp(-lam * r) / r, 0.0)
        out[a:a + chunk] = k @ q
    return out


def log2d(sources, charges, targets=None, chunk: int = 2048) -> np.ndarray:
    """-sum_{j: y_j != x_i} rho_j log|x_i - y_j|  (Eq. 1.1 with the 2D log kernel of
    BASELINE config 3 / Sec. 4.6)."""
    y = np.asarray(sources, dtype=np.float64)
    q = np.asarray(charges, dtype=np.float64)
    x = y if targets is None else np.asarray(targets, dtype=np.float64)
    out = np.empty(x.shape[0])
    for a in range(0, x.shape[0], chunk):
        d = x[a:a + chunk, None, :] - y[None, :, :]
        r = np.sqrt(np.einsum("ijk,ijk->ij", d, d))
        with np.errstate(divide="ignore"):
            k = np.where(r > 0.0, -np.log(np.where(r > 0.0, r, 1.0)), 0.0)
        out[a:a + chunk] = k @ q
    return out


def rel_l2(a, b) -> float:
    """Relative l2 error ||a - b|| / ||b|| (the north-star accuracy metric)."""
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))
