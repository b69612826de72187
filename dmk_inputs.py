"""Seeded synthetic workloads shared by tests, smoke() and bench.py.

Holds none of the method's arithmetic: only point clouds and charges with the
shapes and distributions of BASELINE.json's configs.  Both the oracle and the
CUDA path consume these arrays; neither is imported here.

  uniform     N iid points in [0,1]^3, charges U[-1,1]           (configs 0, 1, 4)
  clusters    90% from 10 isotropic Gaussian clusters (sigma in [1e-3, 1e-2],
              centres uniform in the cube, clipped to [0,1]^3) + 10% uniform;
              standard-normal charges                             (config 2)
  sphere      uniform on the sphere of radius 0.45 centred at (0.5,0.5,0.5)
              (the paper's Sec. 5.1 surface distribution)
  circle2d    2D: noisy circle, radius 0.4 + N(0, 1e-3), zero-mean U[-1,1] charges
                                                                   (config 3)
"""
from __future__ import annotations

import numpy as np


def uniform(n: int, seed: int = 0, dim: int = 3):
    rng = np.random.default_rng(seed)
    x = rng.uniform(0.0, 1.0, size=(n, dim))
    q = rng.uniform(-1.0, 1.0, size=n)
    return x, q


def clusters(n: int, seed: int = 0, nclusters: int = 10):
    rng = np.random.default_rng(seed)
    nc = int(round(0.9 * n))
    centres = rng.uniform(0.0, 1.0, size=(nclusters, 3))
    sig = rng.uniform(1e-3, 1e-2, size=nclusters)
    lab = rng.integers(0, nclusters, size=nc)
    xc = centres[lab] + sig[lab, None] * rng.standard_normal((nc, 3))
    xu = rng.uniform(0.0, 1.0, size=(n - nc, 3))
    x = np.clip(np.concatenate([xc, xu]), 0.0, 1.0)
    x = x[rng.permutation(n)]
    q = rng.standard_normal(n)
    return x, q


def sphere(n: int, seed: int = 0, radius: float = 0.45):
    rng = np.random.default_rng(seed)
    v = rng.standard_normal((n, 3))
    v /= np.linalg.norm(v, axis=1, keepdims=True)
    x = 0.5 + radius * v
    q = rng.uniform(-1.0, 1.0, size=n)
    return x, q


def circle2d(n: int, seed: int = 0, radius: float = 0.4, jitter: float = 1e-3):
    """BASELINE config 3: N points on a noisy circle, radius 0.4 + N(0, jitter) about
    (0.5, 0.5) in [0,1]^2; charges U[-1,1] shifted to zero mean."""
    rng = np.random.default_rng(seed)
    th = rng.uniform(0.0, 2.0 * np.pi, n)
    r = radius + jitter * rng.standard_normal(n)
    x = 0.5 + np.stack([r * np.cos(th), r * np.sin(th)], axis=1)
    q = rng.uniform(-1.0, 1.0, size=n)
    q -= q.mean()
    return x, q


WORKLOADS = {"uniform": uniform, "clusters": clusters, "sphere": sphere, "circle2d": circle2d}


def make(kind: str, n: int, seed: int = 0):
    return WORKLOADS[kind](n, seed=seed)
