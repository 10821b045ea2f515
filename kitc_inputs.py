"""Seeded synthetic inputs shared by the CUDA path, the oracle and the bench.

This module holds NO arithmetic of the method (no nodes, kernels, tree or
weights) -- only the random particle generators and the config table, so that
both sides of every parity test read the same bytes.

Recipe (BASELINE.json configs):
  rng = numpy.random.default_rng(seed)   (PCG64), seed 0 by default
  positions first, then weights, float64, AoS [N, 3]
  uniform: X = rng.uniform(-1, 1, (N, 3)),  W = rng.uniform(-1, 1, (N, 3))
  sphere:  G = rng.standard_normal((N, 3)); X = G / |G|_row;  W = rng.uniform(-1, 1, (N, 3))
The uniform cube stands in for the paper's Example 1 (random organisms in a
cube); the sphere surface stands in for the non-uniform,
flat-box geometry of Example 2.
"""
from __future__ import annotations

import numpy as np

# BASELINE.json configs (C1..C5).  kernel: 0 = Stokeslet, 1 = rotlet.
CONFIGS = {
    "C1": dict(N=1_000, geometry="uniform", kernel=0, eps=0.01, n=4, theta=0.7, N0=100),
    "C2": dict(N=100_000, geometry="uniform", kernel=0, eps=0.01, n=8, theta=0.7, N0=500),
    "C3": dict(N=1_000_000, geometry="uniform", kernel=0, eps=0.01, n=8, theta=0.7, N0=2000),
    "C4": dict(N=1_000_000, geometry="uniform", kernel=1, eps=0.01, n=8, theta=0.7, N0=2000),
    "C5": dict(N=10_000_000, geometry="sphere", kernel=0, eps=0.005, n=8, theta=0.7, N0=2000),
}


def particles(N: int, geometry: str = "uniform", seed: int = 0, m: int = 3):
    """Return (X[N,3], W[N,m]) float64, C-contiguous, per the recipe above."""
    rng = np.random.default_rng(seed)
    if geometry == "uniform":
        X = rng.uniform(-1.0, 1.0, (N, 3))
    elif geometry == "sphere":
        G = rng.standard_normal((N, 3))
        X = G / np.linalg.norm(G, axis=1, keepdims=True)
    elif geometry == "slab":
        # thin slab (extents 2 x 2 x 0.25): exercises 4-way splits
        X = rng.uniform(-1.0, 1.0, (N, 3)) * np.array([1.0, 1.0, 0.125])
    else:
        raise ValueError(f"unknown geometry {geometry!r}")
    W = rng.uniform(-1.0, 1.0, (N, m))
    return np.ascontiguousarray(X), np.ascontiguousarray(W)


def config_particles(name: str, seed: int = 0):
    c = CONFIGS[name]
    return particles(c["N"], c["geometry"], seed)


def sample_targets(N: int, S: int, seed: int = 1) -> np.ndarray:
    """Uniform random sample of S distinct target indices (sorted), int64."""
    if S >= N:
        return np.arange(N, dtype=np.int64)
    rng = np.random.default_rng(seed)
    return np.sort(rng.choice(N, size=S, replace=False)).astype(np.int64)
