"""Seeded synthetic inputs shared by the CUDA path, the oracle and the bench.

This module holds NO arithmetic of the method (no nodes, kernels, tree or
weights) -- only the random particle generators and the config table, so that
both sides of every parity test read the same bytes.

Recipe (BASELINE.json configs):
  rng = numpy.random.default_rng(seed)   (PCG64), seed 0 by default
  positions first, then weights, float64, AoS [N, 3]
  uniform: X = rng.uniform(-1, 1, (N, 3)),  W = rng.uniform(-1, 1, (N, 3))
  sphere:  G = rng.standard_normal((N, 3)); X = G / |G|_row;  W = rng.uniform(-1, 1, (N, 3))
  rods:    the paper's Example 2 geometry: s x s helical rods
           (x0 + 0.3 cos 2z, y0 + 0.3 sin 2z, z), z = 9k/M, k = 0..M (M = 150), base
           points on a centred square grid of spacing 16/15 (s = 15 spans [-8, 8]^2,
           constant density as s grows); positions are deterministic, then
           W = rng.uniform(-1, 1, (N, m)) (force and torque components in [-1, 1]).
  organisms: the paper's Example 1: N/2 microorganisms, each a body at
           b = rng.uniform(0, 10, 3) and a flagellum at b + 0.02 t (t = a normalised standard
           normal 3-vector), carrying the unit forces +t and -t ("unit forces in opposite
           directions along the organism length"); bodies first, then directions, drawn per
           organism in one call each; particle 2i = body i, 2i+1 = flagellum i.
The uniform cube stands in for the paper's Example 1 (random organisms in a
cube), which "organisms" reproduces; the sphere surface stands in for the non-uniform,
flat-box geometry of Example 2, which "rods" reproduces.
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
    # BASELINE config 4 at its other degree (n in {4, 8})
    "C4n4": dict(N=1_000_000, geometry="uniform", kernel=1, eps=0.01, n=4, theta=0.7, N0=2000),
    # not a BASELINE config: the paper's own Example 2 parallel run (Table 5):
    # 80^2 rods x 151 points, Stokeslet + rotlet, eps = 0.3, theta = 0.7, n = 7, N0 = 1000
    "X2": dict(N=966_400, geometry="rods", kernel=2, eps=0.3, n=7, theta=0.7, N0=1000),
    # not BASELINE configs: the paper's Example 1 rows of Table 1:
    # organism pairs in a side-10 cube, Stokeslet, eps = 0.02, theta = 0.7, n = 7, N0 = 2000
    "X1": dict(N=640_000, geometry="organisms", kernel=0, eps=0.02, n=7, theta=0.7, N0=2000),
    "X1L": dict(N=5_120_000, geometry="organisms", kernel=0, eps=0.02, n=7, theta=0.7, N0=2000),
}
ORG_L, ORG_ELL = 10.0, 0.02   # cube side and organism length
ROD_M = 150          # segments per rod
ROD_SPACING = 16.0 / 15.0


def rod_positions(side: int, M: int = ROD_M) -> np.ndarray:
    """side^2 helical rods of M + 1 points each, rod-major, float64 [side^2 (M+1), 3]."""
    g = (np.arange(side) - 0.5 * (side - 1)) * ROD_SPACING
    x0, y0 = np.meshgrid(g, g, indexing="ij")
    z = 9.0 * np.arange(M + 1) / M
    X = np.empty((side * side, M + 1, 3))
    X[:, :, 0] = x0.reshape(-1, 1) + 0.3 * np.cos(2.0 * z)[None, :]
    X[:, :, 1] = y0.reshape(-1, 1) + 0.3 * np.sin(2.0 * z)[None, :]
    X[:, :, 2] = z[None, :]
    return X.reshape(-1, 3)


def particles(N: int, geometry: str = "uniform", seed: int = 0, m: int = 3):
    """Return (X[N,3], W[N,m]) float64, C-contiguous, per the recipe above."""
    rng = np.random.default_rng(seed)
    if geometry == "uniform":
        X = rng.uniform(-1.0, 1.0, (N, 3))
    elif geometry == "sphere":
        G = rng.standard_normal((N, 3))
        X = G / np.linalg.norm(G, axis=1, keepdims=True)
    elif geometry == "rods":
        side = int(round(np.sqrt(N / (ROD_M + 1))))
        if side * side * (ROD_M + 1) != N:
            raise ValueError(f"rods: N must be s^2 x {ROD_M + 1}")
        X = rod_positions(side)
    elif geometry == "organisms":
        if N % 2:
            raise ValueError("organisms: N must be even (body + flagellum pairs)")
        B = rng.uniform(0.0, ORG_L, (N // 2, 3))
        G = rng.standard_normal((N // 2, 3))
        T = G / np.linalg.norm(G, axis=1, keepdims=True)
        X = np.empty((N, 3))
        X[0::2] = B
        X[1::2] = B + ORG_ELL * T
        if m != 3:
            raise ValueError("organisms: Stokeslet forces (m = 3)")
        W = np.empty((N, 3))
        W[0::2] = T
        W[1::2] = -T
        return np.ascontiguousarray(X), np.ascontiguousarray(W)
    elif geometry == "slab":
        # thin slab (extents 2 x 2 x 0.25): exercises 4-way splits
        X = rng.uniform(-1.0, 1.0, (N, 3)) * np.array([1.0, 1.0, 0.125])
    else:
        raise ValueError(f"unknown geometry {geometry!r}")
    W = rng.uniform(-1.0, 1.0, (N, m))
    return np.ascontiguousarray(X), np.ascontiguousarray(W)


def config_particles(name: str, seed: int = 0):
    c = CONFIGS[name]
    return particles(c["N"], c["geometry"], seed, m=6 if c["kernel"] == 2 else 3)


def sample_targets(N: int, S: int, seed: int = 1) -> np.ndarray:
    """Uniform random sample of S distinct target indices (sorted), int64."""
    if S >= N:
        return np.arange(N, dtype=np.int64)
    rng = np.random.default_rng(seed)
    return np.sort(rng.choice(N, size=S, replace=False)).astype(np.int64)
