"""Synthetic datasets with the shapes of BASELINE.json's configs.

Same distribution families as the reference generator (proj/src/synthetic.cpp:
uniform / ``clusters:c:spread`` round-robin Gaussian clusters / ``mixture`` 70%
clusters + 30% uniform background) plus the i.i.d. Exp(1) family the survey adds
for config C4. Drawn with numpy's PCG64 (not libstdc++), so they are fixtures
of the same SHAPE, not byte-copies of the reference generator's output.
"""
from __future__ import annotations

import numpy as np


def generate(spec: str, size: int, dims: int, seed: int = 1) -> np.ndarray:
    parts = spec.split(":")
    kind = parts[0]
    clusters = int(parts[1]) if len(parts) > 1 and parts[1] else 3
    spread = float(parts[2]) if len(parts) > 2 and parts[2] else 0.05
    rng = np.random.default_rng(seed)
    if kind == "uniform":
        return rng.random((size, dims))
    if kind == "exponential":
        return rng.exponential(1.0, (size, dims))
    if kind in ("clusters", "mixture"):
        centers = rng.random((clusters, dims))
        dense = size if kind == "clusters" else int(size * 0.7)
        X = np.empty((size, dims), np.float64)
        lab = np.arange(dense) % clusters
        X[:dense] = centers[lab] + spread * rng.standard_normal((dense, dims))
        if dense < size:
            X[dense:] = rng.random((size - dense, dims))
        return X
    raise ValueError(f"unknown synthetic kind '{kind}'")


# BASELINE.json configs; k, spec, |D|, n
CONFIGS = {
    "C1": dict(spec="uniform", size=100_000, dims=2, k=5),
    "C2": dict(spec="clusters:16:0.05", size=5_000_000, dims=18, k=32),
    "C3": dict(spec="mixture:8:0.05", size=500_000, dims=90, k=16),
    "C4": dict(spec="exponential", size=20_000_000, dims=6, k=64),
    "C5": dict(spec="uniform", size=100_000_000, dims=4, k=32),
    "NS": dict(spec="clusters:16:0.05", size=10_000_000, dims=18, k=32),
}
