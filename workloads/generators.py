"""Seeded input generators.

Values are drawn with NumPy's PCG64 `default_rng(seed).uniform(-1, 1, N)` in
element-major order (e = ex + nx*(ey + ny*ez); node i + n*(j + n*k)).  The
zero-mean projection is the Euclidean one, b <- b - mean(b) (BASELINE.json
configs: "projected to zero mean").  Both the oracle and the CUDA path consume
the same arrays; neither implementation's arithmetic lives here.
"""
import numpy as np


def uniform_vector(n, seed):
    return np.random.default_rng(seed).uniform(-1.0, 1.0, int(n))


def uniform_zero_mean(n, seed):
    b = uniform_vector(n, seed)
    return b - b.mean()
