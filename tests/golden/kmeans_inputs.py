"""Seeded inputs of the k-means golden cases (shared by make_golden.py, which
runs the reference on them, and the tests, which regenerate them instead of
storing megabytes of float64 samples)."""

import numpy as np

# (n, d, k, iters, seed, kind)
SPECS = [(3000, 128, 40, 6, 1, "mixture"), (1500, 128, 7, 10, 2, "gauss"),
         (800, 16, 24, 5, 3, "gauss"), (400, 48, 12, 4, 4, "mixture"),
         (300, 128, 20, 5, 5, "dups"), (200, 16, 30, 3, 6, "dups"), (64, 8, 64, 2, 7, "gauss")]


def samples(case: int) -> np.ndarray:
    n, d, k, _, _, kind = SPECS[case]
    rng = np.random.default_rng(1000 + case)
    if kind == "gauss":
        return rng.standard_normal((n, d))
    if kind == "mixture":
        C = rng.standard_normal((max(4, k // 2), d))
        return C[rng.integers(0, C.shape[0], size=n)] + 0.05 * rng.standard_normal((n, d))
    base = rng.standard_normal((6, d))  # few distinct points: clusters die and are reseeded
    return base[rng.integers(0, 6, size=n)]


def e2e_docs():
    """(sizes, X, ids, Q) of the filter-enabled build_index -> query case."""
    rng = np.random.default_rng(2000)
    d = 128
    sizes = rng.integers(5, 40, size=150)
    Cm = rng.standard_normal((30, d))
    X = Cm[rng.integers(0, 30, size=int(sizes.sum()))] + 0.1 * rng.standard_normal((int(sizes.sum()), d))
    ids = rng.permutation(10_000)[:len(sizes)]
    Q = Cm[rng.integers(0, 30, size=(3, 20))] + 0.1 * rng.standard_normal((3, 20, d))
    return sizes, X, ids, Q
