"""Seeded inputs of the .dsri golden cases (make_golden.py runs the reference's
build_index + save_index on them; the tests rebuild the same indexes)."""

import numpy as np

# name -> (d, C, L, seed, inner_kind, phi, filter kwargs or None, sizes spec)
CASES = {
    "small_filter": (8, 3, 16, 2, "max", None, dict(centroids=4, probe=2, k_filter=8), "small"),
    "small_nofilter": (8, 3, 16, 2, "max", None, None, "small"),
    "wide": (16, 4, 8, 5, "max", None, None, "wide"),
    "avgphi_filter": (16, 6, 32, 7, "avg-phi", "debiased-sigmoid", dict(iters=3, probe=3, k_filter=20),
                      "medium"),
    "many_docs": (8, 2, 8, 9, "max", None, dict(centroids=3, iters=2, probe=1, k_filter=300), "many"),
}


def docs(name: str):
    d = CASES[name][0]
    spec = CASES[name][7]
    rng = np.random.default_rng(sum(map(ord, name)))
    if spec == "small":
        sizes = rng.integers(1, 9, size=12)
    elif spec == "wide":
        sizes = np.array([255, 256, 257, 300, 1, 2, 40])
    elif spec == "medium":
        sizes = rng.integers(1, 60, size=40)
    else:
        sizes = rng.integers(1, 4, size=400)
    ids = rng.permutation(100_000)[:len(sizes)]
    out = []
    for i, m in enumerate(sizes):
        out.append((int(ids[i]), rng.standard_normal((int(m), d))))
    return out


def queries(name: str):
    d = CASES[name][0]
    rng = np.random.default_rng(7 + sum(map(ord, name)))
    return [rng.standard_normal((int(rng.integers(1, 6)), d)) for _ in range(4)]
