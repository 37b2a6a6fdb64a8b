"""Seeded synthetic workloads with the shapes of BASELINE.json's five configs.

BASELINE.json names no public dataset; these
generators stand in for the paper's MS MARCO / LoTTE ColBERT embeddings with
the configs' shapes, sizes and value distributions:

* cfg0 -- N=1,000 sets, m_i ~ U{20..100}, d=128 fp32 N(0,I) unit rows; 16
  query sets of 32 (pick a set, sample 32 rows with replacement, add
  N(0, 0.1^2), renormalise).  L=32, C=6, top-10.  Generated with numpy on the
  host (it is the parity config; tests regenerate it from the seed).
* cfg1 -- N=100,000 sets, m_i = clip(round(N(70, 20)), 8, 180); fp16 unit rows
  normalise(c + 0.05 N(0,I)) with c drawn per vector from 4,096 normalised
  Gaussian centroids; 1,000 query sets built as in cfg0.  L=64, C=7, top-100.
* cfg2 -- 10,000,000 bf16 vectors from the cfg1 mixture, cfg1 set sizes.
  L=64, C=7 (index-build throughput).
* cfg3 -- N=1,000,000 sets (cfg1 sizes) from 65,536 centroids; prefilter
  probe 4, k_filter 4,096; L=32, C=7; top-100.
* cfg4 -- N=8,000,000 sets, m_i = clip(round(N(70, 25)), 8, 180), codes only
  (L=32, C=8), 262,144 centroids; 1,024 query sets; top-1,000.

The large configs are generated on the GPU with torch's seeded generator
(input synthesis only -- not part of the measured path).  Per-vector centroid
draws are used (SURVEY.md 8(d) leaves per-vector vs per-set open).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass(frozen=True)
class WorkloadSpec:
    name: str
    n_sets: int
    L: int
    C: int
    top_k: int
    n_qsets: int
    m_q: int = 32
    d: int = 128
    size_mean: float = 70.0
    size_std: float = 20.0
    n_centroids: int = 4096
    dtype: str = "fp16"


CONFIGS = {
    0: WorkloadSpec("cfg0", 1000, 32, 6, 10, 16, dtype="fp32"),
    1: WorkloadSpec("cfg1", 100_000, 64, 7, 100, 1000),
    2: WorkloadSpec("cfg2", 0, 64, 7, 0, 0, dtype="bf16"),
    3: WorkloadSpec("cfg3", 1_000_000, 32, 7, 100, 256, n_centroids=65536),
    4: WorkloadSpec("cfg4", 8_000_000, 32, 8, 1000, 1024, size_std=25.0,
                    n_centroids=262144, dtype="codes"),
}


def _normalise(X):
    return X / np.linalg.norm(X, axis=1, keepdims=True)


def cfg0_data(seed: int = 0):
    """Returns (sizes (N,), X (sum m, 128) fp32, Q (16, 32, 128) fp32)."""
    rng = np.random.default_rng(seed)
    N, d, n_q, m_q = 1000, 128, 16, 32
    sizes = rng.integers(20, 101, size=N).astype(np.int64)
    X = _normalise(rng.standard_normal((int(sizes.sum()), d))).astype(np.float32)
    off = np.concatenate([[0], np.cumsum(sizes)])
    Q = np.empty((n_q, m_q, d), dtype=np.float32)
    for i in range(n_q):
        s = int(rng.integers(0, N))
        rows = rng.integers(0, sizes[s], size=m_q)
        base = X[off[s] + rows].astype(np.float64)
        Q[i] = _normalise(base + 0.1 * rng.standard_normal((m_q, d))).astype(np.float32)
    return sizes, X, Q


def set_sizes(n_sets: int, mean: float, std: float, seed: int) -> np.ndarray:
    """m_i = clip(round(N(mean, std)), 8, 180) (configs 1-4)."""
    rng = np.random.default_rng(seed)
    return np.clip(np.rint(rng.normal(mean, std, size=n_sets)), 8, 180).astype(np.int64)


def offsets(sizes) -> np.ndarray:
    return np.concatenate([[0], np.cumsum(np.asarray(sizes, dtype=np.int64))]).astype(np.int64)


# ---------------------------------------------------------------- GPU synthesis

def gpu_mixture(n_vec: int, n_centroids: int, d: int, noise: float, seed: int,
                dtype, device="cuda", chunk: int = 1 << 22):
    """normalise(c + noise*N(0,I)) rows, c uniform over normalised N(0,I) centroids.

    Returns (X (n_vec, d) tensor of ``dtype`` on device, centroids fp32 tensor).
    """
    import torch

    g = torch.Generator(device=device)
    g.manual_seed(seed)
    cents = torch.randn(n_centroids, d, generator=g, device=device)
    cents = cents / cents.norm(dim=1, keepdim=True)
    X = torch.empty(n_vec, d, dtype=dtype, device=device)
    for lo in range(0, n_vec, chunk):
        hi = min(n_vec, lo + chunk)
        idx = torch.randint(0, n_centroids, (hi - lo,), generator=g, device=device)
        v = cents[idx] + noise * torch.randn(hi - lo, d, generator=g, device=device)
        X[lo:hi] = (v / v.norm(dim=1, keepdim=True)).to(dtype)
    return X, cents


def gpu_queries(X, off: np.ndarray, n_qsets: int, m_q: int, seed: int, noise: float = 0.1):
    """Query sets: pick a set, 32 rows with replacement, + N(0, noise^2), renormalise."""
    import torch

    rng = np.random.default_rng(seed)
    n_sets = len(off) - 1
    sets = rng.integers(0, n_sets, size=n_qsets)
    sizes = off[sets + 1] - off[sets]
    rows = (off[sets][:, None] + (rng.random((n_qsets, m_q)) * sizes[:, None]).astype(np.int64))
    idx = torch.from_numpy(rows.reshape(-1)).to(X.device)
    g = torch.Generator(device=X.device)
    g.manual_seed(seed + 1)
    base = X[idx].float()
    v = base + noise * torch.randn(base.shape, generator=g, device=X.device)
    v = (v / v.norm(dim=1, keepdim=True)).to(X.dtype)
    return v.reshape(n_qsets, m_q, X.shape[1])


def gpu_codes_only(sizes, config, n_centroids: int, n_qsets: int, m_q: int, seed: int,
                   device="cuda", chunk: int = 1 << 23, noise: float = 0.05):
    """cfg4 synthesis: hash mixture vectors chunk by chunk straight into plane
    records (no raw vectors kept), collecting the query-source rows on the way.

    Returns (records (sum m_i, R) int32, query vectors (n_qsets, m_q, d) fp16).
    Hashing uses the float32 SIMT kernel (input synthesis; parity is defined
    on the resulting codes, which the oracle reads back from the records).
    """
    import torch

    from . import _lib, engine
    from .lsh import sample_srp_family

    fam = sample_srp_family(config.d, config.C, config.L, config.seed)
    planes = fam.device_planes(_lib.HASH_F32, device)
    off = offsets(sizes)
    n_vec = int(off[-1])
    R = engine.record_words(config.L, config.C)
    recs = torch.empty((n_vec, R), dtype=torch.int32, device=device)
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    cents = torch.randn(n_centroids, config.d, generator=g, device=device)
    cents = cents / cents.norm(dim=1, keepdim=True)
    rng = np.random.default_rng(seed)
    src = rng.integers(0, len(sizes), size=n_qsets)
    rows = (off[src][:, None] + (rng.random((n_qsets, m_q)) * sizes[src][:, None]).astype(np.int64))
    flat = rows.reshape(-1)
    order = np.argsort(flat, kind="stable")
    sorted_rows = flat[order]
    gathered = torch.empty((flat.size, config.d), dtype=torch.float32, device=device)
    for lo in range(0, n_vec, chunk):
        hi = min(n_vec, lo + chunk)
        idx = torch.randint(0, n_centroids, (hi - lo,), generator=g, device=device)
        v = cents[idx] + noise * torch.randn(hi - lo, config.d, generator=g, device=device)
        X = (v / v.norm(dim=1, keepdim=True)).to(torch.float16)
        _, r, _ = engine.hash_vectors(X, planes, _lib.HASH_F32, config.L, config.C,
                                      want_codes=False, check_zero=False)
        recs[lo:hi] = r
        a, b = np.searchsorted(sorted_rows, [lo, hi])
        if b > a:
            sel = torch.from_numpy(sorted_rows[a:b] - lo).to(device)
            dst = torch.from_numpy(order[a:b]).to(device)
            gathered[dst] = X[sel].float()
        del X, v, idx
    q = gathered + 0.1 * torch.randn(gathered.shape, generator=g, device=device)
    q = (q / q.norm(dim=1, keepdim=True)).to(torch.float16)
    return recs, q.reshape(n_qsets, m_q, config.d)


def records_to_codes(recs: np.ndarray, L: int, C: int) -> np.ndarray:
    """Host inverse of the plane-record layout (test infrastructure / parity sampling)."""
    W = (L + 31) // 32
    recs = np.asarray(recs).view(np.uint32)
    codes = np.zeros((recs.shape[0], L), dtype=np.int64)
    for t in range(L):
        w, bit = divmod(t, 32)
        for b in range(C):
            codes[:, t] |= ((recs[:, b * W + w] >> np.uint32(bit)) & np.uint32(1)).astype(np.int64) << b
    return codes
