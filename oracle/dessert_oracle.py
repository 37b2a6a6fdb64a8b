"""CPU oracle for the DESSERT scoring hot path -- TEST INFRASTRUCTURE ONLY.

This module restates, in numpy, the reference algorithm of the DESSERT
vector-set search path (reference: /root/reference/pkg/src/dessert/, cited
below as ``lsh.py``, ``sketch.py``, ``index.py``, ``prefilter.py``).  It is
the *checker* for the CUDA path in ``paper_2210_15748_b200``: only
``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import it.  The product path never calls it
(there is no CPU fallback; the product fails loudly without its CUDA
library).

Pinning: every function here is checked against golden vectors produced by
running the *real* reference package in the build container
(``tests/golden/make_golden.py`` -> ``tests/golden/*.npz``) and against the
reference's own known-answer tests (restated in ``tests/test_oracle.py``).

Two scoring restatements live here:

* ``score_port`` -- a line-by-line port of the reference's TinyTable path
  (``build_tiny_table`` sketch.py:51-80, ``collision_keys`` sketch.py:156-178,
  ``_score_one`` index.py:183-216).  This is "the reference's own CPU
  implementation" used as the CPU baseline (kind "port").
* ``score_dense`` -- the closed form the GPU implements: dense code compare
  -> per-query max count -> float64 LUT -> numpy pairwise mean.  Proven equal
  to ``score_port`` (tests) and to the reference (golden vectors).
"""

from __future__ import annotations

import heapq
import math
from dataclasses import dataclass

import numpy as np

MAX_CONCAT_BITS = 24  # lsh.py:17
MAX_SET_SIZE = 65535  # sketch.py:23


# --------------------------------------------------------------------------
# hashing (lsh.py)
# --------------------------------------------------------------------------

def sample_planes(d: int, C: int, L: int, seed: int) -> np.ndarray:
    """SRP hyperplanes, row t*C + c = plane c of table t.  lsh.py:54-66."""
    if d < 1:
        raise ValueError(f"invalid parameter: d must be >= 1, got {d}")
    if C < 1 or C > MAX_CONCAT_BITS:
        raise ValueError(f"invalid parameter: C must be in [1, {MAX_CONCAT_BITS}], got {C}")
    if L < 1:
        raise ValueError(f"invalid parameter: L must be >= 1, got {L}")
    return np.random.default_rng(seed).standard_normal((L * C, d))


def hash_matrix(planes: np.ndarray, L: int, C: int, X) -> np.ndarray:
    """(n, d) -> (n, L) int64 codes; bit c of code t = <plane t*C+c, x> > 0.

    lsh.py:90-106 (float64 GEMM, strict '>' so a zero projection is bit 0,
    bits packed LSB-first by plane index within the table).
    """
    X = np.asarray(X, dtype=np.float64)
    if X.ndim != 2 or X.shape[1] != planes.shape[1]:
        raise ValueError(
            f"dimension mismatch: expected (n, {planes.shape[1]}) matrix, got shape {X.shape}")
    if not np.all(np.any(X, axis=1)):
        raise ValueError("zero vector cannot be hashed (sign of zero projection undefined)")
    bits = (X @ planes.T) > 0.0
    bits = bits.reshape(X.shape[0], L, C)
    weights = np.left_shift(1, np.arange(C, dtype=np.int64))
    return bits @ weights


def projections(planes: np.ndarray, X) -> np.ndarray:
    """float64 projections X @ planes.T (used to classify hash-bit flips)."""
    return np.asarray(X, dtype=np.float64) @ planes.T


def sim_lut(C: int, L: int) -> np.ndarray:
    """count -> similarity table (k/L)^(1/C), table[0] = 0.  lsh.py:130-139."""
    if C < 1:
        raise ValueError(f"invalid parameter: C must be >= 1, got {C}")
    if L < 1:
        raise ValueError(f"invalid parameter: L must be >= 1, got {L}")
    k = np.arange(L + 1, dtype=np.float64)
    table = (k / L) ** (1.0 / C)
    table[0] = 0.0
    return table


# --------------------------------------------------------------------------
# TinyTable (sketch.py) -- the structure the reference scores against
# --------------------------------------------------------------------------

def _offset_dtype(m: int):  # sketch.py:26-28
    return np.dtype(np.uint8) if m <= 255 else np.dtype(np.uint16)


def _id_dtype(m: int):  # sketch.py:31-33
    return np.dtype(np.uint8) if m <= 256 else np.dtype(np.uint16)


@dataclass(frozen=True)
class TinyTable:
    """sketch.py:36-48: offsets (L, r+1), ids (L, m)."""

    m: int
    L: int
    r: int
    offsets: np.ndarray
    ids: np.ndarray


def build_tiny_table(codes, L: int, r: int) -> TinyTable:
    """Per-table counting sort of one set's codes.  sketch.py:51-80."""
    codes = np.asarray(codes)
    if codes.ndim != 2:
        raise ValueError(f"expected (m, L) code matrix, got shape {codes.shape}")
    m = codes.shape[0]
    if m == 0:
        raise ValueError("empty set: cannot sketch zero vectors")
    if m > MAX_SET_SIZE:
        raise ValueError(f"set too large: m must be <= {MAX_SET_SIZE}, got {m}")
    if codes.shape[1] != L:
        raise ValueError(f"expected {L} codes per vector, got {codes.shape[1]}")
    if r < 1:
        raise ValueError(f"invalid parameter: r must be >= 1, got {r}")
    if codes.min() < 0 or codes.max() >= r:
        raise ValueError(f"code out of range: codes must lie in [0, {r})")
    offsets = np.zeros((L, r + 1), dtype=_offset_dtype(m))
    ids = np.zeros((L, m), dtype=_id_dtype(m))
    for t in range(L):
        col = codes[:, t]
        offsets[t, 1:] = np.cumsum(np.bincount(col, minlength=r))
        ids[t] = np.argsort(col, kind="stable")
    return TinyTable(m=m, L=L, r=r, offsets=offsets, ids=ids)


def accumulate_collisions_batch(table: TinyTable, query_codes) -> np.ndarray:
    """(m_q, L) codes -> (m_q, m) collision counts.  sketch.py:118-153 (dense form)."""
    q = np.asarray(query_codes)
    m_q = q.shape[0]
    counts = np.zeros((m_q, table.m), dtype=np.int32)
    for t in range(table.L):
        lo = table.offsets[t, q[:, t]].astype(np.intp)
        hi = table.offsets[t, q[:, t] + 1].astype(np.intp)
        for row in range(m_q):
            counts[row, table.ids[t, lo[row]:hi[row]]] += 1
    return counts


def collision_keys(table: TinyTable, query_codes) -> np.ndarray:
    """One int64 key q*m + j per collision event.  sketch.py:156-178."""
    codes = np.asarray(query_codes)
    m_q = codes.shape[0]
    t_idx = np.arange(table.L)
    starts = table.offsets[t_idx, codes].astype(np.intp)
    lens = (table.offsets[t_idx, codes + 1] - starts).reshape(-1).astype(np.intp)
    total = int(lens.sum())
    if total == 0:
        return np.empty(0, dtype=np.int64)
    flat_starts = (starts + t_idx * table.m).reshape(-1)
    ends_cum = np.cumsum(lens)
    pos = np.arange(total, dtype=np.intp) - np.repeat(ends_cum - lens, lens)
    members = table.ids.reshape(-1)[pos + np.repeat(flat_starts, lens)]
    cell_keys = (np.arange(m_q * table.L, dtype=np.int64) // table.L) * table.m
    return np.repeat(cell_keys, lens) + members


def score_port(table: TinyTable, query_codes, lut: np.ndarray, kind: str = "max",
               weights=None) -> float:
    """index.py:183-216 (_score_one), ported.

    ``lut`` is the aggregand table (_sim_table_for, index.py:170-180): the
    lookup table for kind "max", phi(lookup table) for "avg-phi".  weights
    None means all ones (index.py:219-221).
    """
    keys = collision_keys(table, query_codes)
    m_q = np.asarray(query_codes).shape[0]
    w = np.ones(m_q) if weights is None else np.asarray(weights, dtype=np.float64)
    per_query = np.zeros(m_q)
    if keys.size:
        keys.sort()
        run_starts = np.flatnonzero(np.diff(keys)) + 1
        counts = np.diff(run_starts, prepend=0, append=keys.size)
        rows = keys[np.concatenate(([0], run_starts))] // table.m
        row_bounds = np.searchsorted(rows, np.arange(m_q + 1))
        occupied = row_bounds[:-1] < row_bounds[1:]
        seg_starts = row_bounds[:-1][occupied]
        if kind == "max":
            per_query[occupied] = lut[np.maximum.reduceat(counts, seg_starts)]
        else:
            per_query[occupied] = np.add.reduceat(lut[counts], seg_starts) / table.m
    return float(np.mean(w * per_query))


# --------------------------------------------------------------------------
# dense restatement (what the GPU computes)
# --------------------------------------------------------------------------

def max_counts(query_codes, set_codes) -> np.ndarray:
    """c_q = max_j sum_t [q_t == x_jt]  (m_q,) int -- the integer parity target."""
    q = np.asarray(query_codes)
    x = np.asarray(set_codes)
    eq = (q[:, None, :] == x[None, :, :]).sum(axis=2)
    return eq.max(axis=1)


def pairwise_sum(a) -> float:
    """numpy's float64 pairwise summation (8 accumulators, block 128), restated.

    Mirrors numpy/_core/src/umath/loops_utils.h.src pairwise_sum_DOUBLE, which
    ``np.mean`` (index.py:216) runs over the contiguous per-query array after
    starting from the additive identity 0.0.  tests/test_oracle.py pins it
    against np.mean for n = 1..20000.
    """
    a = [float(v) for v in a]

    def rec(lo: int, n: int) -> float:
        if n < 8:
            r = 0.0
            for i in range(n):
                r += a[lo + i]
            return r
        if n <= 128:
            r = a[lo:lo + 8]
            i = 8
            while i < n - (n % 8):
                for j in range(8):
                    r[j] += a[lo + i + j]
                i += 8
            res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]))
            while i < n:
                res += a[lo + i]
                i += 1
            return res
        n2 = n // 2
        n2 -= n2 % 8
        return rec(lo, n2) + rec(lo + n2, n - n2)

    return 0.0 + rec(0, len(a))


def score_dense(query_codes, set_codes, lut: np.ndarray) -> float:
    """sum_q LUT[c_q] (numpy pairwise order) / m_q."""
    c = max_counts(query_codes, set_codes)
    return float(np.mean(lut[c]))


def score_sets_dense(query_codes, codes, set_off, lut, sets=None) -> np.ndarray:
    """Dense scores of one query set against sets (default: all)."""
    n = len(set_off) - 1
    sets = range(n) if sets is None else sets
    return np.array([score_dense(query_codes, codes[set_off[i]:set_off[i + 1]], lut)
                     for i in sets], dtype=np.float64)


def reduceat_sum(vals) -> float:
    """One np.add.reduceat segment: first element + pairwise(rest).

    numpy's reduceat seeds the output with the segment's first element and
    runs the add reduce loop (pairwise_sum_DOUBLE) over the remainder;
    tests/test_oracle.py pins this against np.add.reduceat.
    """
    v = [float(x) for x in vals]
    if not v:
        raise ValueError("empty segment")
    return v[0] + pairwise_sum(v[1:])


def score_dense_agg(query_codes, set_codes, table: np.ndarray, kind: str = "max",
                    weights=None) -> float:
    """Dense restatement of _score_one for any Scorer (what K3g computes).

    per_query[q] = table[max_j c_qj]                                 (max)
                 = reduceat_sum(table[c_qj] : c_qj > 0, j asc) / m   (avg-phi)
    score = pairwise_sum(w_q * per_query[q]) / m_q
    """
    q = np.asarray(query_codes)
    x = np.asarray(set_codes)
    m_q, m = q.shape[0], x.shape[0]
    w = np.ones(m_q) if weights is None else np.asarray(weights, dtype=np.float64)
    eq = (q[:, None, :] == x[None, :, :]).sum(axis=2) if m else np.zeros((m_q, 0), np.int64)
    pq = np.zeros(m_q)
    for i in range(m_q):
        if kind == "max":
            pq[i] = table[eq[i].max()] if m else 0.0
        else:
            nz = eq[i][eq[i] > 0]
            pq[i] = reduceat_sum(table[nz]) / m if nz.size else 0.0
    return pairwise_sum(w * pq) / m_q


def score_sets_dense_agg(query_codes, codes, set_off, table, kind="max", weights=None,
                         sets=None) -> np.ndarray:
    n = len(set_off) - 1
    sets = range(n) if sets is None else sets
    return np.array([score_dense_agg(query_codes, codes[set_off[i]:set_off[i + 1]], table, kind,
                                     weights) for i in sets], dtype=np.float64)


# --------------------------------------------------------------------------
# ranking (index.py:314-319)
# --------------------------------------------------------------------------

def rank_topk(scores, doc_ids, top_k: int):
    """heapq.nsmallest by (-score, doc_id) -> [(doc_id, score)].  index.py:314-319."""
    ranked = ((float(s), int(d)) for s, d in zip(scores, doc_ids))
    best = heapq.nsmallest(top_k, ranked, key=lambda e: (-e[0], e[1]))
    return [(doc_id, score) for score, doc_id in best]


# --------------------------------------------------------------------------
# centroid prefilter (prefilter.py)
# --------------------------------------------------------------------------

def _unit_rows(X, name: str) -> np.ndarray:  # prefilter.py:37-44
    X = np.asarray(X, dtype=np.float64)
    if X.ndim != 2 or X.shape[0] == 0:
        raise ValueError(f"{name} must be a non-empty (n, d) matrix, got shape {X.shape}")
    norms = np.linalg.norm(X, axis=1, keepdims=True)
    if np.any(norms == 0.0):
        raise ValueError(f"zero vector in {name}: cannot assign to a centroid")
    return X / norms


def train_centroids(samples, k: int, iters: int, seed: int) -> np.ndarray:
    """Spherical Lloyd iterations, prefilter.py:47-82, restated step by step.

    Also spells out the operation order K7 reproduces: dot products as
    X @ C.T (BLAS), sums by in-order np.add.at, row norms by np.linalg.norm,
    dead clusters (empty or norm < 1e-12) reseeded in ascending id from the
    stable argsort of each point's best similarity.
    """
    X = _unit_rows(samples, "samples")
    n = X.shape[0]
    if k < 1:
        raise ValueError(f"invalid parameter: k must be >= 1, got {k}")
    if n < k:
        raise ValueError(f"too few samples: need at least k={k}, got {n}")
    if iters < 1:
        raise ValueError(f"invalid parameter: iters must be >= 1, got {iters}")
    C = X[np.random.default_rng(seed).choice(n, size=k, replace=False)].copy()
    for _ in range(iters):
        sims = X @ C.T
        assign = np.argmax(sims, axis=1)
        sums = np.zeros_like(C)
        np.add.at(sums, assign, X)
        counts = np.bincount(assign, minlength=k)
        norms = np.linalg.norm(sums, axis=1)
        dead = np.flatnonzero((counts == 0) | (norms < 1e-12))
        if dead.size:
            best = sims[np.arange(n), assign]
            far = np.argsort(best, kind="stable")[:dead.size]
            sums[dead] = X[far]
            norms[dead] = 1.0
        C = sums / norms[:, None]
    return C


def build_centroid_index(docs, centroid_vectors) -> list[np.ndarray]:
    """Posting c = ascending doc indices with a vector whose argmax centroid is c.

    prefilter.py:85-108 (set semantics via np.unique; argmax = first on ties).
    """
    k = centroid_vectors.shape[0]
    postings: list[list[int]] = [[] for _ in range(k)]
    for i, S in enumerate(docs):
        X = _unit_rows(S, f"document {i}")
        nearest = np.unique(np.argmax(X @ centroid_vectors.T, axis=1))
        for c in nearest:
            postings[c].append(i)
    return [np.asarray(p, dtype=np.int64) for p in postings]


def filter_candidates(postings, n_docs: int, centroid_vectors, Q, probe: int,
                      k_filter: int) -> np.ndarray:
    """prefilter.py:111-144: stable top-probe centroids per query vector, +1
    per (query vector, probed posting), select (count desc, index asc)[:k_filter]."""
    if probe < 1:
        raise ValueError(f"invalid parameter: probe must be >= 1, got {probe}")
    if k_filter < 1:
        raise ValueError(f"invalid parameter: k_filter must be >= 1, got {k_filter}")
    Q = np.asarray(Q, dtype=np.float64)
    probe = min(probe, centroid_vectors.shape[0])
    sims = Q @ centroid_vectors.T
    probed = np.argsort(-sims, axis=1, kind="stable")[:, :probe]
    counts = np.zeros(n_docs, dtype=np.int64)
    for row in probed:
        for c in row:
            counts[postings[c]] += 1
    touched = np.flatnonzero(counts > 0)
    order = np.lexsort((touched, -counts[touched]))
    return touched[order][:k_filter]


# --------------------------------------------------------------------------
# whole-path helper used by tests / bench reference arm
# --------------------------------------------------------------------------

def query_codes_port(tables, doc_ids, qcodes, lut, top_k, candidates=None):
    """Score candidates with the ported reference path and rank (index.py:300-319)."""
    cand = range(len(tables)) if candidates is None else candidates
    scores = [score_port(tables[i], qcodes, lut) for i in cand]
    return rank_topk(scores, [doc_ids[i] for i in cand], top_k)


def isqrt_ceil(n: int) -> int:  # index.py:153 helper semantics
    return math.isqrt(n - 1) + 1
