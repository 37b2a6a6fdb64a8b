"""Index build and query -- drop-in for dessert.index (reference: pkg/src/dessert/index.py).

Same names, arguments, defaults, results and error messages as the
reference, executed by the sm_100a kernels in ``csrc/``:

* ``build_index``  (index.py:131-167): hash every vector on the GPU (K1),
  lay the codes out per set (K2: size scan -> CSR of bit-sliced records),
  optional centroid prefilter.
* ``query``        (index.py:264-319): hash Q (K1), prefilter (K5) or all
  sets, score (K3), top-k by (score desc, doc_id asc) (K4).
* ``query_batch``  (new, batched form of ``query`` for many query sets).
* ``score_candidate`` (index.py:230-247).
* ``add_sets``     (new: append sets to a built index; equals building over
  the concatenated docs when the prefilter is off).

The index is immutable during queries (queries never write to it), so
concurrent queries on different streams are safe.
"""

from __future__ import annotations

import gc
import math
import os
import threading
from dataclasses import dataclass, field, replace

import numpy as np
import torch

from . import engine
from .lsh import (SimLookup, SrpFamily, build_sim_lookup, default_mode, hash_device, sample_srp_family,
                  to_device_matrix)
from . import scoring
from .scoring import Scorer, avg_phi_aggregation, default_scorer, max_aggregation
from .sketch import SketchView

RankedResults = list[tuple[int, float]]

MAX_TRAIN_SAMPLES = 1 << 20
# Scores materialised per exhaustive pass before a top-k merge (bytes).
SCORE_BUFFER_BYTES = 4 << 30


@dataclass(frozen=True)
class FilterConfig:
    """Centroid prefilter settings; centroids=0 means ceil(sqrt(total vectors)) (index.py:35-44)."""

    enabled: bool = True
    centroids: int = 0
    iters: int = 10
    probe: int = 1
    k_filter: int = 4096


@dataclass(frozen=True)
class IndexConfig:
    """index.py:46-62."""

    d: int
    C: int = 7
    L: int = 32
    seed: int = 0
    inner_kind: str = "max"
    phi: str | None = None
    filter: FilterConfig = field(default_factory=FilterConfig)

    @property
    def code_range(self) -> int:
        return 1 << self.C

    def scorer(self) -> Scorer:
        inner = max_aggregation() if self.inner_kind == "max" else avg_phi_aggregation(self.phi)
        return Scorer(inner=inner, weights=None)


PROFILES: dict[str, dict] = {  # index.py:66-71 (paper App. B)
    "msmarco-k10-fast": {"C": 7, "L": 32, "k_filter": 4096, "probe": 1},
    "msmarco-k10-slow": {"C": 7, "L": 64, "k_filter": 4096, "probe": 2},
    "msmarco-k1000-fast": {"C": 6, "L": 32, "k_filter": 8192, "probe": 4},
    "msmarco-k1000-slow": {"C": 7, "L": 32, "k_filter": 16384, "probe": 4},
}


def apply_profile(config: IndexConfig, name: str) -> IndexConfig:
    """index.py:74-84."""
    if name not in PROFILES:
        raise ValueError(f"unknown profile: {name!r} (choose from {sorted(PROFILES)})")
    p = PROFILES[name]
    return replace(config, C=p["C"], L=p["L"],
                   filter=replace(config.filter, probe=p["probe"], k_filter=p["k_filter"]))


@dataclass
class DessertIndex:
    """N sets in the device layout plus the shared hash family, LUT and prefilter.

    Device state: ``records`` (sum m_i, R) int32 bit-sliced codes,
    ``set_off`` (N+1) int64, ``codes`` (sum m_i, L) raw codes (optional),
    ``lut_dev`` (L+1) float64, ``doc_ids_dev`` (N) int64.
    """

    config: IndexConfig
    family: SrpFamily
    lookup: SimLookup
    doc_ids: np.ndarray
    sizes: np.ndarray
    filter: tuple | None
    records: torch.Tensor
    set_off: torch.Tensor
    codes: torch.Tensor | None
    lut_dev: torch.Tensor
    doc_ids_dev: torch.Tensor
    _graphs: dict = field(default_factory=dict, repr=False, compare=False)

    @property
    def n_docs(self) -> int:
        return int(self.sizes.shape[0])

    @property
    def m_max(self) -> int:
        return int(self.sizes.max())

    @property
    def sketches(self) -> SketchView:
        return SketchView(self)

    @property
    def device(self):
        return self.records.device


# --------------------------------------------------------------------- build
def _validated_docs(docs, d: int):
    """index.py:108-128 (shape checks on the host; zero rows are found by K1)."""
    out, seen = [], set()
    for doc_id, S in docs:
        doc_id = int(doc_id)
        if doc_id in seen:
            raise ValueError(f"duplicate doc id: {doc_id}")
        seen.add(doc_id)
        X = S if isinstance(S, torch.Tensor) else np.asarray(S)
        if X.ndim != 2 or X.shape[0] == 0:
            raise ValueError(f"empty set: document {doc_id} has no vectors")
        if X.shape[1] != d:
            raise ValueError(
                f"dimension mismatch: document {doc_id} has d={X.shape[1]}, expected {d}")
        out.append((doc_id, X))
    if not out:
        raise ValueError("empty collection: nothing to index")
    return out


def _stack(items, device):
    mats = [X for _, X in items]
    if all(isinstance(X, torch.Tensor) for X in mats):
        dt = mats[0].dtype
        if any(X.dtype != dt for X in mats):
            mats = [X.to(torch.float64) for X in mats]
        return torch.cat([X.to(device) for X in mats], dim=0).contiguous()
    arrs = [X.cpu().numpy() if isinstance(X, torch.Tensor) else np.asarray(X) for X in mats]
    dt = arrs[0].dtype
    if dt not in (np.float32, np.float64, np.float16) or any(a.dtype != dt for a in arrs):
        arrs = [a.astype(np.float64) for a in arrs]
    return torch.from_numpy(np.ascontiguousarray(np.concatenate(arrs, axis=0))).to(device)


def _zero_row_doc(items) -> int:
    for doc_id, X in items:
        a = X.float().cpu().numpy() if isinstance(X, torch.Tensor) else np.asarray(X, np.float64)
        if np.any(np.linalg.norm(a, axis=1) == 0.0):
            return doc_id
    return -1


def _layout(sizes: np.ndarray, device):
    sizes_dev = torch.from_numpy(np.ascontiguousarray(sizes, dtype=np.int64)).to(device)
    set_off, bad = engine.sizes_to_offsets(sizes_dev)
    if int(bad.item()) != 0:
        raise ValueError("set too large: m must be <= 65535")
    return set_off


def build_from_vectors(X: torch.Tensor, sizes: np.ndarray, doc_ids, config: IndexConfig,
                       keep_codes: bool = True, hash_mode: int | None = None,
                       filt=None) -> DessertIndex:
    """Build from one device matrix of all vectors grouped by set (fast path)."""
    family = sample_srp_family(config.d, config.C, config.L, config.seed)
    lookup = build_sim_lookup(config.C, config.L)
    codes, recs = hash_device(family, X, mode=hash_mode, want_codes=keep_codes)
    set_off = _layout(sizes, X.device)
    ids = np.asarray(doc_ids, dtype=np.uint64)
    return DessertIndex(
        config=config, family=family, lookup=lookup, doc_ids=ids,
        sizes=np.asarray(sizes, dtype=np.int64), filter=filt, records=recs, set_off=set_off,
        codes=codes, lut_dev=torch.from_numpy(lookup.table).to(X.device),
        doc_ids_dev=torch.from_numpy(ids.view(np.int64)).to(X.device))


def build_from_codes(codes: torch.Tensor, sizes: np.ndarray, doc_ids, config: IndexConfig,
                     keep_codes: bool = True, filt=None) -> DessertIndex:
    """Build from precomputed (sum m_i, L) codes on the device (codes-only configs)."""
    family = sample_srp_family(config.d, config.C, config.L, config.seed)
    lookup = build_sim_lookup(config.C, config.L)
    recs, bad = engine.codes_to_records(codes, config.L, config.C)
    if int(bad.item()) != 0:
        raise ValueError(f"code out of range: codes must lie in [0, {config.code_range})")
    set_off = _layout(sizes, codes.device)
    ids = np.asarray(doc_ids, dtype=np.uint64)
    return DessertIndex(
        config=config, family=family, lookup=lookup, doc_ids=ids,
        sizes=np.asarray(sizes, dtype=np.int64), filter=filt, records=recs, set_off=set_off,
        codes=codes if keep_codes else None,
        lut_dev=torch.from_numpy(lookup.table).to(codes.device),
        doc_ids_dev=torch.from_numpy(ids.view(np.int64)).to(codes.device))


def build_from_records(records: torch.Tensor, sizes: np.ndarray, doc_ids, config: IndexConfig,
                       filt=None) -> DessertIndex:
    """Adopt device plane records (sum m_i, R) directly (codes-only configs)."""
    family = sample_srp_family(config.d, config.C, config.L, config.seed)
    lookup = build_sim_lookup(config.C, config.L)
    set_off = _layout(sizes, records.device)
    ids = np.asarray(doc_ids, dtype=np.uint64)
    return DessertIndex(
        config=config, family=family, lookup=lookup, doc_ids=ids,
        sizes=np.asarray(sizes, dtype=np.int64), filter=filt, records=records, set_off=set_off,
        codes=None, lut_dev=torch.from_numpy(lookup.table).to(records.device),
        doc_ids_dev=torch.from_numpy(ids.view(np.int64)).to(records.device))


def build_index(docs, config: IndexConfig, device="cuda", keep_codes: bool = True,
                hash_mode: int | None = None) -> DessertIndex:
    """Sketch every (doc_id, vector set) pair on the GPU and build the optional prefilter.

    index.py:131-167.  Deterministic in the inputs and config.seed.
    """
    items = _validated_docs(docs, config.d)
    X = _stack(items, device)
    sizes = np.array([x.shape[0] for _, x in items], dtype=np.int64)
    try:
        index = build_from_vectors(X, sizes, [i for i, _ in items], config, keep_codes, hash_mode)
    except ValueError as e:
        if str(e).startswith("zero vector"):
            raise ValueError(f"zero vector in document {_zero_row_doc(items)}") from None
        raise
    if config.filter.enabled:
        from .prefilter import build_centroid_index, train_centroids

        n = X.shape[0]
        pool_idx = None
        if n > MAX_TRAIN_SAMPLES:
            rng = np.random.default_rng([config.seed, 0xF117E2])
            pool_idx = rng.choice(n, size=MAX_TRAIN_SAMPLES, replace=False)
        n_pool = n if pool_idx is None else MAX_TRAIN_SAMPLES
        k = config.filter.centroids or math.isqrt(n_pool - 1) + 1
        k = min(k, n_pool)
        pool = X if pool_idx is None else X[torch.from_numpy(pool_idx).to(X.device)]
        centroids = train_centroids(pool, k, config.filter.iters, config.seed)
        cindex = build_centroid_index(X, centroids, set_off=index.set_off, n_docs=index.n_docs)
        index.filter = (centroids, cindex)
    return index


def add_sets(index: DessertIndex, docs) -> DessertIndex:
    """Append sets (new API).  Same result as building over the concatenated docs
    when the prefilter is off; with a prefilter the new sets are assigned to the
    existing centroids (no retraining)."""
    items = _validated_docs(docs, index.config.d)
    existing = set(int(i) for i in index.doc_ids)
    for doc_id, _ in items:
        if doc_id in existing:
            raise ValueError(f"duplicate doc id: {doc_id}")
    X = _stack(items, index.device)
    sizes = np.array([x.shape[0] for _, x in items], dtype=np.int64)
    try:
        codes, recs = hash_device(index.family, X, want_codes=index.codes is not None)
    except ValueError as e:
        if str(e).startswith("zero vector"):
            raise ValueError(f"zero vector in document {_zero_row_doc(items)}") from None
        raise
    # validate and build every new piece first; the index is updated only when all
    # of them succeeded (a failed call leaves it unchanged)
    all_sizes = np.concatenate([index.sizes, sizes])
    set_off = _layout(all_sizes, index.device)          # raises "set too large"
    new_filter = None
    if index.filter is not None:
        from .prefilter import extend_centroid_index

        centroids, cindex = index.filter
        new_filter = (centroids, extend_centroid_index(cindex, X, centroids, sizes))
    records = torch.cat([index.records, recs])
    codes_all = torch.cat([index.codes, codes]) if index.codes is not None else None
    doc_ids = np.concatenate([index.doc_ids, np.array([i for i, _ in items], np.uint64)])
    doc_ids_dev = torch.from_numpy(doc_ids.view(np.int64)).to(index.device)
    index.records, index.codes, index.set_off, index.sizes = records, codes_all, set_off, all_sizes
    index.doc_ids, index.doc_ids_dev = doc_ids, doc_ids_dev
    if new_filter is not None:
        index.filter = new_filter
    return index


# --------------------------------------------------------------------- query
def _rank(scores: torch.Tensor, top_k: int, ids: torch.Tensor, n_valid=None, cand=None):
    """Row-wise (score desc, doc_id asc) top-k on the device (K4, any k).  With ``cand``
    (candidate set indices per row), element i of row r has doc id ids[cand[r, i]]."""
    rows, n = scores.shape
    k = max(1, min(top_k, n))
    if cand is not None:  # ids gathered inside the kernel
        return engine.topk(scores, k, ids=ids, n_valid=n_valid, id_index=cand.contiguous())
    return engine.topk(scores, k, ids=ids, n_valid=n_valid)


_NP_DTYPE = {torch.float64: np.float64, torch.int64: np.int64, torch.int32: np.int32,
             torch.uint8: np.uint8, torch.float32: np.float32}


def _results(out_s, out_i) -> list[RankedResults]:
    """(scores, ids) as device / host tensors or numpy arrays -> ranked (doc id, score) lists."""
    s = out_s if isinstance(out_s, np.ndarray) else out_s.cpu().numpy()
    ids = (out_i if isinstance(out_i, np.ndarray) else out_i.cpu().numpy()).view(np.uint64)
    res = []
    for r in range(s.shape[0]):
        valid = s[r] >= 0.0
        res.append(list(zip(ids[r][valid].tolist(), s[r][valid].tolist())))  # (int, float) pairs
    return res


def _candidates(index: DessertIndex, Qdev: torch.Tensor, m_q: int, probe, k_filter):
    from .prefilter import filter_candidates_device

    centroids, cindex = index.filter
    cfg = index.config.filter
    return filter_candidates_device(cindex, centroids, Qdev, m_q,
                                    cfg.probe if probe is None else probe,
                                    cfg.k_filter if k_filter is None else k_filter)


@dataclass
class ScorePlan:
    """A non-default Scorer resolved for the device (K3g, dsrt_score_agg)."""

    kind: int                    # 0 max, 1 avg-phi
    table: torch.Tensor          # (L+1) float64: lut or phi(lut)
    weights: torch.Tensor | None  # (m_q) float64 or None (all ones)
    m_cap: int                   # largest set size (avg-phi count scratch)


def score_plan(index: DessertIndex, scorer: Scorer | None, m_q: int) -> ScorePlan | None:
    """Resolve ``scorer or index.config.scorer()`` (index.py:285-287); None = fast path."""
    scorer = scorer or index.config.scorer()
    weights = scoring.resolve_weights(scorer, m_q)
    kind = scoring.inner_kind_code(scorer)
    if kind == 0 and weights is None and _fast_kernels(index.config.L, index.config.C):
        return None  # shapes outside the K3 register envelope take the general kernel
    table = scoring.table_for(index.lookup.table, scorer)
    return ScorePlan(
        kind=kind,
        table=torch.from_numpy(np.ascontiguousarray(table, dtype=np.float64)).to(index.device),
        weights=(None if weights is None else
                 torch.from_numpy(np.ascontiguousarray(weights)).to(index.device)),
        m_cap=index.m_max if kind == 1 else 0)


def _score_plan_sets(index: DessertIndex, qrecs, m_q: int, plan: ScorePlan, cand=None,
                     n_cand=None, n_q=None, cand_ld=None):
    return engine.score_agg(index.records, index.set_off, qrecs, m_q, index.config.L,
                            index.config.C, plan.table, plan.kind, weights=plan.weights,
                            m_cap=plan.m_cap, cand=cand, n_cand=n_cand, cand_ld=cand_ld,
                            n_qsets=n_q)


def _rank_records_plan(index: DessertIndex, qrecs, m_q: int, top_k: int, plan: ScorePlan,
                       cand, n_cand):
    n_q = qrecs.shape[0] // m_q
    N = index.n_docs
    if cand is not None:
        scores = _score_plan_sets(index, qrecs, m_q, plan, cand=cand, n_cand=n_cand)
        out_s, out_i, _ = _rank(scores, top_k, index.doc_ids_dev, n_valid=n_cand, cand=cand)
        return out_s, out_i
    if plan.kind == 0 and _fast_kernels(index.config.L, index.config.C):
        # weighted sigma = max: the fused exhaustive search (weights in the K3 epilogue)
        return _search(index, qrecs, m_q, top_k, plan.weights, 0)
    chunk = max(1, min(N, SCORE_BUFFER_BYTES // (8 * n_q)))
    if chunk >= N:
        scores = _score_plan_sets(index, qrecs, m_q, plan, n_q=n_q, cand_ld=N)
        out_s, out_i, _ = _rank(scores, top_k, index.doc_ids_dev)
        return out_s, out_i
    parts_s, parts_i = [], []
    for s0 in range(0, N, chunk):
        s1 = min(N, s0 + chunk)
        sets = torch.arange(s0, s1, device=index.device).expand(n_q, s1 - s0).contiguous()
        scores = _score_plan_sets(index, qrecs, m_q, plan, cand=sets)
        ps, pi, _ = _rank(scores, top_k, index.doc_ids_dev[s0:s1])
        parts_s.append(ps)
        parts_i.append(pi)
    out_s, out_i, _ = _rank(torch.cat(parts_s, dim=1).contiguous(), top_k,
                            torch.cat(parts_i, dim=1).contiguous())
    return out_s, out_i


def _fast_kernels(L: int, C: int) -> bool:
    """The K3 kernels' envelope (score_max_fast_supported in score.cu)."""
    return 1 <= L <= 128 and 1 <= C <= 16 and C * ((L + 31) // 32) <= 32


def rank_records(index: DessertIndex, qrecs: torch.Tensor, m_q: int, top_k: int,
                 cand=None, n_cand=None, plan: ScorePlan | None = None, exhaustive_mode: int = 0):
    """Score query-set records (n_qsets*m_q, R) and rank; returns (scores, ids) (n_qsets, k).

    ``plan`` (from ``score_plan``) selects the general aggregation kernel for
    a non-default Scorer; None runs the sigma=max / unit-weight kernels.
    """
    if plan is not None:
        return _rank_records_plan(index, qrecs, m_q, top_k, plan, cand, n_cand)
    n_q = qrecs.shape[0] // m_q
    L, C = index.config.L, index.config.C
    N = index.n_docs
    if cand is not None:
        scores, _ = engine.score_candidates(index.records, index.set_off, qrecs, m_q, L, C,
                                            index.lut_dev, cand=cand, n_cand=n_cand)
        out_s, out_i, _ = _rank(scores, top_k, index.doc_ids_dev, n_valid=n_cand, cand=cand)
        return out_s, out_i
    return _search(index, qrecs, m_q, top_k, None, exhaustive_mode)


def _search(index: DessertIndex, qrecs, m_q: int, top_k: int, weights, mode: int):
    """Exhaustive ranking of every set (dsrt_search_all: K3 + K4 without the score
    matrix).  Threshold mode (0) reruns materialised (1) when a survivor list
    overflowed; mode 1 alone inside CUDA-graph capture (no host sync)."""
    L, C = index.config.L, index.config.C
    k = max(1, min(top_k, index.n_docs))
    args = (index.records, index.set_off, index.doc_ids_dev, qrecs, m_q, L, C, index.lut_dev, k)
    if mode == 0 and torch.cuda.is_current_stream_capturing():
        mode = 1
    out_s, out_i, ovf = engine.search_all(*args, weights=weights, mode=mode,
                                          score_buffer_bytes=SCORE_BUFFER_BYTES)
    if mode == 0 and int(ovf.item()) != 0:
        out_s, out_i, _ = engine.search_all(*args, weights=weights, mode=1,
                                            score_buffer_bytes=SCORE_BUFFER_BYTES)
    return out_s, out_i


# ------------------------------------------------- CUDA-graph query path
# query() on one query set is a fixed sequence of ~12 small kernels; replaying
# it as a CUDA graph removes the host launch overhead from batch-1 latency.
# A graph is captured per (query shape, dtype, top_k, probe, k_filter) and is
# rebuilt when the index's device buffers or prefilter change (add_sets,
# filter reassignment).  DSRT_QUERY_GRAPHS=0 disables the path.
_GRAPH_CACHE = 8


class _QueryGraph:
    # Holds the captured tensors (deps) but not the index itself: an index <-> graph
    # reference cycle would leave dropped indexes to the cyclic GC, which could then
    # destroy their graphs (and free their pools) in the middle of another capture.
    def __init__(self, index: DessertIndex, q: torch.Tensor, top_k: int, probe, k_filter):
        self.top_k, self.probe, self.k_filter = top_k, probe, k_filter
        self.deps = self._deps(index)
        self.lock = threading.Lock()
        self.done = None  # event: last replay's outputs copied out
        self.q_in = torch.empty(q.shape, dtype=q.dtype, device=index.device)
        self.q_in.copy_(q)
        warm = self._run(index)  # eager warm-up: lazy initialisation outside the capture
        torch.cuda.synchronize()
        # Host queries: the H2D copy of the query and the D2H copies of the results are
        # nodes of the graph (pinned staging buffers), so a call is one host memcpy, one
        # replay and one synchronisation instead of a pageable copy in and four
        # synchronous copies out (batch-1 p50 0.240 -> see DESIGN K5 "small batches").
        self.host_io = not q.is_cuda
        self.q_host = self.out_host = None
        if self.host_io:
            self.q_host = torch.empty(q.shape, dtype=q.dtype, pin_memory=True)
            self.q_host.copy_(q)
            # one pinned buffer for (scores, ids, zero-row count, candidate counts): a single
            # pack kernel writes it over the bus (a D2H copy node per tensor costs ~3.5 us each)
            self.out_meta = [None if t is None else (tuple(t.shape), _NP_DTYPE[t.dtype], t.numel() * t.element_size())
                             for t in warm]
            self.out_offs, total = engine.pack_layout(warm)
            self.out_host = torch.empty(total, dtype=torch.uint8, pin_memory=True)
            self.out_np = self.out_host.numpy()
        del warm
        self.graph = torch.cuda.CUDAGraph()
        gc_on = gc.isenabled()
        gc.disable()
        try:
            with torch.cuda.graph(self.graph, capture_error_mode="thread_local"):
                if self.host_io:
                    engine.copy_async(self.q_in, self.q_host)
                self.out = self._run(index)
                if self.host_io:
                    self.out = tuple(None if t is None else t.contiguous() for t in self.out)
                    engine.pack4(self.out_host, self.out)
        finally:
            if gc_on:
                gc.enable()

    @staticmethod
    def _deps(index):
        return (index.records, index.set_off, index.lut_dev, index.doc_ids_dev, index.filter)

    def valid(self, index) -> bool:
        return all(a is b for a, b in zip(self.deps, self._deps(index)))

    def _run(self, ix: DessertIndex):
        q = self.q_in
        m_q = q.shape[-2]
        Qdev = to_device_matrix(q.reshape(-1, q.shape[-1]), ix.config.d, ix.device)
        mode = default_mode(Qdev.dtype, Qdev.shape[1], ix.config.C, Qdev.shape[0], ix.config.L)
        _, qrecs, zero = engine.hash_vectors(Qdev, ix.family.device_planes(mode, ix.device), mode,
                                             ix.config.L, ix.config.C, want_codes=False,
                                             want_records=True, check_zero=True)
        cand = n_cand = None
        if ix.filter is not None:
            cand, n_cand = _candidates(ix, Qdev, m_q, self.probe, self.k_filter)
        out_s, out_i = rank_records(ix, qrecs, m_q, self.top_k, cand, n_cand, exhaustive_mode=1)
        return out_s, out_i, zero, n_cand

    def __call__(self, q: torch.Tensor, to_host: bool = True):
        # The captured buffers (q_in, outputs) are shared by every caller: the next
        # caller's stream waits until the previous replay and its output copies
        # finished (they may run on another stream when to_host=False).
        stream = torch.cuda.current_stream()
        if self.done is not None:
            stream.wait_event(self.done)
        if self.host_io:
            self.q_host.copy_(q)  # the graph's first node uploads it
        else:
            self.q_in.copy_(q, non_blocking=True)
        self.graph.replay()
        if to_host and self.host_io:
            stream.synchronize()
            self.done = None
            raw = self.out_np.copy()  # the pinned buffer is reused by the next call
            out = []
            for meta, off in zip(self.out_meta, self.out_offs):
                if meta is None:
                    out.append(None)
                    continue
                shape, dtype, nbytes = meta
                out.append(raw[off:off + nbytes].view(dtype).reshape(shape))  # numpy views of the copy
            return tuple(out)
        if to_host:
            out = tuple(None if t is None else t.cpu() for t in self.out)
        else:
            out = tuple(None if t is None else t.clone() for t in self.out)
        self.done = torch.cuda.Event()
        self.done.record(stream)
        return out


def _graph_ok(index: DessertIndex, n_q: int) -> bool:
    """Graphs pin their scratch: used for the prefiltered path and for exhaustive
    scoring whose score buffer stays small."""
    return (index.device.type == "cuda" and os.environ.get("DSRT_QUERY_GRAPHS", "1") != "0"
            and (index.filter is not None or n_q * index.n_docs * 8 <= (256 << 20)))


def _query_graphed(index: DessertIndex, Qa, top_k: int, probe, k_filter, to_host: bool = True):
    """query() / query_batch() through a cached CUDA graph; None when the graph is
    busy (another thread) so the caller runs the eager path.  Returns
    (out_s, out_i, n_cand) on the host (to_host) or as device copies."""
    q = Qa if isinstance(Qa, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(Qa))
    key = (tuple(q.shape), q.dtype, str(q.device), top_k, probe, k_filter)
    g = index._graphs.get(key)
    if g is not None and not g.valid(index):
        index._graphs.pop(key, None)
        g = None
    if g is None:
        if len(index._graphs) >= _GRAPH_CACHE:
            index._graphs.pop(next(iter(index._graphs)))
        g = _QueryGraph(index, q, top_k, probe, k_filter)
        index._graphs[key] = g
    if not g.lock.acquire(blocking=False):
        return None
    try:
        out_s, out_i, zero, n_cand = g(q, to_host)
    finally:
        g.lock.release()
    if int(zero[0].item() if isinstance(zero, torch.Tensor) and zero.is_cuda else zero[0]) != 0:
        raise ValueError("zero vector cannot be hashed (sign of zero projection undefined)")
    return out_s, out_i, n_cand


def query(index: DessertIndex, Q, top_k: int, probe: int | None = None,
          k_filter: int | None = None, scorer: Scorer | None = None,
          threads: int = 1) -> RankedResults:
    """Rank the top_k sets for one query vector set (index.py:264-319).

    ``threads`` is accepted for signature compatibility; results never depend
    on it (the device path is deterministic).
    """
    if top_k < 1:
        raise ValueError(f"invalid parameter: top_k must be >= 1, got {top_k}")
    Qa = Q if isinstance(Q, torch.Tensor) else np.asarray(Q, dtype=np.float64)
    if Qa.ndim != 2 or Qa.shape[0] == 0:
        raise ValueError("empty query: need at least one query vector")
    plan = score_plan(index, scorer, Qa.shape[0])
    if plan is None and Qa.shape[1] == index.config.d and _graph_ok(index, 1):
        res = _query_graphed(index, Qa, top_k, probe, k_filter)
        if res is not None:
            out_s, out_i, n_cand = res
            if n_cand is not None and int(n_cand[0]) == 0:
                return []
            return _results(out_s, out_i)[0]
    Qdev = to_device_matrix(Qa, index.config.d, index.device)
    _, qrecs = hash_device(index.family, Qdev, want_codes=False)
    m_q = Qdev.shape[0]
    cand = n_cand = None
    if index.filter is not None:
        cand, n_cand = _candidates(index, Qdev, m_q, probe, k_filter)
        if int(n_cand[0].item()) == 0:
            return []
    out_s, out_i = rank_records(index, qrecs, m_q, top_k, cand, n_cand, plan)
    return _results(out_s, out_i)[0]


def query_batch(index: DessertIndex, Qs, top_k: int, probe: int | None = None,
                k_filter: int | None = None, scorer: Scorer | None = None,
                return_tensors: bool = False):
    """Batched ``query`` over n_qsets query sets of equal size m_q.

    Qs: (n_qsets, m_q, d).  Returns a list of RankedResults, or the device
    tensors (scores (n_qsets, k), doc ids (n_qsets, k)) with return_tensors.
    """
    if top_k < 1:
        raise ValueError(f"invalid parameter: top_k must be >= 1, got {top_k}")
    if isinstance(Qs, torch.Tensor):
        t = Qs
    else:
        t = torch.from_numpy(np.ascontiguousarray(np.asarray(Qs)))
    if t.dim() != 3 or t.shape[1] == 0:
        raise ValueError("empty query: need at least one query vector")
    n_q, m_q, d = t.shape
    plan = score_plan(index, scorer, m_q)
    if plan is None and d == index.config.d and _graph_ok(index, n_q):
        res = _query_graphed(index, t, top_k, probe, k_filter, to_host=not return_tensors)
        if res is not None:
            out_s, out_i, _ = res
            return (out_s, out_i) if return_tensors else _results(out_s, out_i)
    Qdev = to_device_matrix(t.reshape(n_q * m_q, d), index.config.d, index.device)
    _, qrecs = hash_device(index.family, Qdev, want_codes=False)
    cand = n_cand = None
    if index.filter is not None:
        cand, n_cand = _candidates(index, Qdev, m_q, probe, k_filter)
    out_s, out_i = rank_records(index, qrecs, m_q, top_k, cand, n_cand, plan)
    if return_tensors:
        return out_s, out_i
    return _results(out_s, out_i)


def query_codes_batch(index: DessertIndex, qcodes, top_k: int, return_tensors=False,
                      scorer: Scorer | None = None):
    """Rank from precomputed query codes (n_qsets, m_q, L) -- the parity hook
    ("both sides given the same hash codes")."""
    t = qcodes if isinstance(qcodes, torch.Tensor) else torch.from_numpy(np.asarray(qcodes))
    n_q, m_q, L = t.shape
    if L != index.config.L:
        raise ValueError(f"expected (m_q, {index.config.L}) code matrix, got shape {tuple(t.shape)}")
    codes = t.reshape(n_q * m_q, L).to(index.device).to(torch.int32).contiguous()
    qrecs, bad = engine.codes_to_records(codes, L, index.config.C)
    out_s, out_i = rank_records(index, qrecs, m_q, top_k, plan=score_plan(index, scorer, m_q))
    if return_tensors:
        return out_s, out_i
    return _results(out_s, out_i)


def score_candidate(index: DessertIndex, i: int, query_codes, scorer: Scorer | None = None) -> float:
    """index.py:230-247: relevance of set i for an (m_q, L) code matrix."""
    if not 0 <= i < index.n_docs:
        raise IndexError(f"set index out of range: {i} (N={index.n_docs})")
    qc = np.asarray(query_codes)
    if qc.ndim != 2 or qc.shape[1] != index.config.L:
        raise ValueError(f"expected (m_q, {index.config.L}) code matrix, got shape {qc.shape}")
    if qc.shape[0] == 0:
        scoring.resolve_weights(scorer or index.config.scorer(), 0)
        return float("nan")  # np.mean of an empty array (reference warns and returns nan)
    plan = score_plan(index, scorer, qc.shape[0])
    codes = torch.from_numpy(qc.astype(np.int32)).to(index.device)
    qrecs, _ = engine.codes_to_records(codes, index.config.L, index.config.C, check=False)
    cand = torch.tensor([[i]], dtype=torch.int64, device=index.device)
    if plan is not None:
        return float(_score_plan_sets(index, qrecs, qc.shape[0], plan, cand=cand)[0, 0].item())
    scores, _ = engine.score_candidates(index.records, index.set_off, qrecs, qc.shape[0],
                                        index.config.L, index.config.C, index.lut_dev, cand=cand)
    return float(scores[0, 0].item())


def score_matrix(index: DessertIndex, qcodes, sets=None, want_counts=False,
                 scorer: Scorer | None = None):
    """Scores (and optional integer max counts c_q) of query code sets vs sets (parity API).

    With a non-default ``scorer`` returns (scores, None) from the general kernel."""
    t = qcodes if isinstance(qcodes, torch.Tensor) else torch.from_numpy(np.asarray(qcodes))
    n_q, m_q, L = t.shape
    codes = t.reshape(n_q * m_q, L).to(index.device).to(torch.int32).contiguous()
    qrecs, _ = engine.codes_to_records(codes, L, index.config.C, check=False)
    plan = score_plan(index, scorer, m_q)
    if plan is not None:
        if want_counts:
            raise ValueError("invalid parameter: want_counts needs the default scorer")
        if sets is None:
            return _score_plan_sets(index, qrecs, m_q, plan, n_q=n_q, cand_ld=index.n_docs), None
        cand = sets if isinstance(sets, torch.Tensor) else torch.from_numpy(np.asarray(sets, np.int64))
        return _score_plan_sets(index, qrecs, m_q, plan, cand=cand.to(index.device).contiguous()), None
    if sets is None:
        if n_q >= 8:
            return engine.score_all(index.records, index.set_off, qrecs, m_q, L, index.config.C,
                                    index.lut_dev, want_counts=want_counts)
        return engine.score_candidates(index.records, index.set_off, qrecs, m_q, L,
                                       index.config.C, index.lut_dev, cand_ld=index.n_docs,
                                       n_qsets=n_q, want_counts=want_counts)
    cand = sets if isinstance(sets, torch.Tensor) else torch.from_numpy(np.asarray(sets, np.int64))
    cand = cand.to(index.device).contiguous()
    return engine.score_candidates(index.records, index.set_off, qrecs, m_q, L, index.config.C,
                                   index.lut_dev, cand=cand, want_counts=want_counts)


__all__ = ["FilterConfig", "IndexConfig", "PROFILES", "apply_profile", "DessertIndex",
           "RankedResults", "build_index", "build_from_vectors", "build_from_codes",
           "build_from_records", "add_sets",
           "query", "query_batch", "query_codes_batch", "score_candidate", "score_matrix",
           "default_scorer", "ScorePlan", "score_plan"]
