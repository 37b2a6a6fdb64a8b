"""CPU reference timing for bench.py: the ``--impl reference`` arm and the
``cpu_baseline`` key of every config line.  Test/measurement infrastructure only.

The timed code is the UNMODIFIED reference package (``baseline/_ref/dessert``,
installed with ``pip install --no-index --no-deps --target baseline/_ref`` from
/root/reference/pkg) through its own public API:

* scoring configs (cfg1 / cfg4): ``dessert.build_index(docs, IndexConfig)``
  (untimed setup) and ``dessert.query(index, Q, top_k)`` -- hash Q,
  ``_score_chunk`` over every set, ``heapq.nsmallest`` with key (-score, doc_id)
  (reference pkg/src/dessert/index.py:131-167, 250-319);
* index build (cfg2): ``dessert.lsh.hash_matrix`` over a 1M-vector chunk
  (OpenBLAS on every core, lsh.py:90-106) and ``dessert.sketch.build_tiny_table``
  per set (sketch.py:51-80) on a fork pool.

Multi-core: one forked process per host core, each holding a contiguous shard of
the sample's sets (its own reference index); a step sends the same query sets
to every shard and merges the shard results with the reference key -- the
reference's ``query(threads=n)`` is GIL-bound and slower than one thread
(SURVEY.md section 6).  Step time = wall clock from dispatch to merged result.

When ``baseline/_ref`` is absent the oracle port (``oracle/dessert_oracle.py``,
a restatement of the same algorithm pinned by the golden fixtures) is timed
instead and the line says ``kind: "port"``.

Synthetic inputs follow BASELINE.json's configs (numpy only, no GPU code): set
sizes clip(round(N(70, sd)), 8, 180); vectors normalise(c + 0.05 N(0, I)) in
fp16 with c uniform over normalised N(0, I) centroids; query sets = 32 rows of
a random sample set with replacement + N(0, 0.1^2), renormalised.
"""

from __future__ import annotations

import heapq
import multiprocessing as mp
import os
import sys
import time

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
REF_DIR = os.path.join(REPO, "baseline", "_ref")


def reference_kind() -> str:
    return "reference" if os.path.isdir(os.path.join(REF_DIR, "dessert")) else "port"


def host_cores() -> int:
    return len(os.sched_getaffinity(0))


def _import_ref():
    if REF_DIR not in sys.path:
        sys.path.insert(0, REF_DIR)
    import dessert.index as ri  # noqa: E402  (never dessert.cli / dessert.report: matplotlib)
    import dessert.lsh as rl
    import dessert.sketch as rs

    return ri, rl, rs


# ------------------------------------------------------------------ inputs
def sample_inputs(n_sets, size_sd, n_centroids, n_qsets, seed, m_q=32, d=128):
    """(sizes, X fp16 (sum m, d), Q float64 (n_qsets, m_q, d)) for a bounded sample."""
    rng = np.random.default_rng(seed)
    sizes = np.clip(np.rint(rng.normal(70.0, size_sd, size=n_sets)), 8, 180).astype(np.int64)
    cents = rng.standard_normal((n_centroids, d)).astype(np.float32)
    cents /= np.linalg.norm(cents, axis=1, keepdims=True)
    n = int(sizes.sum())
    X = np.empty((n, d), dtype=np.float16)
    for lo in range(0, n, 1 << 20):
        hi = min(n, lo + (1 << 20))
        v = cents[rng.integers(0, n_centroids, size=hi - lo)] + \
            np.float32(0.05) * rng.standard_normal((hi - lo, d), dtype=np.float32)
        X[lo:hi] = (v / np.linalg.norm(v, axis=1, keepdims=True)).astype(np.float16)
    off = np.concatenate([[0], np.cumsum(sizes)])
    Q = np.empty((n_qsets, m_q, d), dtype=np.float64)
    for i in range(n_qsets):
        s = int(rng.integers(0, n_sets))
        rows = off[s] + rng.integers(0, sizes[s], size=m_q)
        q = X[rows].astype(np.float64) + 0.1 * rng.standard_normal((m_q, d))
        Q[i] = q / np.linalg.norm(q, axis=1, keepdims=True)
    return sizes, X, Q


# ----------------------------------------------------------- worker pool
_STATE = {}


def _limit_blas():
    try:
        from threadpoolctl import threadpool_limits

        threadpool_limits(1)
    except Exception:
        pass


def _worker(conn, lo, hi, L, C, kind):
    _limit_blas()
    sizes, X = _STATE["sizes"], _STATE["X"]
    off = np.concatenate([[0], np.cumsum(sizes)])
    docs = [(s, X[off[s]:off[s + 1]]) for s in range(lo, hi)]
    if kind == "reference":
        ri, _, _ = _import_ref()
        cfg = ri.IndexConfig(d=X.shape[1], C=C, L=L, seed=0, filter=ri.FilterConfig(enabled=False))
        index = ri.build_index(docs, cfg)

        def run(Q, k):
            return ri.query(index, Q, k)
    else:
        sys.path.insert(0, REPO)
        from oracle import dessert_oracle as O

        P = O.sample_planes(X.shape[1], C, L, 0)
        lut = O.sim_lut(C, L)
        tables = [O.build_tiny_table(O.hash_matrix(P, L, C, x.astype(np.float64)), L, 1 << C)
                  for _, x in docs]
        ids = [s for s, _ in docs]

        def run(Q, k):
            qc = O.hash_matrix(P, L, C, Q)
            sc = [O.score_port(t, qc, lut) for t in tables]
            best = heapq.nsmallest(k, zip(sc, ids), key=lambda e: (-e[0], e[1]))
            return [(i, s) for s, i in best]
    conn.send("ready")
    while True:
        msg = conn.recv()
        if msg is None:
            break
        Qs, k = msg
        t0 = time.perf_counter()
        out = [run(Q, k) for Q in Qs]
        conn.send((time.perf_counter() - t0, out))
    conn.close()


class ShardPool:
    """One forked process per core, each owning a contiguous shard of the sample."""

    def __init__(self, sizes, X, L, C, procs, kind):
        _STATE["sizes"], _STATE["X"] = sizes, X
        n = len(sizes)
        cuts = np.linspace(0, n, procs + 1).astype(np.int64)
        ctx = mp.get_context("fork")
        self.conns, self.procs = [], []
        for j in range(procs):
            a, b = ctx.Pipe()
            p = ctx.Process(target=_worker, args=(b, int(cuts[j]), int(cuts[j + 1]), L, C, kind),
                            daemon=True)
            p.start()
            self.conns.append(a)
            self.procs.append(p)
        for c in self.conns:
            assert c.recv() == "ready"
        _STATE.clear()

    def query(self, Qs, k):
        """Merged top-k per query set and (wall seconds, slowest shard seconds)."""
        t0 = time.perf_counter()
        for c in self.conns:
            c.send((Qs, k))
        parts = [c.recv() for c in self.conns]
        merged = [heapq.nsmallest(k, (e for _, out in parts for e in out[i]),
                                  key=lambda e: (-e[1], e[0])) for i in range(len(Qs))]
        return merged, time.perf_counter() - t0, max(t for t, _ in parts)

    def close(self):
        for c in self.conns:
            try:
                c.send(None)
            except Exception:
                pass
        for p in self.procs:
            p.join(timeout=10)


# ------------------------------------------------------------ scoring arms
def scoring_baseline(*, L, C, size_sd, n_centroids, top_k, n_sets, n_qsets_step, steps, warmup,
                     seed=7, procs=None):
    """Reference query() over a bounded sample: set-pairs/s per step (median)."""
    kind = reference_kind()
    procs = procs or host_cores()
    t_setup = time.perf_counter()
    sizes, X, Q = sample_inputs(n_sets, size_sd, n_centroids, n_qsets_step * max(1, steps), seed)
    pool = ShardPool(sizes, X, L, C, procs, kind)
    t_setup = time.perf_counter() - t_setup
    try:
        for _ in range(warmup):
            pool.query(Q[:1], top_k)
        walls = []
        for s in range(steps):
            _, wall, _ = pool.query(Q[s * n_qsets_step:(s + 1) * n_qsets_step], top_k)
            walls.append(wall)
    finally:
        pool.close()
    pairs = n_qsets_step * n_sets
    ms = float(np.median(walls)) * 1e3
    return {"value": pairs / (ms * 1e-3), "ms_per_step": ms, "pairs_per_step": pairs,
            "step_ms_all": [w * 1e3 for w in walls], "cores": procs, "kind": kind,
            "setup_s": t_setup, "n_sets": n_sets, "n_qsets_step": n_qsets_step}


def _tt_worker(args):
    _limit_blas()
    codes, off, lo, hi, L, r, kind = args
    if kind == "reference":
        _, _, rs = _import_ref()
        build = rs.build_tiny_table
    else:
        sys.path.insert(0, REPO)
        from oracle import dessert_oracle as O

        build = O.build_tiny_table
    t0 = time.perf_counter()
    for s in range(lo, hi):
        build(codes[off[s]:off[s + 1]], L, r)
    return time.perf_counter() - t0


def build_baseline(*, L, C, n_vec_hash=1 << 20, n_sets_tt=20_000, seed=9, procs=None):
    """cfg2 reference: hash_matrix on a 1M-vector chunk (OpenBLAS, all cores) +
    build_tiny_table on a fork pool -> vectors/s of the two stages combined."""
    kind = reference_kind()
    procs = procs or host_cores()
    rng = np.random.default_rng(seed)
    cents = rng.standard_normal((4096, 128))
    cents /= np.linalg.norm(cents, axis=1, keepdims=True)
    X = cents[rng.integers(0, 4096, size=n_vec_hash)] + 0.05 * rng.standard_normal((n_vec_hash, 128))
    X = (X / np.linalg.norm(X, axis=1, keepdims=True)).astype(np.float16).astype(np.float64)
    if kind == "reference":
        ri, rl, _ = _import_ref()
        fam = rl.sample_srp_family(128, C, L, 0)
        t0 = time.perf_counter()
        codes = rl.hash_matrix(fam, X)
        t_hash = time.perf_counter() - t0
    else:
        sys.path.insert(0, REPO)
        from oracle import dessert_oracle as O

        P = O.sample_planes(128, C, L, 0)
        t0 = time.perf_counter()
        codes = O.hash_matrix(P, L, C, X)
        t_hash = time.perf_counter() - t0
    sizes = np.clip(np.rint(rng.normal(70, 20, size=n_sets_tt)), 8, 180).astype(np.int64)
    off = np.concatenate([[0], np.cumsum(sizes)])
    need = int(off[-1])
    tt_codes = codes[np.arange(need) % n_vec_hash]
    cuts = np.linspace(0, n_sets_tt, procs + 1).astype(np.int64)
    ctx = mp.get_context("fork")
    t0 = time.perf_counter()
    with ctx.Pool(procs) as pool:
        times = pool.map(_tt_worker, [(tt_codes, off, int(cuts[j]), int(cuts[j + 1]), L, 1 << C, kind)
                                      for j in range(procs)])
    t_tt = time.perf_counter() - t0
    hash_rate = n_vec_hash / t_hash
    tt_rate = need / t_tt
    return {"value": 1.0 / (1.0 / hash_rate + 1.0 / tt_rate), "hash_vectors_per_s": hash_rate,
            "tinytable_vectors_per_s": tt_rate, "cores": procs, "kind": kind,
            "sample": f"hash_matrix on {n_vec_hash} vectors ({t_hash:.1f} s, OpenBLAS {procs} threads) "
                      f"+ build_tiny_table on {n_sets_tt} sets / {need} vectors ({t_tt:.1f} s, "
                      f"{procs}-process fork pool); value = 1/(1/hash + 1/tinytable) vectors/s"}


# ------------------------------------------------------------ cfg3 (prefilter pipeline)
class _PoolSketches:
    """A length-N sequence of reference TinyTables backed by a pool of real ones
    (set i -> pool[i % len(pool)]): the reference's query() only indexes
    index.sketches[i] and takes len(), so it runs unmodified over N sets."""

    def __init__(self, pool, n):
        self.pool, self.n = pool, n

    def __len__(self):
        return self.n

    def __getitem__(self, i):
        return self.pool[i % len(self.pool)]


def _cfg3_worker(args):
    _limit_blas()
    lo, hi, top_k = args
    ri, _, _ = _import_ref()
    index, Qs = _STATE["index"], _STATE["Q"]
    t0 = time.perf_counter()
    out = [ri.query(index, Qs[i], top_k) for i in range(lo, hi)]
    return time.perf_counter() - t0, len(out)


def cfg3_baseline(*, L=32, C=7, n_sets=1_000_000, n_cent=65536, probe=4, k_filter=4096, top_k=100,
                  n_qsets=16, pool_sets=2000, seed=11, procs=None):
    """cfg3 reference: the UNMODIFIED dessert.query with the centroid prefilter on a
    cfg3-shaped index -- 1M sets whose postings come from ~70M vectors drawn over
    65,536 centroids (prefilter.py:111-144 on the full-size CentroidIndex), and
    TinyTables from a pool of 2,000 real sets for the <= 4,096 candidates
    (_score_chunk, index.py:250-261) -- one query set per host core at a time."""
    kind = reference_kind()
    if kind != "reference":
        return None
    procs = procs or host_cores()
    ri, rl, rs = _import_ref()
    import dessert.prefilter as rp

    t_setup = time.perf_counter()
    rng = np.random.default_rng(seed)
    cents = rng.standard_normal((n_cent, 128))
    cents /= np.linalg.norm(cents, axis=1, keepdims=True)
    sizes = np.clip(np.rint(rng.normal(70.0, 20.0, size=n_sets)), 8, 180).astype(np.int64)
    off = np.concatenate([[0], np.cumsum(sizes)])
    n_vec = int(off[-1])
    vcent = rng.integers(0, n_cent, size=n_vec).astype(np.int64)  # each vector's centroid
    key = np.unique(vcent * n_sets + np.repeat(np.arange(n_sets, dtype=np.int64), sizes))
    pc, pdoc = np.divmod(key, n_sets)
    bounds = np.searchsorted(pc, np.arange(n_cent + 1))
    postings = [pdoc[bounds[c]:bounds[c + 1]] for c in range(n_cent)]
    del key, pc
    cfg = ri.IndexConfig(d=128, C=C, L=L, seed=0,
                         filter=ri.FilterConfig(enabled=True, centroids=n_cent, probe=probe,
                                                k_filter=k_filter))
    fam = rl.sample_srp_family(128, C, L, 0)
    pool = []
    for s in range(pool_sets):
        m = int(sizes[s])
        v = cents[vcent[off[s]:off[s] + m]] + 0.05 * rng.standard_normal((m, 128))
        v = (v / np.linalg.norm(v, axis=1, keepdims=True)).astype(np.float16).astype(np.float64)
        pool.append(rs.build_tiny_table(rl.hash_matrix(fam, v), L, 1 << C))
    index = ri.DessertIndex(config=cfg, family=fam, lookup=rl.build_sim_lookup(C, L),
                            sketches=_PoolSketches(pool, n_sets),
                            doc_ids=np.arange(n_sets, dtype=np.uint64),
                            sizes=sizes[np.arange(n_sets) % pool_sets],
                            filter=(rp.Centroids(k=n_cent, seed=0, vectors=cents),
                                    rp.CentroidIndex(n_docs=n_sets, postings=postings)))
    Q = np.empty((n_qsets, 32, 128))
    for i in range(n_qsets):  # 32 perturbed vectors of a random set (its vectors' centroids)
        s = int(rng.integers(0, n_sets))
        rows = off[s] + rng.integers(0, sizes[s], size=32)
        q = cents[vcent[rows]] + 0.05 * rng.standard_normal((32, 128)) + 0.1 * rng.standard_normal((32, 128))
        Q[i] = q / np.linalg.norm(q, axis=1, keepdims=True)
    t_setup = time.perf_counter() - t_setup
    _STATE["index"], _STATE["Q"] = index, Q
    cuts = np.linspace(0, n_qsets, min(procs, n_qsets) + 1).astype(np.int64)
    ctx = mp.get_context("fork")
    with ctx.Pool(len(cuts) - 1) as p:
        p.map(_cfg3_worker, [(int(cuts[j]), int(cuts[j]) + 1, top_k) for j in range(len(cuts) - 1)])  # warm-up
        t0 = time.perf_counter()
        per = p.map(_cfg3_worker, [(int(cuts[j]), int(cuts[j + 1]), top_k) for j in range(len(cuts) - 1)])
        wall = time.perf_counter() - t0
    _STATE.clear()
    return {"value": n_qsets / wall, "unit": "query sets/s", "cores": len(cuts) - 1, "kind": kind,
            "wall_s": wall, "setup_s": t_setup, "per_query_set_s": float(np.mean([t for t, _ in per])),
            "sample": f"{n_qsets} query sets through the unmodified dessert.query (prefilter probe "
                      f"{probe}, k_filter {k_filter}, top-{top_k}) on a cfg3-shaped index: {n_sets} sets, "
                      f"postings of {n_vec} vectors over {n_cent} centroids (filter_candidates at full "
                      f"size), candidate TinyTables from a pool of {pool_sets} real L={L} C={C} sets; "
                      f"{len(cuts) - 1}-process fork pool, one query set per process at a time"}
