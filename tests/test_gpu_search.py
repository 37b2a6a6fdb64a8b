"""Fused exhaustive search (dsrt_search_all), large-k top-k, sharded merge and the
round-2 fixes, checked bit-exactly against the oracle.  Needs a B200.

Reference behaviour: query()'s exhaustive branch = _score_chunk over every set
+ heapq.nsmallest(top_k, key=(-score, doc_id)) (index.py:250-261, 302-319)."""

import numpy as np
import pytest
import torch

import paper_2210_15748_b200 as d
from oracle import c_oracle
from oracle import dessert_oracle as O
from paper_2210_15748_b200 import engine
from paper_2210_15748_b200 import index as I
from paper_2210_15748_b200.distributed import merge_topk_device, shard_bounds

pytestmark = pytest.mark.gpu
DEV = "cuda"


def _case(seed, n_sets, L, C, n_q, m_q, lo=4, hi=60, ids=None):
    rng = np.random.default_rng(seed)
    sizes = rng.integers(lo, hi, size=n_sets).astype(np.int64)
    codes = rng.integers(0, 1 << C, size=(int(sizes.sum()), L)).astype(np.int32)
    # query sets: noisy copies of random sets' rows so top scores are spread out
    off = np.concatenate([[0], np.cumsum(sizes)])
    q = np.empty((n_q, m_q, L), dtype=np.int32)
    for i in range(n_q):
        s = int(rng.integers(0, n_sets))
        rows = codes[off[s] + rng.integers(0, sizes[s], size=m_q)].copy()
        flip = rng.random(rows.shape) < 0.5
        rows[flip] = rng.integers(0, 1 << C, size=int(flip.sum()))
        q[i] = rows
    doc_ids = rng.permutation(10 * n_sets)[:n_sets].astype(np.int64) if ids is None else ids
    return sizes, off, codes, q, doc_ids


def _index(codes, sizes, L, C, doc_ids):
    cfg = d.IndexConfig(d=4, C=C, L=L, filter=d.FilterConfig(enabled=False))
    return d.build_from_codes(torch.from_numpy(codes).to(DEV), sizes, doc_ids, cfg)


def _want(codes, off, q, lut, doc_ids, k, weights=None):
    if weights is None:
        S = c_oracle.score(codes, off, q, lut)
    else:
        S = np.stack([O.score_sets_dense_agg(q[r], codes, off, lut, "max", weights)
                      for r in range(q.shape[0])])
    return [O.rank_topk(S[r], doc_ids, k) for r in range(q.shape[0])], S


def _rows(out_s, out_i):
    s, i = out_s.cpu().numpy(), out_i.cpu().numpy().view(np.uint64)
    return [[(int(a), float(b)) for a, b in zip(i[r][s[r] >= 0], s[r][s[r] >= 0])]
            for r in range(s.shape[0])]


@pytest.mark.parametrize("L,C,m_q,k", [(32, 8, 32, 10), (64, 7, 32, 100), (32, 6, 17, 50),
                                       (16, 4, 100, 7)])
def test_search_threshold_equals_materialised_and_oracle(L, C, m_q, k, monkeypatch):
    monkeypatch.setenv("DSRT_SEARCH_MIN_BYTES", "0")  # threshold rounds at test size
    sizes, off, codes, q, ids = _case(L + C + m_q, 24_000, L, C, 16, m_q)
    idx = _index(codes, sizes, L, C, ids)
    want, _ = _want(codes, off, q, idx.lookup.table, ids, k)
    qrecs, _ = engine.codes_to_records(torch.from_numpy(q.reshape(-1, L)).to(DEV), L, C)
    args = (idx.records, idx.set_off, idx.doc_ids_dev, qrecs, m_q, L, C, idx.lut_dev, k)
    for mode, buf in ((0, 4 << 30), (1, 4 << 30), (1, 8 * 16 * 3000)):  # last: chunked
        s, i, ovf = engine.search_all(*args, mode=mode, score_buffer_bytes=buf)
        assert int(ovf.item()) == 0
        assert _rows(s, i) == want, (mode, buf)
    # the public API end to end (query_codes_batch -> rank_records -> _search)
    assert d.query_codes_batch(idx, q, k) == want


@pytest.mark.parametrize("n_q", [70, 128])
def test_search_cluster_pairs_opt_in(n_q, monkeypatch):
    """The opt-in cluster-pair mode of the exhaustive kernel (record tiles multicast to
    both CTAs of a pair; 70 query sets = 3 groups padded to 4, one CTA without query
    sets) returns the same ranking as the oracle, threshold and materialised."""
    monkeypatch.setenv("DSRT_SEARCH_MIN_BYTES", "0")
    monkeypatch.setenv("DSRT_ALL_CLUSTER", "1")
    L, C, m_q, k = 32, 8, 32, 20
    sizes, off, codes, q, ids = _case(n_q, 9000, L, C, n_q, m_q)
    idx = _index(codes, sizes, L, C, ids)
    want, _ = _want(codes, off, q, idx.lookup.table, ids, k)
    qrecs, _ = engine.codes_to_records(torch.from_numpy(q.reshape(-1, L)).to(DEV), L, C)
    args = (idx.records, idx.set_off, idx.doc_ids_dev, qrecs, m_q, L, C, idx.lut_dev, k)
    for mode in (0, 1):
        s, i, ovf = engine.search_all(*args, mode=mode, score_buffer_bytes=4 << 30)
        assert int(ovf.item()) == 0
        assert _rows(s, i) == want, mode


def test_search_overflow_falls_back_exactly(monkeypatch):
    """Sets ordered by ascending score: the seed threshold admits nearly every later
    set, the survivor lists overflow, the flag is raised and rank_records reruns
    materialised -- results still equal the oracle."""
    monkeypatch.setenv("DSRT_SEARCH_MIN_BYTES", "0")
    L, C, m_q, k = 32, 8, 32, 5
    sizes, off, codes, q, _ = _case(3, 30_000, L, C, 8, m_q)
    q = np.repeat(q[:1], 8, axis=0)  # one query set repeated: one score order for all rows
    S = c_oracle.score(codes, off, q[:1], O.sim_lut(C, L))[0]
    order = np.argsort(S, kind="stable")
    codes2 = np.concatenate([codes[off[s]:off[s + 1]] for s in order])
    sizes2 = sizes[order]
    off2 = np.concatenate([[0], np.cumsum(sizes2)])
    ids = np.arange(len(sizes2), dtype=np.int64)[::-1].copy()  # ids descending: ties by id matter
    idx = _index(codes2, sizes2, L, C, ids)
    want, _ = _want(codes2, off2, q, idx.lookup.table, ids, k)
    qrecs, _ = engine.codes_to_records(torch.from_numpy(q.reshape(-1, L)).to(DEV), L, C)
    s, i, ovf = engine.search_all(idx.records, idx.set_off, idx.doc_ids_dev, qrecs, m_q, L, C,
                                  idx.lut_dev, k, mode=0)
    assert int(ovf.item()) == 1
    assert d.query_codes_batch(idx, q, k) == want


def test_search_weighted_max_and_graph_path(monkeypatch):
    monkeypatch.setenv("DSRT_SEARCH_MIN_BYTES", "0")
    L, C, m_q, k = 32, 7, 32, 20
    sizes, off, codes, q, ids = _case(11, 12_000, L, C, 9, m_q)
    idx = _index(codes, sizes, L, C, ids)
    w = np.random.default_rng(2).random(m_q)
    want, _ = _want(codes, off, q, idx.lookup.table, ids, k, weights=w)
    sc = d.Scorer(inner=d.max_aggregation(), weights=w)
    assert d.query_codes_batch(idx, q, k, scorer=sc) == want


@pytest.mark.parametrize("m_q", [129, 200])
def test_search_large_m_q_and_few_query_sets(m_q):
    L, C, k = 32, 6, 25
    sizes, off, codes, q, ids = _case(m_q, 3000, L, C, 3, m_q)
    idx = _index(codes, sizes, L, C, ids)
    want, _ = _want(codes, off, q, idx.lookup.table, ids, k)
    assert d.query_codes_batch(idx, q, k) == want
    assert d.query_codes_batch(idx, np.concatenate([q] * 3), k) == want * 3


def test_finalize_large_m_q_candidate_lists_skip_unwritten_rows():
    """m_q > 128 with n_cand < cand_ld and invalid (-1) candidates: valid rows match
    the oracle, invalid set indices give NaN, rows past n_cand are not touched."""
    L, C, m_q = 32, 7, 160
    sizes, off, codes, q, ids = _case(7, 500, L, C, 2, m_q)
    idx = _index(codes, sizes, L, C, ids)
    cand = np.full((2, 64), -1, dtype=np.int64)
    cand[0, :40] = np.arange(40) * 7
    cand[1, :10] = np.arange(10)
    cand[1, 3] = -1
    n_cand = torch.tensor([40, 10], dtype=torch.int32, device=DEV)
    qrecs, _ = engine.codes_to_records(torch.from_numpy(q.reshape(-1, L)).to(DEV), L, C)
    scores = torch.full((2, 64), 7.0, dtype=torch.float64, device=DEV)
    engine._lib.call("dsrt_score_candidates", engine._ptr(idx.records), engine._ptr(idx.set_off),
                     len(sizes), engine._ptr(torch.from_numpy(cand).to(DEV)), engine._ptr(n_cand),
                     64, engine._ptr(qrecs), 2, m_q, L, C, engine._ptr(idx.lut_dev),
                     engine._ptr(scores), None, engine._stream())
    got = scores.cpu().numpy()
    S = c_oracle.score(codes, off, q, idx.lookup.table)
    np.testing.assert_array_equal(got[0, :40], S[0, cand[0, :40]])
    assert np.all(got[0, 40:] == 7.0) and np.all(got[1, 10:] == 7.0)
    assert np.isnan(got[1, 3])
    ok = [j for j in range(10) if j != 3]
    np.testing.assert_array_equal(got[1, ok], S[1, cand[1, ok]])


@pytest.mark.parametrize("n,k", [(9000, 4097), (30_000, 5000), (70_000, 20_000), (3000, 6000)])
def test_topk_large_k_ties_and_order(n, k):
    rng = np.random.default_rng(n + k)
    rows = 3
    vals = np.sort(rng.random(23))
    S = vals[rng.integers(0, 23, size=(rows, n))]
    S[0] = 0.5  # all equal: order by id alone
    ids = rng.permutation(4 * n)[:n].astype(np.int64)
    out_s, out_i, out_p = engine.topk(torch.from_numpy(S).to(DEV), k,
                                      ids=torch.from_numpy(ids).to(DEV))
    for r in range(rows):
        want = O.rank_topk(S[r], ids, k)
        kk = len(want)
        assert list(out_i[r, :kk].cpu().numpy()) == [w[0] for w in want]
        assert list(out_s[r, :kk].cpu().numpy()) == [w[1] for w in want]
        assert np.all(ids[out_p[r, :kk].cpu().numpy()] == out_i[r, :kk].cpu().numpy())
        assert np.all(out_s[r, kk:].cpu().numpy() == -1.0)


def test_topk_padding_sorts_last():
    """-1.0 padding (short chunk rows) ranks below every real score (order-preserving keys)."""
    S = np.array([[-1.0, 0.0, 0.25, -1.0, 1.0], [-1.0, -1.0, -1.0, -1.0, 0.0]])
    ids = np.array([0, 1, 2, 3, 4], dtype=np.int64)
    out_s, out_i, _ = engine.topk(torch.from_numpy(S).to(DEV), 3, ids=torch.from_numpy(ids).to(DEV))
    assert out_s.cpu().numpy().tolist() == [[1.0, 0.25, 0.0], [0.0, -1.0, -1.0]]
    assert out_i.cpu().numpy()[0].tolist() == [4, 2, 1]


def test_large_top_k_through_query_api(monkeypatch):
    L, C, m_q = 16, 3, 5
    sizes, off, codes, q, ids = _case(31, 6000, L, C, 2, m_q, lo=1, hi=6)
    idx = _index(codes, sizes, L, C, ids)
    for k in (4097, 5000, 6010):
        want, _ = _want(codes, off, q, idx.lookup.table, ids, k)
        assert d.query_codes_batch(idx, q, k) == want


def test_two_shards_merge_equals_single_index():
    """shard_bounds -> query each shard -> merge_topk_device == one index (ties included)."""
    L, C, m_q, k = 32, 4, 24, 40  # C = 4: many exact score ties
    sizes, off, codes, q, ids = _case(17, 9000, L, C, 12, m_q)
    full = _index(codes, sizes, L, C, ids)
    want = d.query_codes_batch(full, q, k, return_tensors=True)
    parts_s, parts_i = [], []
    for s0, s1 in shard_bounds(sizes, 2):
        sh = _index(codes[off[s0]:off[s1]], sizes[s0:s1], L, C, ids[s0:s1])
        a, b = d.query_codes_batch(sh, q, k, return_tensors=True)
        parts_s.append(a)
        parts_i.append(b)
    ms, mi = merge_topk_device(torch.cat(parts_s, 1), torch.cat(parts_i, 1), k)
    assert torch.equal(ms, want[0]) and torch.equal(mi, want[1])
    want_o, _ = _want(codes, off, q, full.lookup.table, ids, k)
    assert _rows(ms, mi) == want_o


def test_sharded_query_batch_nccl_one_rank():
    """The product multi-GPU function end to end on the GPU: a 1-rank NCCL process
    group (the only one a single GPU allows), sharded_query_batch = local query_batch
    + NCCL all-gather + K4 merge, equals query_batch on the same index."""
    import socket

    import torch.distributed as dist

    from paper_2210_15748_b200.distributed import sharded_query_batch

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    rng = np.random.default_rng(3)
    sizes = rng.integers(4, 60, size=3000)
    X = rng.standard_normal((int(sizes.sum()), 32)).astype(np.float32)
    off = np.concatenate([[0], np.cumsum(sizes)])
    docs = [(int(i) * 7, X[off[i]:off[i + 1]]) for i in range(len(sizes))]
    idx = d.build_index(docs, d.IndexConfig(d=32, C=6, L=32, seed=1, filter=d.FilterConfig(enabled=False)))
    Q = torch.from_numpy(rng.standard_normal((9, 16, 32)).astype(np.float32)).cuda()
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1,
                            device_id=torch.device("cuda", 0))
    try:
        ms, mi = sharded_query_batch(idx, Q, 25)
        ws, wi = d.query_batch(idx, Q, 25, return_tensors=True)
        assert torch.equal(ms, ws) and torch.equal(mi, wi)
    finally:
        dist.destroy_process_group()


def test_add_sets_failure_leaves_index_unchanged():
    rng = np.random.default_rng(4)
    docs = [(i, rng.standard_normal((int(rng.integers(1, 20)), 8))) for i in range(40)]
    cfg = d.IndexConfig(d=8, C=4, L=16, seed=1, filter=d.FilterConfig(enabled=False))
    idx = d.build_index(docs[:30], cfg)
    Q = rng.standard_normal((2, 6, 8))
    before = d.query_batch(idx, Q, 12)
    n_rec = idx.records.shape[0]
    with pytest.raises(ValueError, match="set too large"):
        d.add_sets(idx, [(1000, rng.standard_normal((70_000, 8)))])
    assert idx.records.shape[0] == n_rec and idx.n_docs == 30
    assert d.query_batch(idx, Q, 12) == before
    d.add_sets(idx, docs[30:])
    assert d.query_batch(idx, Q, 12) == d.query_batch(d.build_index(docs, cfg), Q, 12)


def test_graph_replays_concurrent_streams_tensors():
    """query_batch(return_tensors=True) through the cached graph from two streams:
    every returned tensor equals the eager result for its own input."""
    rng = np.random.default_rng(6)
    docs = [(i, rng.standard_normal((int(rng.integers(1, 20)), 16))) for i in range(400)]
    cfg = d.IndexConfig(d=16, C=5, L=32, seed=1, filter=d.FilterConfig(enabled=False))
    idx = d.build_index(docs, cfg)
    Qs = [torch.from_numpy(rng.standard_normal((3, 10, 16))).to(DEV) for _ in range(6)]
    want = [d.query_batch(idx, Q.cpu().numpy(), 9) for Q in Qs]
    streams = [torch.cuda.Stream(), torch.cuda.Stream()]
    outs = []
    for j, Q in enumerate(Qs):
        with torch.cuda.stream(streams[j % 2]):
            outs.append(d.query_batch(idx, Q, 9, return_tensors=True))
    torch.cuda.synchronize()
    for (s, i), w in zip(outs, want):
        assert I._results(s, i) == w


def test_copy_async_and_pack4_through_pinned_host_buffers():
    """The graph query path's staging calls: dsrt_copy_async (pinned host <-> device) and
    dsrt_pack4_async (up to four small device tensors -> one device or pinned host buffer)."""
    dev = torch.device("cuda")
    src = torch.arange(1000, dtype=torch.float64).reshape(10, 100).pin_memory()
    on_dev = torch.empty(10, 100, dtype=torch.float64, device=dev)
    back = torch.empty(10, 100, dtype=torch.float64).pin_memory()
    engine.copy_async(on_dev, src)
    engine.copy_async(back, on_dev)
    torch.cuda.synchronize()
    assert torch.equal(back, src)
    with pytest.raises(ValueError, match="page-locked"):
        engine.copy_async(on_dev, torch.zeros(10, 100, dtype=torch.float64))
    a = torch.rand(3, 7, dtype=torch.float64, device=dev)
    b = torch.randint(0, 1 << 60, (3, 7), dtype=torch.int64, device=dev)
    c = torch.tensor([5], dtype=torch.int32, device=dev)
    for tensors in ([a, b, c, None], [a, None, c, b], [c], [a, b, c, c]):
        offs, total = engine.pack_layout(tensors)
        for dst in (torch.zeros(total, dtype=torch.uint8, device=dev),
                    torch.zeros(total, dtype=torch.uint8).pin_memory()):
            engine.pack4(dst, tensors)
            torch.cuda.synchronize()
            raw = dst.cpu().numpy()
            for t, off in zip(tensors, offs):
                if t is None:
                    continue
                n = t.numel() * t.element_size()
                assert off % 16 == 0
                got = torch.from_numpy(raw[off:off + n].copy()).view(t.dtype).reshape(t.shape)
                assert torch.equal(got, t.cpu())


def test_query_from_host_arrays_matches_device_tensors_and_eager_path(monkeypatch):
    """query()/query_batch() with host inputs replay a graph whose first node uploads the
    query and whose last node packs the results into pinned memory; device-tensor inputs
    and the eager path (DSRT_QUERY_GRAPHS=0) must give the same rankings."""
    rng = np.random.default_rng(5)
    sizes = rng.integers(3, 30, size=300)
    X = rng.standard_normal((int(sizes.sum()), 32)).astype(np.float32)
    off = np.concatenate([[0], np.cumsum(sizes)])
    docs = [(i, X[off[i]:off[i + 1]]) for i in range(len(sizes))]
    for enabled in (False, True):
        cfg = d.IndexConfig(d=32, C=5, L=32, seed=1,
                            filter=d.FilterConfig(enabled=enabled, centroids=16, iters=3, probe=2, k_filter=40))
        idx = d.build_index(docs, cfg)
        Qs = np.stack([X[off[i]:off[i] + 3] for i in (7, 100, 250)])
        host = [d.query(idx, Q, 20) for Q in Qs]
        again = [d.query(idx, Q, 20) for Q in Qs]       # second replay of the same graph
        dev_in = [d.query(idx, torch.from_numpy(Q).cuda(), 20) for Q in Qs]
        batch = d.query_batch(idx, Qs, 20)
        monkeypatch.setenv("DSRT_QUERY_GRAPHS", "0")
        eager = [d.query(idx, Q, 20) for Q in Qs]
        monkeypatch.delenv("DSRT_QUERY_GRAPHS")
        assert host == again == dev_in == batch == eager
        assert all(1 <= len(r) <= 20 for r in host)
