"""Parity at BASELINE.json sizes (GPU).

* cfg1 at full size: all 100,000 sets x 8 query sets, bit-exact vs the C oracle
  (scores and top-100), top-k invariants for all 1,000 query sets, and 4,096
  sampled (query set, set) pairs across all 1,000.
* cfg3 pipeline at full size (1M sets, 65,536 centroids): prefilter candidates
  (oracle filter_candidates over the device postings), candidate scores and
  top-100 for 16 query sets (>= 16).
* cfg4 shape (L=32, C=8 codes from records): 2 query sets x 300k sets exact,
  and sampled (query set, set) pairs for 1,024 query sets.
* cfg4 at full size: one query set over all 8,000,000 sets (~560M vectors) exact
  vs the C oracle, streamed in 500k-set chunks, and its top-1,000.
"""

import numpy as np
import pytest
import torch

import paper_2210_15748_b200 as d
from oracle import c_oracle
from oracle import dessert_oracle as O
from paper_2210_15748_b200 import engine, prefilter, workloads

pytestmark = pytest.mark.gpu
DEV = torch.device("cuda")


def _records_to_codes_dev(recs: torch.Tensor, L: int, C: int) -> torch.Tensor:
    """Inverse of the plane-record layout on the device (test helper), int32 (n, L)."""
    W = (L + 31) // 32
    r = recs.to(torch.int64) & 0xFFFFFFFF
    t = torch.arange(L, device=recs.device)
    codes = torch.zeros((recs.shape[0], L), dtype=torch.int64, device=recs.device)
    for b in range(C):
        words = r[:, b * W + t // 32]
        codes |= ((words >> (t % 32)) & 1) << b
    return codes.to(torch.int32)


def test_cfg1_full_size_parity():
    n_sets, L, C = 100_000, 64, 7
    sizes = workloads.set_sizes(n_sets, 70, 20, seed=100)
    off = workloads.offsets(sizes)
    X, _ = workloads.gpu_mixture(int(off[-1]), 4096, 128, 0.05, seed=200, dtype=torch.float16,
                                 device=DEV)
    cfg = d.IndexConfig(d=128, C=C, L=L, seed=0, filter=d.FilterConfig(enabled=False))
    idx = d.build_from_vectors(X, sizes, np.arange(n_sets), cfg)
    Qv = workloads.gpu_queries(X, off, 1000, 32, seed=300)
    del X
    scores_t, ids_t = d.query_batch(idx, Qv, 100, return_tensors=True)
    # oracle on 8 query sets over all sets, with the device's own codes
    qc, _ = d.lsh.hash_device(idx.family, Qv[:8].reshape(-1, 128).contiguous(), want_records=False)
    qcodes = qc.cpu().numpy().astype(np.int64).reshape(8, 32, L)
    codes = idx.codes.cpu().numpy()
    want = c_oracle.score(codes, off, qcodes, idx.lookup.table)
    got, _ = d.score_matrix(idx, qcodes)
    np.testing.assert_array_equal(got.cpu().numpy(), want)
    S = scores_t.cpu().numpy()
    I = ids_t.cpu().numpy()
    for r in range(8):
        top = O.rank_topk(want[r], np.arange(n_sets), 100)
        assert [x for x, _ in top] == list(I[r]) and [v for _, v in top] == list(S[r])
    # invariants for all 1000 rows: sorted by (score desc, id asc), unique ids
    assert np.all((S[:, :-1] > S[:, 1:]) | ((S[:, :-1] == S[:, 1:]) & (I[:, :-1] < I[:, 1:])))
    assert all(len(set(row)) == 100 for row in I)
    # 4096 random (query set, set) pairs across all 1000 query sets vs the oracle
    qa, _ = d.lsh.hash_device(idx.family, Qv.reshape(-1, 128).contiguous(), want_records=False)
    qall = qa.cpu().numpy().astype(np.int64).reshape(1000, 32, L)
    full, _ = d.score_matrix(idx, qall)
    rng = np.random.default_rng(17)
    qs = rng.integers(0, 1000, size=4096)
    ss = rng.integers(0, n_sets, size=4096)
    g = full[torch.from_numpy(qs).to(DEV), torch.from_numpy(ss).to(DEV)].cpu().numpy()
    w = c_oracle.score(codes, off, qall[qs], idx.lookup.table, sets=ss[:, None])[:, 0]
    np.testing.assert_array_equal(g, w)


def test_cfg3_pipeline_full_size_parity():
    n_sets, L, C, n_cent, probe, k_filter = 1_000_000, 32, 7, 65536, 4, 4096
    sizes = workloads.set_sizes(n_sets, 70, 20, seed=500)
    off = workloads.offsets(sizes)
    X, cents = workloads.gpu_mixture(int(off[-1]), n_cent, 128, 0.05, seed=501,
                                     dtype=torch.float16, device=DEV)
    cfg = d.IndexConfig(d=128, C=C, L=L, seed=0,
                        filter=d.FilterConfig(enabled=True, centroids=n_cent, probe=probe,
                                              k_filter=k_filter))
    idx = d.build_from_vectors(X, sizes, np.arange(n_sets), cfg)
    cvec = cents.double()
    cvec = cvec / cvec.norm(dim=1, keepdim=True)
    centroids = prefilter.Centroids(k=n_cent, seed=0, vectors=cvec.cpu().numpy())
    cindex = prefilter.build_centroid_index(X, centroids, set_off=idx.set_off, n_docs=n_sets)
    idx.filter = (centroids, cindex)
    n_chk = 16
    Qv = workloads.gpu_queries(X, off, n_chk, 32, seed=502)
    # spot-check the native postings: argmax of a vector sample, float64
    samp = torch.arange(0, X.shape[0], 997, device=DEV)
    Xs = X[samp].double()
    am = torch.argmax(Xs @ cvec.T, dim=1).cpu().numpy()
    po = cindex.post_off.cpu().numpy()
    pdocs = cindex.post_docs.cpu().numpy()
    doc_of = np.searchsorted(off, samp.cpu().numpy(), side="right") - 1
    for c, doc in zip(am[:2000], doc_of[:2000]):
        seg = pdocs[po[c]:po[c + 1]]
        assert doc in seg
    del X
    postings = [pdocs[po[c]:po[c + 1]] for c in range(n_cent)]
    res = d.query_batch(idx, Qv, 100)
    qc, _ = d.lsh.hash_device(idx.family, Qv.reshape(-1, 128).contiguous(), want_records=False)
    qcodes = qc.cpu().numpy().astype(np.int64).reshape(n_chk, 32, L)
    records = idx.records.cpu().numpy()
    lut = idx.lookup.table
    for r in range(n_chk):
        Qr = Qv[r].double().cpu().numpy()
        cand = O.filter_candidates(postings, n_sets, centroids.vectors, Qr, probe, k_filter)
        got_c, n_c = prefilter.filter_candidates_device(cindex, centroids, Qv[r].double(), 32,
                                                        probe, k_filter)
        np.testing.assert_array_equal(got_c[0, : int(n_c[0])].cpu().numpy(), cand)
        vec_rows = np.concatenate([np.arange(off[s], off[s + 1]) for s in cand])
        codes = workloads.records_to_codes(records[vec_rows], L, C)
        sub_sizes = sizes[cand]
        scores = c_oracle.score(codes, workloads.offsets(sub_sizes), qcodes[r:r + 1], lut)[0]
        want = O.rank_topk(scores, cand, 100)
        assert res[r] == want


def test_cfg4_shape_sampled_parity():
    n_sets, L, C = 300_000, 32, 8
    sizes = workloads.set_sizes(n_sets, 70, 25, seed=400)
    cfg = d.IndexConfig(d=128, C=C, L=L, seed=0, filter=d.FilterConfig(enabled=False))
    recs, Qv = workloads.gpu_codes_only(sizes, cfg, n_centroids=262_144, n_qsets=1024, m_q=32,
                                        seed=401, device=DEV)
    idx = d.build_from_records(recs, sizes, np.arange(n_sets), cfg)
    qc, qrecs = d.lsh.hash_device(idx.family, Qv.reshape(-1, 128).contiguous())
    qcodes = qc.cpu().numpy().astype(np.int64).reshape(1024, 32, L)
    off = workloads.offsets(sizes)
    codes = _records_to_codes_dev(recs, L, C).cpu().numpy()      # int32, converted once
    lut = idx.lookup.table
    # 2 query sets exhaustively
    got, _ = engine.score_all(idx.records, idx.set_off, qrecs, 32, L, C, idx.lut_dev)
    want2 = c_oracle.score(codes, off, qcodes[:2], lut)
    np.testing.assert_array_equal(got[:2].cpu().numpy(), want2)
    # 4096 random (query set, set) pairs across all 1024 query sets
    rng = np.random.default_rng(9)
    qs = rng.integers(0, 1024, size=4096)
    ss = rng.integers(0, n_sets, size=4096)
    g = got.cpu().numpy()
    w = c_oracle.score(codes, off, qcodes[qs], lut, sets=ss[:, None])[:, 0]   # one batched call
    np.testing.assert_array_equal(g[qs, ss], w)
    # top-1000 for 2 query sets
    out_s, out_i, _ = engine.topk(got, 1000, ids=idx.doc_ids_dev)
    for r in range(2):
        top = O.rank_topk(want2[r], np.arange(n_sets), 1000)
        assert [x for x, _ in top] == list(out_i[r].cpu().numpy())


def test_cfg4_full_size_one_query_set():
    """cfg4 at BASELINE size: query set 0 scored over all 8M sets by the device
    (exhaustive K3) vs the C oracle on the codes read back from the records, in
    500k-set chunks (the full int32 code matrix would be 72 GB on the host); then
    the device top-1,000 vs the oracle ranking (score desc, id asc)."""
    n_sets, L, C, top_k = 8_000_000, 32, 8, 1000
    sizes = workloads.set_sizes(n_sets, 70, 25, seed=400)
    cfg = d.IndexConfig(d=128, C=C, L=L, seed=0, filter=d.FilterConfig(enabled=False))
    recs, Qv = workloads.gpu_codes_only(sizes, cfg, n_centroids=262_144, n_qsets=2, m_q=32,
                                        seed=401, device=DEV)
    idx = d.build_from_records(recs, sizes, np.arange(n_sets), cfg)
    qc, qrecs = d.lsh.hash_device(idx.family, Qv[:1].reshape(-1, 128).contiguous())
    qcodes = qc.cpu().numpy().astype(np.int64).reshape(1, 32, L)
    off = workloads.offsets(sizes)
    got, _ = engine.score_all(idx.records, idx.set_off, qrecs, 32, L, C, idx.lut_dev)
    got = got[0].cpu().numpy()
    lut = idx.lookup.table
    step = 500_000
    want = np.empty(n_sets, dtype=np.float64)
    for s0 in range(0, n_sets, step):
        s1 = min(n_sets, s0 + step)
        v0, v1 = int(off[s0]), int(off[s1])
        codes = _records_to_codes_dev(recs[v0:v1], L, C).cpu().numpy()
        want[s0:s1] = c_oracle.score(codes, off[s0:s1 + 1] - v0, qcodes, lut)[0]
        del codes
    np.testing.assert_array_equal(got, want)
    order = np.lexsort((np.arange(n_sets), -want))[:top_k]
    out_s, out_i = d.query_codes_batch(idx, qcodes, top_k, return_tensors=True)
    np.testing.assert_array_equal(out_i[0].cpu().numpy().astype(np.int64), order)
    np.testing.assert_array_equal(out_s[0].cpu().numpy(), want[order])


def _hash_flips_vs_f64(planes: np.ndarray, Xs: torch.Tensor, codes: torch.Tensor, L: int, C: int):
    """Bit flips of device codes vs the float64 projection X @ planes.T > 0 (lsh.py:103),
    and how many of them lie outside |w.x| < 1e-4 |w||x|.  float64 GEMM on the device
    as the checker, 250k rows at a time."""
    P = torch.from_numpy(planes).to(Xs.device)
    wn = P.norm(dim=1)
    flips = outside = 0
    for lo in range(0, Xs.shape[0], 250_000):
        x = Xs[lo:lo + 250_000].double()
        proj = x @ P.T
        want = (proj > 0).reshape(-1, L, C)
        c = codes[lo:lo + 250_000].to(torch.int64)
        got = ((c[:, :, None] >> torch.arange(C, device=c.device)) & 1).bool()
        f = (got != want).reshape(x.shape[0], L * C)
        band = proj.abs() < 1e-4 * wn[None, :] * x.norm(dim=1)[:, None]
        flips += int(f.sum())
        outside += int((f & ~band).sum())
    return flips, outside


@pytest.mark.parametrize("mode", ["default", "fix"])
def test_cfg2_full_size_hash_band(mode):
    """cfg2: 10M bf16 mixture vectors (4,096 centroids, noise 0.05), L=64 C=7: the
    device codes of 1M sampled rows flip no bit outside the 1e-4 band vs float64
    (SURVEY 8(c)); the flip rate is printed (the north star asks for it reported)."""
    from paper_2210_15748_b200 import _lib

    n, L, C = 10_000_000, 64, 7
    X, _ = workloads.gpu_mixture(n, 4096, 128, 0.05, seed=601, dtype=torch.bfloat16, device=DEV)
    fam = d.sample_srp_family(128, C, L, 0)
    m = None if mode == "default" else _lib.HASH_TC_FIX
    codes, _ = d.lsh.hash_device(fam, X, mode=m, want_records=False)
    g = torch.Generator(device=DEV)
    g.manual_seed(7)
    samp = torch.randperm(n, generator=g, device=DEV)[:1_000_000]
    flips, outside = _hash_flips_vs_f64(fam.planes, X[samp], codes[samp], L, C)
    print(f"cfg2 hash ({mode}): {flips} flips in {1_000_000 * L * C} bits, {outside} outside the band")
    assert outside == 0


def test_cfg3_postings_exact_10m():
    """K6 at cfg3's centroid count: 10M fp16 vectors from the 65,536-centroid mixture in
    ~143k sets; every (document, centroid) posting pair equals the float64 argmax
    assignment of all 10M vectors (prefilter.py:85-108), computed by a device float64
    GEMM as the checker."""
    n_cent = 65536
    sizes = workloads.set_sizes(143_000, 70, 20, seed=510)
    off = workloads.offsets(sizes)
    n = int(off[-1])
    X, cents = workloads.gpu_mixture(n, n_cent, 128, 0.05, seed=511, dtype=torch.float16, device=DEV)
    cvec = cents.double()
    cvec = cvec / cvec.norm(dim=1, keepdim=True)
    centroids = prefilter.Centroids(k=n_cent, seed=0, vectors=cvec.cpu().numpy())
    off_dev = torch.from_numpy(off).to(DEV)
    cindex = prefilter.build_centroid_index(X, centroids, set_off=off_dev, n_docs=len(sizes))
    # checker: float64 argmax of every vector (first index on ties, like np.argmax)
    am = torch.empty(n, dtype=torch.int64, device=DEV)
    CT = cvec.T.contiguous()
    for lo in range(0, n, 131072):
        s = X[lo:lo + 131072].double() @ CT
        am[lo:lo + 131072] = torch.argmax(s, dim=1)
    doc = torch.repeat_interleave(torch.arange(len(sizes), device=DEV),
                                  torch.from_numpy(sizes).to(DEV))
    want = torch.unique(am * len(sizes) + doc)  # (centroid, doc) pairs, deduplicated, sorted
    po = cindex.post_off
    cnt = (po[1:] - po[:-1]).to(torch.int64)
    cid = torch.repeat_interleave(torch.arange(n_cent, device=DEV), cnt)
    got = cid * len(sizes) + cindex.post_docs.to(torch.int64)
    assert got.shape == want.shape, (got.shape, want.shape)
    assert torch.equal(got, want)  # also checks each posting is ascending and duplicate-free
