"""CUDA path vs the oracle / reference golden vectors (bit-exact).  Needs a B200."""

import numpy as np
import pytest
import torch

import paper_2210_15748_b200 as d
from conftest import small_case
from oracle import c_oracle
from oracle import dessert_oracle as O
from paper_2210_15748_b200 import _lib, engine

pytestmark = pytest.mark.gpu
DEV = "cuda"


def _index_from_codes(codes, sizes, L, C, doc_ids=None):
    cfg = d.IndexConfig(d=4, C=C, L=L, filter=d.FilterConfig(enabled=False))
    cd = torch.from_numpy(np.ascontiguousarray(codes).astype(np.int32)).to(DEV)
    ids = np.arange(len(sizes)) if doc_ids is None else doc_ids
    return d.build_from_codes(cd, sizes, ids, cfg)


# ------------------------------------------------------------------ scoring
def test_small_shapes_scores_and_counts_bit_exact(golden_small):
    g = golden_small
    for n in range(int(g["n_shapes"])):
        c = small_case(g, n)
        idx = _index_from_codes(c["codes"], c["sizes"], c["L"], c["C"], c["doc_ids"])
        # all three scoring entry points: exhaustive (n_q<8 -> candidate kernel), explicit sets
        s, mc = d.score_matrix(idx, c["qcodes"], want_counts=True)
        np.testing.assert_array_equal(s.cpu().numpy(), c["scores"], err_msg=f"shape {n}")
        np.testing.assert_array_equal(mc.cpu().numpy().astype(np.int32), c["maxcounts"])
        # replicate query sets to >= 8 so the shared-tile exhaustive kernel runs
        qrep = np.concatenate([c["qcodes"]] * 3)
        s8, mc8 = d.score_matrix(idx, qrep, want_counts=True)
        np.testing.assert_array_equal(s8.cpu().numpy(), np.concatenate([c["scores"]] * 3))
        np.testing.assert_array_equal(mc8.cpu().numpy().astype(np.int32),
                                      np.concatenate([c["maxcounts"]] * 3))
        sets = np.stack([np.random.default_rng(n).permutation(len(c["sizes"]))] * 3)
        sc, _ = d.score_matrix(idx, c["qcodes"], sets=sets)
        np.testing.assert_array_equal(sc.cpu().numpy(),
                                      np.take_along_axis(c["scores"], sets, axis=1))
        for q in range(3):
            i = int(sets[0, q])
            assert d.score_candidate(idx, i, c["qcodes"][q]) == c["scores"][q, i]


def test_cfg0_scores_counts_topk_bit_exact(golden_cfg0):
    g = golden_cfg0
    idx = _index_from_codes(g["codes"], g["sizes"], 32, 6)
    s, mc = d.score_matrix(idx, g["qcodes"], want_counts=True)
    np.testing.assert_array_equal(s.cpu().numpy(), g["scores"])
    np.testing.assert_array_equal(mc.cpu().numpy().astype(np.uint8), g["maxcounts"])
    res = d.query_codes_batch(idx, g["qcodes"], 10)
    for q, r in enumerate(res):
        assert [x for x, _ in r] == list(g["top_ids"][q])
        assert [v for _, v in r] == list(g["top_scores"][q])


def test_cfg0_end_to_end_from_vectors(golden_cfg0):
    """Full path: vectors -> K1 hash -> K2 layout -> K3 -> K4 vs the reference's query()."""
    from paper_2210_15748_b200 import workloads
    g = golden_cfg0
    sizes, X, Q = workloads.cfg0_data(0)
    off = workloads.offsets(sizes)
    cfg = d.IndexConfig(d=128, C=6, L=32, seed=0, filter=d.FilterConfig(enabled=False))
    idx = d.build_from_vectors(torch.from_numpy(X).to(DEV), sizes, np.arange(len(sizes)), cfg)
    codes = idx.codes.cpu().numpy()
    mism = int((codes != g["codes"]).sum())
    assert mism == 0, f"{mism} hash codes differ from the reference"
    for q in range(len(Q)):
        r = d.query(idx, Q[q], top_k=10)
        assert [x for x, _ in r] == list(g["top_ids"][q])
        assert [v for _, v in r] == list(g["top_scores"][q])
    out_s, out_i = d.query_batch(idx, Q, 10, return_tensors=True)
    np.testing.assert_array_equal(out_i.cpu().numpy(), g["top_ids"])
    np.testing.assert_array_equal(out_s.cpu().numpy(), g["top_scores"])
    del off


# ------------------------------------------------------------------ hashing
def test_hash_golden_f64(golden_lsh):
    g = golden_lsh
    fam = d.sample_srp_family(128, 6, 32, 0)
    got = d.hash_matrix(fam, g["X"])
    np.testing.assert_array_equal(got, g["codes"])
    with pytest.raises(ValueError, match="zero vector"):
        d.hash_matrix(fam, np.zeros((2, 128)))
    with pytest.raises(ValueError, match="dimension"):
        d.hash_matrix(fam, np.ones((2, 5)))


@pytest.mark.parametrize("mode", [_lib.HASH_F64, _lib.HASH_F32])
@pytest.mark.parametrize("dtype", [torch.float32, torch.float16, torch.bfloat16, torch.float64])
def test_hash_modes_flip_only_in_band(mode, dtype):
    rng = np.random.default_rng(11)
    X = rng.standard_normal((4096, 128))
    X /= np.linalg.norm(X, axis=1, keepdims=True)
    Xt = torch.from_numpy(X).to(dtype)
    Xexact = Xt.to(torch.float64).numpy()          # the values the device sees
    fam = d.sample_srp_family(128, 7, 64, 3)
    codes, recs = d.lsh.hash_device(fam, Xt.to(DEV).contiguous(), mode=mode)
    want = O.hash_matrix(fam.planes, 64, 7, Xexact)
    got = codes.cpu().numpy().astype(np.int64)
    proj = O.projections(fam.planes, Xexact)
    band = np.abs(proj) < 1e-4 * np.linalg.norm(fam.planes, axis=1)[None, :] * \
        np.linalg.norm(Xexact, axis=1)[:, None]
    bits_got = ((got[:, :, None] >> np.arange(7)) & 1).reshape(4096, 448)
    bits_want = ((want[:, :, None] >> np.arange(7)) & 1).reshape(4096, 448)
    flips = bits_got != bits_want
    assert not np.any(flips & ~band), f"{int((flips & ~band).sum())} flips outside the band"
    if mode == _lib.HASH_F64:
        assert int(flips.sum()) == 0
    # records agree with codes
    recs2, _ = engine.codes_to_records(codes, 64, 7)
    assert torch.equal(recs, recs2)


TC_CASES = [(torch.float16, _lib.HASH_TC_F16X2), (torch.float16, _lib.HASH_TC_FIX),
            (torch.bfloat16, _lib.HASH_TC_FIX), (torch.bfloat16, _lib.HASH_TC_BF16X2)]


@pytest.mark.parametrize("dtype,mode", TC_CASES)
@pytest.mark.parametrize("L,C", [(64, 7), (32, 8), (40, 5), (32, 7), (16, 3)])
def test_hash_tensor_core_flip_only_in_band(dtype, mode, L, C):
    """tcgen05 hash (TMA + UMMA + TMEM + fused sign/pack) vs the float64 oracle:
    codes and plane records agree except inside |w.x| < 1e-4 |w||x|; counts reported."""
    rng = np.random.default_rng(L * 10 + C)
    n = 5000  # not a multiple of 128: exercises the ragged last tile
    X = rng.standard_normal((n, 128))
    X /= np.linalg.norm(X, axis=1, keepdims=True)
    Xt = torch.from_numpy(X).to(dtype)
    Xexact = Xt.to(torch.float64).numpy()
    fam = d.sample_srp_family(128, C, L, 5)
    codes, recs = d.lsh.hash_device(fam, Xt.to(DEV).contiguous(), mode=mode)
    want = O.hash_matrix(fam.planes, L, C, Xexact)
    got = codes.cpu().numpy().astype(np.int64)
    proj = O.projections(fam.planes, Xexact)
    band = np.abs(proj) < 1e-4 * np.linalg.norm(fam.planes, axis=1)[None, :] * \
        np.linalg.norm(Xexact, axis=1)[:, None]
    bits_got = ((got[:, :, None] >> np.arange(C)) & 1).reshape(n, L * C)
    bits_want = ((want[:, :, None] >> np.arange(C)) & 1).reshape(n, L * C)
    flips = bits_got != bits_want
    outside = int((flips & ~band).sum())
    assert outside == 0, f"{outside} flips outside the band ({int(flips.sum())} total)"
    recs2, _ = engine.codes_to_records(codes, L, C)
    assert torch.equal(recs, recs2)
    # zero rows are detected
    Xz = Xt.clone()
    Xz[17] = 0
    with pytest.raises(ValueError, match="zero vector"):
        d.lsh.hash_device(fam, Xz.to(DEV).contiguous(), mode=mode)


def _band_check(fam, X64, got, L, C):
    """flips of GPU codes vs the float64 oracle, and whether each lies in the 1e-4 band"""
    n = X64.shape[0]
    want = O.hash_matrix(fam.planes, L, C, X64)
    proj = O.projections(fam.planes, X64)
    band = np.abs(proj) < 1e-4 * np.linalg.norm(fam.planes, axis=1)[None, :] * \
        np.linalg.norm(X64, axis=1)[:, None]
    bg = ((got[:, :, None] >> np.arange(C)) & 1).reshape(n, L * C)
    bw = ((want[:, :, None] >> np.arange(C)) & 1).reshape(n, L * C)
    return bg != bw, band


@pytest.mark.parametrize("dtype", [torch.float16, torch.bfloat16])
def test_hash_fix_mode_near_zero_projections(dtype):
    """TC_FIX on vectors built to sit almost on planes (|w.x| ~ 1e-6..1e-2 |w||x| for
    chosen (row, plane) pairs): thousands of bits go through the fix-up, none may
    differ from the float64 reference outside the 1e-4 band."""
    rng = np.random.default_rng(77)
    L, C, n = 64, 7, 6000
    fam = d.sample_srp_family(128, C, L, 9)
    W = fam.planes
    X = rng.standard_normal((n, 128))
    p = rng.integers(0, L * C, size=n)
    for k in range(3):  # project three planes each (almost) out of every row
        p = (p + 37 * k) % (L * C)
        w = W[p]
        X -= ((X * w).sum(1) / (w * w).sum(1))[:, None] * w
        X += (10.0 ** rng.uniform(-6, -2, size=n))[:, None] * w / np.linalg.norm(w, axis=1)[:, None]
    X /= np.linalg.norm(X, axis=1, keepdims=True)
    Xt = torch.from_numpy(X).to(dtype)
    X64 = Xt.to(torch.float64).numpy()
    codes, recs = d.lsh.hash_device(fam, Xt.to(DEV).contiguous(), mode=_lib.HASH_TC_FIX)
    got = codes.cpu().numpy().astype(np.int64)
    flips, band = _band_check(fam, X64, got, L, C)
    assert int((flips & ~band).sum()) == 0
    proj = O.projections(W, X64) / np.linalg.norm(W, axis=1)[None, :]
    assert int((np.abs(proj) < 1e-2).sum()) > 3 * n  # the fix-up path really ran
    recs2, _ = engine.codes_to_records(codes, L, C)
    assert torch.equal(recs, recs2)


def test_hash_fix_mode_bf16_extreme_magnitudes():
    """bf16 rows spanning 1e-30 .. 1e30 in scale (and rows with subnormal-range
    elements) are scaled per row before the fp16 rounding: same bits as the float64
    reference outside the band; codes equal the fp16-input result for rows that are
    exact in both types."""
    rng = np.random.default_rng(5)
    L, C, n = 32, 8, 4500
    fam = d.sample_srp_family(128, C, L, 2)
    X = rng.standard_normal((n, 128))
    X /= np.linalg.norm(X, axis=1, keepdims=True)
    X *= (10.0 ** rng.uniform(-30, 30, size=n))[:, None]
    X[::7, ::3] *= 1e-6  # elements far below the row maximum (fp16 subnormal range)
    Xt = torch.from_numpy(X).to(torch.bfloat16)
    X64 = Xt.to(torch.float64).numpy()
    codes, _ = d.lsh.hash_device(fam, Xt.to(DEV).contiguous(), mode=_lib.HASH_TC_FIX)
    flips, band = _band_check(fam, X64, codes.cpu().numpy().astype(np.int64), L, C)
    assert int((flips & ~band).sum()) == 0


def test_hash_fix_mode_ragged_and_unsupported():
    rng = np.random.default_rng(1)
    fam = d.sample_srp_family(128, 5, 40, 4)
    X = rng.standard_normal((4099, 128)).astype(np.float16)
    codes, _ = d.lsh.hash_device(fam, torch.from_numpy(X).to(DEV), mode=_lib.HASH_TC_FIX)
    flips, band = _band_check(fam, X.astype(np.float64), codes.cpu().numpy().astype(np.int64), 40, 5)
    assert int((flips & ~band).sum()) == 0
    with pytest.raises(ValueError, match="fp16 or bf16"):
        d.lsh.hash_device(fam, torch.from_numpy(X.astype(np.float32)).to(DEV), mode=_lib.HASH_TC_FIX)


# ------------------------------------------------------------------- layout
def test_layout_roundtrip_and_tinytable_export(golden_small):
    g = golden_small
    for n in range(int(g["n_shapes"])):
        c = small_case(g, n)
        idx = _index_from_codes(c["codes"], c["sizes"], c["L"], c["C"])
        np.testing.assert_array_equal(idx.set_off.cpu().numpy(), c["off"])
        for i in range(3):
            tt = idx.sketches[i]
            np.testing.assert_array_equal(tt.offsets, g[f"s{n}_tt{i}_offsets"])
            np.testing.assert_array_equal(tt.ids, g[f"s{n}_tt{i}_ids"])
            assert tt.offsets.dtype == g[f"s{n}_tt{i}_offsets"].dtype
        tt = d.build_tiny_table(c["codes"][: c["sizes"][0]], c["L"], 1 << c["C"])
        np.testing.assert_array_equal(tt.ids, g[f"s{n}_tt0_ids"])


def test_tinytable_known_answer():  # pkg/tests/test_sketch.py:37-40
    t = d.build_tiny_table(np.array([[2], [0], [2]]), L=1, r=4)
    np.testing.assert_array_equal(t.offsets[0], [0, 1, 1, 3, 3])
    np.testing.assert_array_equal(t.ids[0], [1, 0, 2])
    with pytest.raises(ValueError, match="out of range"):
        d.build_tiny_table(np.array([[4]]), L=1, r=4)


def test_counting_sort_stable():
    rng = np.random.default_rng(3)
    n_sets, n = 1000, 50000
    set_of = rng.integers(0, n_sets, size=n)
    so, perm = engine.counting_sort(torch.from_numpy(set_of).to(DEV), n_sets)
    want = np.argsort(set_of, kind="stable")
    np.testing.assert_array_equal(perm.cpu().numpy(), want)
    np.testing.assert_array_equal(so.cpu().numpy(),
                                  np.concatenate([[0], np.cumsum(np.bincount(set_of, minlength=n_sets))]))
    rows = torch.from_numpy(rng.integers(0, 1 << 30, size=(n, 4)).astype(np.int32)).to(DEV)
    got = engine.gather_rows(rows, perm)
    np.testing.assert_array_equal(got.cpu().numpy(), rows.cpu().numpy()[want])


def test_sizes_to_offsets_large_and_bad():
    rng = np.random.default_rng(4)
    sizes = rng.integers(1, 181, size=300_001).astype(np.int64)
    so, bad = engine.sizes_to_offsets(torch.from_numpy(sizes).to(DEV))
    np.testing.assert_array_equal(so.cpu().numpy(), np.concatenate([[0], np.cumsum(sizes)]))
    assert int(bad.item()) == 0
    sizes[7] = 0
    sizes[9] = 70000
    _, bad = engine.sizes_to_offsets(torch.from_numpy(sizes).to(DEV))
    assert int(bad.item()) == 2


# -------------------------------------------------------------------- top-k
@pytest.mark.parametrize("n,k", [(1, 1), (5, 10), (1000, 10), (100_000, 100), (40_000, 1000),
                                 (9000, 4096)])
def test_topk_ties_and_order(n, k):
    rng = np.random.default_rng(n + k)
    rows = 6
    # heavy ties: scores from a small value set, ids a random permutation
    vals = np.sort(rng.random(17))
    S = vals[rng.integers(0, 17, size=(rows, n))]
    S[0] = 0.25  # all equal
    ids = rng.permutation(10 * n)[:n].astype(np.int64)
    out_s, out_i, out_p = engine.topk(torch.from_numpy(S).to(DEV), k,
                                      ids=torch.from_numpy(ids).to(DEV))
    for r in range(rows):
        want = O.rank_topk(S[r], ids, k)
        kk = len(want)
        assert list(out_i[r, :kk].cpu().numpy()) == [w[0] for w in want]
        assert list(out_s[r, :kk].cpu().numpy()) == [w[1] for w in want]
        assert np.all(ids[out_p[r, :kk].cpu().numpy()] == out_i[r, :kk].cpu().numpy())


def test_topk_n_valid_and_per_row_ids():
    rng = np.random.default_rng(9)
    S = rng.random((4, 300))
    ids = rng.integers(0, 1 << 40, size=(4, 300)).astype(np.int64)
    nv = np.array([0, 1, 150, 300], dtype=np.int32)
    out_s, out_i, _ = engine.topk(torch.from_numpy(S).to(DEV), 20,
                                  ids=torch.from_numpy(ids).to(DEV),
                                  n_valid=torch.from_numpy(nv).to(DEV))
    for r in range(4):
        want = O.rank_topk(S[r, : nv[r]], ids[r, : nv[r]], 20)
        kk = len(want)
        assert list(out_i[r, :kk].cpu().numpy()) == [w[0] for w in want]
        assert np.all(out_s[r, kk:].cpu().numpy() == -1.0)


@pytest.mark.parametrize("n", [300, 5000])
def test_topk_indexed_matches_gathered_ids(n):
    """dsrt_topk_indexed (doc ids read through a candidate index in the kernel) equals the
    gathered-ids top-k and the oracle ranking; many score ties so the id tie-break decides."""
    rng = np.random.default_rng(19)
    rows, k = 6, 50
    S = np.round(rng.random((rows, n)), 2)                     # heavy ties
    doc_ids = rng.permutation(1 << 20)[:7000].astype(np.int64)
    cand = np.stack([rng.permutation(7000)[:n] for _ in range(rows)]).astype(np.int64)
    nv = np.array([0, 1, n // 2, n, n - 3, 7], dtype=np.int32)
    St, Ct = torch.from_numpy(S).to(DEV), torch.from_numpy(cand).to(DEV)
    Dt, Nt = torch.from_numpy(doc_ids).to(DEV), torch.from_numpy(nv).to(DEV)
    a_s, a_i, a_p = engine.topk(St, k, ids=Dt, n_valid=Nt, id_index=Ct)
    b_s, b_i, b_p = engine.topk(St, k, ids=Dt[Ct], n_valid=Nt)
    assert torch.equal(a_s, b_s) and torch.equal(a_i, b_i) and torch.equal(a_p, b_p)
    for r in range(rows):
        want = O.rank_topk(S[r, : nv[r]], doc_ids[cand[r, : nv[r]]], k)
        assert list(a_i[r, : len(want)].cpu().numpy()) == [w[0] for w in want]


# ----------------------------------------------------------------- prefilter
@pytest.mark.parametrize("gemm2", ["0", "1"])  # chunk-max candidates / second screen GEMM
def test_prefilter_golden(golden_prefilter, gemm2, monkeypatch):
    monkeypatch.setenv("DSRT_SCREEN_GEMM2", gemm2)
    g = golden_prefilter
    sizes = g["doc_sizes"]
    off = np.concatenate([[0], np.cumsum(sizes)])
    docs = [g["docs"][off[i]:off[i + 1]] for i in range(len(sizes))]
    cents = d.Centroids(k=g["centroids"].shape[0], seed=3, vectors=g["centroids"])
    cindex = d.build_centroid_index(docs, cents)
    np.testing.assert_array_equal(cindex.post_off.cpu().numpy(), g["post_off"])
    np.testing.assert_array_equal(cindex.post_docs.cpu().numpy(), g["post_docs"])
    for t, (probe, kf) in enumerate(g["cases"]):
        got = d.filter_candidates(cindex, cents, g[f"q{t}"], int(probe), int(kf))
        np.testing.assert_array_equal(got, g[f"r{t}"], err_msg=f"case {t}")


def test_prefilter_random_vs_oracle():
    rng = np.random.default_rng(21)
    d_, k = 16, 300
    docs = [rng.standard_normal((int(rng.integers(1, 12)), d_)) for _ in range(2000)]
    C = rng.standard_normal((k, d_))
    C /= np.linalg.norm(C, axis=1, keepdims=True)
    cents = d.Centroids(k=k, seed=0, vectors=C)
    cindex = d.build_centroid_index(docs, cents)
    post = O.build_centroid_index(docs, C)
    for t in range(12):
        Q = rng.standard_normal((int(rng.integers(1, 40)), d_))
        probe, kf = int(rng.integers(1, 9)), int(rng.choice([1, 7, 100, 4096]))
        got = d.filter_candidates(cindex, cents, Q, probe, kf)
        want = O.filter_candidates(post, len(docs), C, Q, probe, kf)
        np.testing.assert_array_equal(got, want)


# ------------------------------------------------------- reference API tests
def test_end_to_end_golden_build_and_query(golden_e2e):
    g = golden_e2e
    for n in range(int(g["n_cases"])):
        dd, C, L, seed, top_k = (int(x) for x in g[f"e{n}_shape"])
        sizes = g[f"e{n}_sizes"]
        off = np.concatenate([[0], np.cumsum(sizes)])
        X = g[f"e{n}_X"]
        ids = g[f"e{n}_ids"]
        docs = [(int(ids[i]), X[off[i]:off[i + 1]]) for i in range(len(sizes))]
        idx = d.build_index(docs, d.IndexConfig(d=dd, C=C, L=L, seed=seed,
                                                filter=d.FilterConfig(enabled=False)))
        np.testing.assert_array_equal(idx.codes.cpu().numpy().astype(np.int64), g[f"e{n}_codes"])
        for q in range(2):
            r = d.query(idx, g[f"e{n}_Q"][q], top_k=top_k)
            assert [x for x, _ in r] == list(g[f"e{n}_top_ids"][q]), f"case {n} q {q}"
            assert [v for _, v in r] == list(g[f"e{n}_top_scores"][q])


# ------------------------------------------------ general aggregation (f3)
def test_agg_golden_all_scorers(golden_agg):
    """K3g vs the reference's _score_chunk for every Scorer kind, bit-exact, through
    score_matrix (all sets and an explicit candidate list) and score_candidate."""
    from conftest import agg_case, agg_scorer
    g = golden_agg
    for n in range(int(g["n_shapes"])):
        c = agg_case(g, n)
        cfg = d.IndexConfig(d=4, C=c["C"], L=c["L"], filter=d.FilterConfig(enabled=False))
        idx = d.build_from_codes(torch.from_numpy(c["codes"]).to(DEV), c["sizes"],
                                 np.arange(len(c["sizes"])), cfg)
        N = len(c["sizes"])
        for name in (str(x) for x in g["scorers"]):
            sc = agg_scorer(name, c["weights"])
            want = g[f"a{n}_{name}"]
            got, _ = d.score_matrix(idx, c["qcodes"], scorer=sc)
            np.testing.assert_array_equal(got.cpu().numpy(), want, err_msg=f"{n} {name}")
            sets = np.stack([np.arange(N)[::-1], np.roll(np.arange(N), 3)])
            got2, _ = d.score_matrix(idx, c["qcodes"], sets=sets, scorer=sc)
            np.testing.assert_array_equal(got2.cpu().numpy(),
                                          np.take_along_axis(want, sets, axis=1))
            assert d.score_candidate(idx, 1, c["qcodes"][0], scorer=sc) == want[0, 1]


def test_agg_default_scorer_matches_fast_path(golden_small):
    """max with explicit unit weights (general kernel) == sigma max fast kernels."""
    g = golden_small
    for n in range(int(g["n_shapes"])):
        c = small_case(g, n)
        if c["L"] > 128:
            continue
        cfg = d.IndexConfig(d=4, C=c["C"], L=c["L"], filter=d.FilterConfig(enabled=False))
        idx = d.build_from_codes(torch.from_numpy(c["codes"]).to(DEV), c["sizes"],
                                 c["doc_ids"], cfg)
        sc = d.Scorer(inner=d.max_aggregation(), weights=np.ones(c["m_q"]))
        got, _ = d.score_matrix(idx, c["qcodes"], scorer=sc)
        np.testing.assert_array_equal(got.cpu().numpy(), c["scores"])


def test_agg_end_to_end_query(golden_agg):
    """build_index with inner_kind='avg-phi' -> query / query_batch vs the reference."""
    g = golden_agg
    for n in range(int(g["n_e2e"])):
        dd, C, L, seed, top_k = (int(x) for x in g[f"e{n}_shape"])
        phi = str(g[f"e{n}_phi"])
        sizes = g[f"e{n}_sizes"]
        off = np.concatenate([[0], np.cumsum(sizes)])
        X, ids = g[f"e{n}_X"], g[f"e{n}_ids"]
        docs = [(int(ids[i]), X[off[i]:off[i + 1]]) for i in range(len(sizes))]
        cfg = d.IndexConfig(d=dd, C=C, L=L, seed=seed, inner_kind="avg-phi", phi=phi,
                            filter=d.FilterConfig(enabled=False))
        idx = d.build_index(docs, cfg)
        for q in range(2):
            r = d.query(idx, g[f"e{n}_Q"][q], top_k=top_k)
            assert [x for x, _ in r] == list(g[f"e{n}_top_ids"][q]), f"case {n} q {q}"
            assert [v for _, v in r] == list(g[f"e{n}_top_scores"][q])
        out_s, out_i = d.query_batch(idx, g[f"e{n}_Q"], top_k, return_tensors=True)
        np.testing.assert_array_equal(out_i.cpu().numpy(), g[f"e{n}_top_ids"])
        np.testing.assert_array_equal(out_s.cpu().numpy(), g[f"e{n}_top_scores"])


@pytest.mark.parametrize("m_q", [1, 7, 33, 129, 300])
def test_agg_weighted_and_avgphi_any_mq(m_q):
    """Weighted max across the K3 variants (m_q <= 128 single pass, > 128 slices +
    finalize) and avg-phi across K3a (m_q <= 32) / K3g (larger m_q), vs the dense
    oracle, bit-exact; exhaustive (>= 8 query sets) and candidate lists."""
    from oracle import dessert_oracle as O
    from paper_2210_15748_b200 import scoring
    rng = np.random.default_rng(m_q)
    L, C = 32, 5
    sizes = rng.integers(1, 60, size=40)
    hot = rng.integers(0, 32, size=L)
    codes = rng.integers(0, 32, size=(int(sizes.sum()), L))
    mask = rng.random(codes.shape) < 0.5
    codes[mask] = np.broadcast_to(hot, codes.shape)[mask]
    off = np.concatenate([[0], np.cumsum(sizes)])
    n_q = 9
    qc = rng.integers(0, 32, size=(n_q, m_q, L))
    qm = rng.random(qc.shape) < 0.5
    qc[qm] = np.broadcast_to(hot, qc.shape)[qm]
    cfg = d.IndexConfig(d=4, C=C, L=L, filter=d.FilterConfig(enabled=False))
    idx = d.build_from_codes(torch.from_numpy(codes.astype(np.int32)).to(DEV), sizes,
                             np.arange(len(sizes)), cfg)
    w = rng.uniform(0, 1, size=m_q)
    sets = np.stack([rng.permutation(len(sizes))[:25] for _ in range(n_q)])
    for sc in (d.Scorer(d.max_aggregation(), w), d.Scorer(d.avg_phi_aggregation("exp-minus-one"), w),
               d.Scorer(d.avg_phi_aggregation("identity"))):
        table = scoring.table_for(idx.lookup.table, sc)
        kind = sc.inner.kind
        want = np.stack([O.score_sets_dense_agg(qc[r], codes, off, table, kind, sc.weights)
                         for r in range(n_q)])
        got, _ = d.score_matrix(idx, qc, scorer=sc)
        np.testing.assert_array_equal(got.cpu().numpy(), want, err_msg=f"{kind} all")
        got2, _ = d.score_matrix(idx, qc, sets=sets, scorer=sc)
        np.testing.assert_array_equal(got2.cpu().numpy(), np.take_along_axis(want, sets, axis=1),
                                      err_msg=f"{kind} cand")


def test_agg_random_long_sets_vs_oracle():
    """Sets with up to 600 vectors (several recursive pairwise levels), m_q = 70,
    avg-phi with weights, against the dense restatement."""
    from oracle import dessert_oracle as O
    from paper_2210_15748_b200 import scoring
    rng = np.random.default_rng(5)
    L, C, m_q = 24, 3, 70
    sizes = np.array([600, 1, 257, 129, 130, 8, 9, 450])
    hot = rng.integers(0, 8, size=L)
    codes = rng.integers(0, 8, size=(int(sizes.sum()), L))
    mask = rng.random(codes.shape) < 0.5
    codes[mask] = np.broadcast_to(hot, codes.shape)[mask]
    qc = rng.integers(0, 8, size=(1, m_q, L))
    off = np.concatenate([[0], np.cumsum(sizes)])
    cfg = d.IndexConfig(d=4, C=C, L=L, filter=d.FilterConfig(enabled=False))
    idx = d.build_from_codes(torch.from_numpy(codes.astype(np.int32)).to(DEV), sizes,
                             np.arange(len(sizes)), cfg)
    w = rng.uniform(0, 1, size=m_q)
    for phi in d.PHI_KINDS:
        sc = d.Scorer(inner=d.avg_phi_aggregation(phi), weights=w)
        table = scoring.table_for(idx.lookup.table, sc)
        want = O.score_sets_dense_agg(qc[0], codes, off, table, "avg-phi", w)
        got, _ = d.score_matrix(idx, qc, scorer=sc)
        np.testing.assert_array_equal(got.cpu().numpy()[0], want)


@pytest.mark.parametrize("L,C", [(32, 7), (64, 7), (32, 8), (16, 3)])
def test_candidate_split_lane_mapping(L, C, monkeypatch):
    """Candidate lists with 16 < m_q <= 32 take the split-lane kernel (two query
    vectors per lane, half-warps on alternate set vectors).  Odd / even / 1-vector
    sets, sets spanning several staging pieces, duplicate and invalid candidates,
    uint16 max counts; equal to the oracle and to the plain mapping (DSRT_QS=-1)."""
    rng = np.random.default_rng(L * 100 + C)
    r = 1 << C
    sizes = np.concatenate([[1, 2, 3, 4, 5, 96, 97, 191, 193, 300], rng.integers(1, 140, size=50)])
    hot = rng.integers(0, r, size=L)
    codes = rng.integers(0, r, size=(int(sizes.sum()), L))
    mask = rng.random(codes.shape) < 0.6
    codes[mask] = np.broadcast_to(hot, codes.shape)[mask]
    off = np.concatenate([[0], np.cumsum(sizes)])
    idx = _index_from_codes(codes, sizes, L, C)
    N = len(sizes)
    for m_q in (17, 24, 31, 32):
        n_q = 5
        qc = rng.integers(0, r, size=(n_q, m_q, L))
        qm = rng.random(qc.shape) < 0.6
        qc[qm] = np.broadcast_to(hot, qc.shape)[qm]
        sets = np.stack([rng.permutation(N)[:40] for _ in range(n_q)])
        sets[0, 3] = sets[0, 4]  # a duplicate candidate
        want = c_oracle.score(codes.astype(np.int64), off, qc, idx.lookup.table, sets=sets)
        got, _ = d.score_matrix(idx, qc, sets=sets)
        np.testing.assert_array_equal(got.cpu().numpy(), want, err_msg=f"m_q={m_q}")
        monkeypatch.setenv("DSRT_QS", "-1")
        plain, _ = d.score_matrix(idx, qc, sets=sets)
        monkeypatch.delenv("DSRT_QS")
        np.testing.assert_array_equal(plain.cpu().numpy(), want)
        # raw ABI: invalid set index -> NaN, max counts
        qrecs, _ = engine.codes_to_records(torch.from_numpy(qc.reshape(-1, L).astype(np.int32)).to(DEV), L, C)
        cand = torch.from_numpy(sets).to(DEV).clone()
        cand[1, 0] = N + 5
        n_cand = torch.tensor([40, 39, 1, 0, 40], dtype=torch.int32, device=DEV)
        out, mc = engine.score_candidates(idx.records, idx.set_off, qrecs, m_q, L, C, idx.lut_dev,
                                          cand, n_cand, want_counts=True)
        o = out.cpu().numpy()
        assert np.isnan(o[1, 0])
        for q, n in enumerate([40, 39, 1, 0, 40]):
            lo = 1 if q == 1 else 0
            np.testing.assert_array_equal(o[q, lo:n], want[q, lo:n])
        cnt = c_oracle.score(codes.astype(np.int64), off, qc, idx.lookup.table, sets=sets,
                             want_counts=True)[1]
        np.testing.assert_array_equal(mc.cpu().numpy()[0].astype(np.uint16), cnt[0])
        np.testing.assert_array_equal(mc.cpu().numpy()[4].astype(np.uint16), cnt[4])


# ------------------------------------------------------ k-means (K7, f4)
def test_train_centroids_golden(golden_kmeans):
    """Native train_centroids vs the reference's, bit for bit (TC path at d=128,
    SIMT path otherwise, dead-cluster reseeding in the 'dups' cases)."""
    import kmeans_inputs as KI
    g = golden_kmeans
    for c, (n, dd, k, iters, seed, _) in enumerate(KI.SPECS):
        S = KI.samples(c)
        got = d.train_centroids(S, k, iters, seed).vectors
        want = g[f"k{c}_C"]
        np.testing.assert_array_equal(got, want, err_msg=f"case {c}: max |diff| "
                                      f"{np.abs(got - want).max():.3e}")
        # deterministic: a second run (and a device-resident input) gives the same bytes
        got2 = d.train_centroids(torch.from_numpy(S).to(DEV), k, iters, seed).vectors
        np.testing.assert_array_equal(got2, got)


def test_train_centroids_errors():
    with pytest.raises(ValueError, match="zero vector"):
        d.train_centroids(np.zeros((3, 4)), 0, 1, 0)
    with pytest.raises(ValueError, match="k must be"):
        d.train_centroids(np.ones((3, 4)), 0, 1, 0)
    with pytest.raises(ValueError, match="too few samples"):
        d.train_centroids(np.ones((3, 4)), 4, 1, 0)
    with pytest.raises(ValueError, match="iters"):
        d.train_centroids(np.ones((3, 4)), 2, 0, 0)
    with pytest.raises(ValueError, match="non-empty"):
        d.train_centroids(np.ones((0, 4)), 1, 1, 0)


def test_filter_enabled_build_query_golden(golden_kmeans):
    """build_index with the prefilter on (trained centroids, postings) -> query,
    against the reference end to end."""
    import kmeans_inputs as KI
    g = golden_kmeans
    sizes, X, ids, Q = KI.e2e_docs()
    off = np.concatenate([[0], np.cumsum(sizes)])
    docs = [(int(ids[i]), X[off[i]:off[i + 1]]) for i in range(len(sizes))]
    cfg = d.IndexConfig(d=128, C=6, L=32, seed=11,
                        filter=d.FilterConfig(enabled=True, iters=4, probe=3, k_filter=40))
    idx = d.build_index(docs, cfg)
    centroids, cindex = idx.filter
    np.testing.assert_array_equal(centroids.vectors, g["e_centroids"])
    np.testing.assert_array_equal(cindex.post_off.cpu().numpy(), g["e_post_off"])
    np.testing.assert_array_equal(cindex.post_docs.cpu().numpy(), g["e_post_docs"])
    for q in range(Q.shape[0]):
        r = d.query(idx, Q[q], top_k=10)
        assert [x for x, _ in r] == list(g["e_top_ids"][q])
        assert [v for _, v in r] == list(g["e_top_scores"][q])


def test_reference_index_semantics():  # pkg/tests/test_index.py restated
    nf = d.FilterConfig(enabled=False)
    rng = np.random.default_rng(0)
    S = rng.standard_normal((5, 8))
    idx = d.build_index([(0, S)], d.IndexConfig(d=8, C=3, L=16, filter=nf))
    assert d.score_candidate(idx, 0, d.hash_matrix(idx.family, S)) == pytest.approx(1.0)
    v = np.random.default_rng(1).standard_normal(8)
    idx = d.build_index([(0, v[None, :])], d.IndexConfig(d=8, C=1, L=32, filter=nf))
    assert d.score_candidate(idx, 0, d.hash_matrix(idx.family, -v[None, :])) == 0.0
    with pytest.raises(IndexError):
        d.score_candidate(idx, 1, d.hash_matrix(idx.family, v[None, :]))
    idx = d.build_index([(7, np.ones((1, 4)))], d.IndexConfig(d=4, C=2, L=3, filter=nf))
    assert idx.n_docs == 1 and idx.sketches[0].m == 1 and list(idx.doc_ids) == [7]
    with pytest.raises(ValueError, match="empty query"):
        d.query(idx, np.ones((0, 4)), 1)
    with pytest.raises(ValueError, match="invalid parameter"):
        d.query(idx, np.ones((1, 4)), 0)
    with pytest.raises(ValueError, match="dimension"):
        d.query(idx, np.ones((1, 5)), 1)
    with pytest.raises(ValueError, match="zero vector"):
        d.query(idx, np.zeros((1, 4)), 1)
    with pytest.raises(ValueError, match="zero vector"):
        d.build_index([(0, np.array([[1.0, 1.0], [0.0, 0.0]]))], d.IndexConfig(d=2, filter=nf))
    # permutation invariance + threads invariance
    S = rng.standard_normal((6, 8))
    Q = rng.standard_normal((2, 8))
    a = d.build_index([(0, S)], d.IndexConfig(d=8, C=3, L=16, seed=11, filter=nf))
    b = d.build_index([(0, S[::-1])], d.IndexConfig(d=8, C=3, L=16, seed=11, filter=nf))
    assert d.query(a, Q, 1) == d.query(b, Q, 1)
    docs = [(i, rng.standard_normal((int(rng.integers(1, 6)), 8))) for i in range(30)]
    idx = d.build_index(docs, d.IndexConfig(d=8, C=2, L=16, seed=24, filter=nf))
    assert d.query(idx, Q, 10, threads=1) == d.query(idx, Q, 10, threads=4)
    out = d.query(idx, Q, top_k=30)
    assert len(out) == 30 and [s for _, s in out] == sorted([s for _, s in out], reverse=True)


def test_add_sets_equals_full_build():
    rng = np.random.default_rng(5)
    docs = [(i * 3, rng.standard_normal((int(rng.integers(1, 30)), 16))) for i in range(120)]
    cfg = d.IndexConfig(d=16, C=5, L=32, seed=2, filter=d.FilterConfig(enabled=False))
    full = d.build_index(docs, cfg)
    part = d.build_index(docs[:50], cfg)
    d.add_sets(part, docs[50:])
    Q = rng.standard_normal((4, 20, 16))
    assert d.query_batch(full, Q, 15) == d.query_batch(part, Q, 15)
    with pytest.raises(ValueError, match="duplicate"):
        d.add_sets(part, docs[:1])


@pytest.mark.parametrize("dd", [16, 48, 200])
def test_centroid_index_any_d_matches_oracle(dd):
    """K6 for d != 128 (float64 SIMT path) vs the oracle's build_centroid_index,
    float64 and float32 documents, with duplicated centroids (exact ties)."""
    rng = np.random.default_rng(dd)
    k = 37
    C = rng.standard_normal((k, dd))
    C[5] = C[4]
    C = C / np.linalg.norm(C, axis=1, keepdims=True)
    docs = [rng.standard_normal((int(rng.integers(1, 12)), dd)) for _ in range(150)]
    docs[3][0] = C[4] * 2.0  # exact tie between centroids 4 and 5
    cents = d.Centroids(k=k, seed=0, vectors=C)
    want = O.build_centroid_index(docs, C)
    for dt in (np.float64, np.float32):
        cindex = d.build_centroid_index([x.astype(dt) for x in docs], cents)
        got = cindex.postings
        for c in range(k):
            np.testing.assert_array_equal(got[c], want[c], err_msg=f"centroid {c}")


def test_add_sets_with_prefilter_equals_full_build():
    """add_sets extends the postings natively (new docs appended per centroid)."""
    rng = np.random.default_rng(8)
    docs = [(i, rng.standard_normal((int(rng.integers(1, 20)), 128))) for i in range(300)]
    cfg = d.IndexConfig(d=128, C=6, L=32, seed=3,
                        filter=d.FilterConfig(enabled=True, centroids=20, iters=3, probe=3,
                                              k_filter=60))
    full = d.build_index(docs, cfg)
    part = d.build_index(docs[:180], cfg)
    part.filter = (full.filter[0], d.build_centroid_index([x for _, x in docs[:180]],
                                                          full.filter[0]))
    d.add_sets(part, docs[180:])
    np.testing.assert_array_equal(part.filter[1].post_off.cpu().numpy(),
                                  full.filter[1].post_off.cpu().numpy())
    np.testing.assert_array_equal(part.filter[1].post_docs.cpu().numpy(),
                                  full.filter[1].post_docs.cpu().numpy())
    Q = rng.standard_normal((3, 16, 128))
    assert d.query_batch(full, Q, 10) == d.query_batch(part, Q, 10)


def test_prefilter_small_and_large_batch_paths_agree():
    """The chunk-parallel selection (small batches) and the single-CTA ordered scan
    (large batches) give the oracle's candidates; many ties at c* (low k_filter)."""
    from paper_2210_15748_b200 import prefilter as pf
    rng = np.random.default_rng(12)
    dd, k = 128, 300
    C = rng.standard_normal((k, dd))
    C /= np.linalg.norm(C, axis=1, keepdims=True)
    docs = [rng.standard_normal((int(rng.integers(1, 10)), dd)) for _ in range(200_000 // 50)]
    cents = d.Centroids(k=k, seed=0, vectors=C)
    cindex = d.build_centroid_index(docs, cents)
    post = cindex.postings
    n_q, m_q = 40, 16
    Q = rng.standard_normal((n_q * m_q, dd))
    for probe, k_filter in ((2, 7), (4, 300), (3, 4096)):
        big, nb = pf.filter_candidates_device(cindex, cents, torch.from_numpy(Q).to(DEV), m_q, probe,
                                              k_filter)
        for q in range(n_q):
            want = O.filter_candidates(post, len(docs), C, Q[q * m_q:(q + 1) * m_q], probe, k_filter)
            np.testing.assert_array_equal(big[q, : int(nb[q])].cpu().numpy(), want)
            one, n1 = pf.filter_candidates_device(cindex, cents,
                                                  torch.from_numpy(Q[q * m_q:(q + 1) * m_q]).to(DEV),
                                                  m_q, probe, k_filter)
            np.testing.assert_array_equal(one[0, : int(n1[0])].cpu().numpy(), want)


@pytest.mark.parametrize("mq_probe", [(8, 5), (64, 8)])  # u8 and u16 (m_q*probe > 255) counters
@pytest.mark.parametrize("fused", ["1", "0"])
@pytest.mark.parametrize("k_filter", [1, 5, 64, 1000, 4096, 16384])
def test_prefilter_selection_many_chunks(k_filter, fused, mq_probe, monkeypatch):
    """Selection over 330k docs (6 counter chunks of 64k docs) with hand-made postings:
    dense postings give counts 1..m_q*probe with equal counts spread over every chunk,
    so the per-count slot bases, the cross-chunk tie ranks and the < k_filter case are
    all exercised; batch 1 and a batch of 24 query sets vs the oracle, through the fused
    cluster kernel and the two-kernel count -> place path."""
    from paper_2210_15748_b200 import prefilter as pf
    monkeypatch.setenv("DSRT_FUSED_SELECT", fused)
    rng = np.random.default_rng(5)
    n_docs, k, dd = 330_000, 48, 128
    C = rng.standard_normal((k, dd))
    C /= np.linalg.norm(C, axis=1, keepdims=True)
    post = []
    for c in range(k):
        frac = [0.3, 0.05, 0.002, 0.0002][c % 4]
        lo = int(rng.integers(0, n_docs // 2))
        cand_docs = np.arange(lo, n_docs) if c % 5 else np.arange(n_docs)
        post.append(np.sort(rng.choice(cand_docs, size=max(1, int(frac * len(cand_docs))),
                                       replace=False)).astype(np.int64))
    off = np.concatenate([[0], np.cumsum([len(p) for p in post])])
    cindex = pf.CentroidIndex(n_docs=n_docs, post_off=torch.from_numpy(off).to(DEV),
                              post_docs=torch.from_numpy(np.concatenate(post)).to(DEV))
    cents = d.Centroids(k=k, seed=0, vectors=C)
    n_q, (m_q, probe) = 24, mq_probe
    Q = rng.standard_normal((n_q * m_q, dd))
    got, n = pf.filter_candidates_device(cindex, cents, torch.from_numpy(Q).to(DEV), m_q, probe, k_filter)
    for q in (0, 1, 7, 23):
        want = O.filter_candidates(post, n_docs, C, Q[q * m_q:(q + 1) * m_q], probe, k_filter)
        assert int(n[q]) == len(want)
        np.testing.assert_array_equal(got[q, : int(n[q])].cpu().numpy(), want)
        assert np.all(got[q, int(n[q]):].cpu().numpy() == -1)
        one, n1 = pf.filter_candidates_device(cindex, cents, torch.from_numpy(Q[q * m_q:(q + 1) * m_q]).to(DEV),
                                              m_q, probe, k_filter)
        np.testing.assert_array_equal(one[0, : int(n1[0])].cpu().numpy(), want)


def test_chunked_exhaustive_partial_last_chunk(monkeypatch):
    """rank_records with a score buffer smaller than N (last chunk partial, row-strided
    view into the buffer) equals the unchunked ranking."""
    from paper_2210_15748_b200 import index as I
    rng = np.random.default_rng(21)
    L, C = 32, 6
    sizes = rng.integers(1, 40, size=1003)
    codes = rng.integers(0, 64, size=(int(sizes.sum()), L)).astype(np.int32)
    cfg = d.IndexConfig(d=4, C=C, L=L, filter=d.FilterConfig(enabled=False))
    idx = d.build_from_codes(torch.from_numpy(codes).to(DEV), sizes, rng.permutation(5000)[:1003], cfg)
    qc = rng.integers(0, 64, size=(16, 24, L))
    want = d.query_codes_batch(idx, qc, 37)
    monkeypatch.setattr(I, "SCORE_BUFFER_BYTES", 8 * 16 * 300)  # 300-set chunks -> 4 chunks
    got = d.query_codes_batch(idx, qc, 37)
    assert got == want


def test_top_k_beyond_selector(monkeypatch):
    """top_k > 4096 (device two-key stable sort), exhaustive, chunked and from a
    candidate list, equals heapq ranking of the oracle scores (ties by doc id)."""
    from paper_2210_15748_b200 import index as I
    rng = np.random.default_rng(31)
    L, C, N = 16, 3, 6000
    sizes = rng.integers(1, 6, size=N)
    codes = rng.integers(0, 8, size=(int(sizes.sum()), L)).astype(np.int32)
    off = np.concatenate([[0], np.cumsum(sizes)])
    ids = rng.permutation(100_000)[:N]
    cfg = d.IndexConfig(d=4, C=C, L=L, filter=d.FilterConfig(enabled=False))
    idx = d.build_from_codes(torch.from_numpy(codes).to(DEV), sizes, ids, cfg)
    qc = rng.integers(0, 8, size=(2, 5, L))
    scores = c_oracle.score(codes.astype(np.int64), off, qc, idx.lookup.table)
    for k in (4097, 5000, N + 10):
        want = [O.rank_topk(scores[r], ids, k) for r in range(2)]
        assert d.query_codes_batch(idx, qc, k) == want
        monkeypatch.setattr(I, "SCORE_BUFFER_BYTES", 8 * 2 * 2500)  # chunked
        assert d.query_codes_batch(idx, qc, k) == want
        monkeypatch.undo()
    # candidate lists (prefilter output form) with k above the selector
    cand = torch.from_numpy(np.stack([rng.permutation(N)[:4500] for _ in range(2)])).to(DEV)
    n_cand = torch.tensor([4500, 4321], dtype=torch.int32, device=DEV)
    qrecs, _ = d.engine.codes_to_records(torch.from_numpy(qc.reshape(-1, L).astype(np.int32)).to(DEV), L, C)
    out_s, out_i = I.rank_records(idx, qrecs, 5, 4400, cand=cand, n_cand=n_cand)
    for r in range(2):
        cr = cand[r, : int(n_cand[r])].cpu().numpy()
        want = O.rank_topk(scores[r][cr], ids[cr], 4400)
        got_s, got_i = out_s[r].cpu().numpy(), out_i[r].cpu().numpy()
        valid = got_s >= 0
        assert [(int(a), float(b)) for a, b in zip(got_i[valid], got_s[valid])] == want


def test_query_graph_invalidation_and_threads(monkeypatch):
    """query() runs through a cached CUDA graph: it must follow add_sets / filter
    changes, agree with the eager path, and stay correct under concurrent threads."""
    import threading
    rng = np.random.default_rng(44)
    docs = [(i, rng.standard_normal((int(rng.integers(1, 15)), 32))) for i in range(300)]
    cfg = d.IndexConfig(d=32, C=5, L=32, seed=4, filter=d.FilterConfig(enabled=False))
    full = d.build_index(docs, cfg)
    part = d.build_index(docs[:150], cfg)
    Qs = [rng.standard_normal((7, 32)) for _ in range(12)]
    before = [d.query(part, q, 9) for q in Qs]           # graphs captured on `part`
    d.add_sets(part, docs[150:])
    after = [d.query(part, q, 9) for q in Qs]
    assert after == [d.query(full, q, 9) for q in Qs]
    monkeypatch.setenv("DSRT_QUERY_GRAPHS", "0")
    assert after == [d.query(part, q, 9) for q in Qs]     # eager path agrees
    assert before != after
    monkeypatch.delenv("DSRT_QUERY_GRAPHS")
    results = {}

    def worker(t):
        for r in range(20):
            i = (t * 7 + r) % len(Qs)
            results[(t, r)] = (i, d.query(full, Qs[i], 9))

    threads = [threading.Thread(target=worker, args=(t,)) for t in range(4)]
    for th in threads:
        th.start()
    for th in threads:
        th.join()
    for i, res in results.values():
        assert res == after[i]


def test_filtered_query_matches_reference_pipeline():
    """build_index with the prefilter on: candidates from K5, then K3/K4 over them,
    equals the oracle pipeline given the same centroids and postings."""
    rng = np.random.default_rng(8)
    docs = [(i, rng.standard_normal((int(rng.integers(2, 10)), 16))) for i in range(400)]
    cfg = d.IndexConfig(d=16, C=4, L=32, seed=1,
                        filter=d.FilterConfig(enabled=True, centroids=24, probe=2, k_filter=50))
    idx = d.build_index(docs, cfg)
    cents, cindex = idx.filter
    post = cindex.postings
    codes = idx.codes.cpu().numpy()
    off = idx.set_off.cpu().numpy()
    lut = O.sim_lut(4, 32)
    for t in range(6):
        Q = rng.standard_normal((int(rng.integers(1, 20)), 16))
        got = d.query(idx, Q, top_k=10)
        cand = O.filter_candidates(post, 400, cents.vectors, Q, 2, 50)
        qc = O.hash_matrix(idx.family.planes, 32, 4, Q)
        s = O.score_sets_dense(qc, codes, off, lut, sets=cand)
        want = O.rank_topk(s, [int(i) for i in idx.doc_ids[cand]], 10)
        assert got == want


@pytest.mark.parametrize("phi", ["identity", "debiased-sigmoid"])
def test_filtered_avgphi_query_matches_oracle_pipeline(phi):
    """avg-phi + weights behind the prefilter (candidate lists with n_cand padding,
    K3a streaming kernel) through query / query_batch vs the oracle pipeline."""
    from paper_2210_15748_b200 import scoring
    rng = np.random.default_rng(81)
    docs = [(i, rng.standard_normal((int(rng.integers(2, 40)), 16))) for i in range(500)]
    cfg = d.IndexConfig(d=16, C=4, L=32, seed=1, inner_kind="avg-phi", phi=phi,
                        filter=d.FilterConfig(enabled=True, centroids=24, probe=2, k_filter=60))
    idx = d.build_index(docs, cfg)
    cents, cindex = idx.filter
    post = cindex.postings
    codes = idx.codes.cpu().numpy()
    off = idx.set_off.cpu().numpy()
    table = scoring.phi_function(phi)(O.sim_lut(4, 32))
    Qs = rng.standard_normal((5, 12, 16))
    w = rng.uniform(0, 1, size=12)
    sc = d.Scorer(d.avg_phi_aggregation(phi), w)
    batch = d.query_batch(idx, Qs, 10, scorer=sc)
    for t in range(5):
        cand = O.filter_candidates(post, 500, cents.vectors, Qs[t], 2, 60)
        qc = O.hash_matrix(idx.family.planes, 32, 4, Qs[t])
        s_w = O.score_sets_dense_agg(qc, codes, off, table, "avg-phi", w, sets=cand)
        want_w = O.rank_topk(s_w, [int(i) for i in idx.doc_ids[cand]], 10)
        assert batch[t] == want_w
        s0 = O.score_sets_dense_agg(qc, codes, off, table, "avg-phi", None, sets=cand)
        assert d.query(idx, Qs[t], top_k=10) == O.rank_topk(s0, [int(i) for i in idx.doc_ids[cand]], 10)


@pytest.mark.parametrize("seed", range(24))
def test_random_shapes_sweep(seed):
    """Randomised (L, C, m_q, set sizes) sweep through every scoring entry point,
    bit-exact against the C oracle (scores and integer max counts) and the heapq
    ranking; hot codes make collisions and ties frequent."""
    rng = np.random.default_rng(1000 + seed)
    L = int(rng.choice([1, 5, 8, 16, 31, 32, 33, 48, 63, 64, 65, 96, 127, 128]))
    C = int(rng.integers(1, 17))
    while C * ((L + 31) // 32) > 32:
        C = int(rng.integers(1, 17))
    m_q = int(rng.choice([1, 2, 7, 8, 9, 31, 32, 33, 64, 100, 128, 129, 257]))
    n_sets = int(rng.integers(1, 120))
    sizes = rng.integers(1, int(rng.choice([3, 40, 300])) + 1, size=n_sets)
    r = 1 << C
    hot = rng.integers(0, r, size=L)
    codes = rng.integers(0, r, size=(int(sizes.sum()), L))
    m = rng.random(codes.shape) < rng.uniform(0.2, 0.9)
    codes[m] = np.broadcast_to(hot, codes.shape)[m]
    n_q = int(rng.choice([1, 3, 8, 11]))
    qc = rng.integers(0, r, size=(n_q, m_q, L))
    qm = rng.random(qc.shape) < rng.uniform(0.2, 0.9)
    qc[qm] = np.broadcast_to(hot, qc.shape)[qm]
    off = np.concatenate([[0], np.cumsum(sizes)])
    idx = _index_from_codes(codes, sizes, L, C)
    lut = O.sim_lut(C, L)
    want, wmc = c_oracle.score(codes, off, qc, lut, want_counts=True)
    got, mc = d.score_matrix(idx, qc, want_counts=True)
    np.testing.assert_array_equal(got.cpu().numpy(), want)
    np.testing.assert_array_equal(mc.cpu().numpy().astype(np.int64).reshape(wmc.shape), wmc)
    sets = np.stack([rng.permutation(n_sets)[: max(1, n_sets // 2)] for _ in range(n_q)])
    got2, _ = d.score_matrix(idx, qc, sets=sets)
    np.testing.assert_array_equal(got2.cpu().numpy(), np.take_along_axis(want, sets, axis=1))
    k = int(rng.integers(1, n_sets + 3))
    res = d.query_codes_batch(idx, qc, k)
    for q in range(n_q):
        assert res[q] == O.rank_topk(want[q], np.arange(n_sets), k)


# ------------------------------------------------------------ larger shapes
def test_cfg1_shape_sampled_parity():
    """cfg1 shapes (L=64, C=7, m_i ~ N(70,20) clipped) at 20k sets: 16 query sets
    exhaustive vs the C oracle, all bit-exact, plus top-100."""
    from paper_2210_15748_b200 import workloads
    sizes = workloads.set_sizes(20_000, 70, 20, seed=1)
    off = workloads.offsets(sizes)
    rng = np.random.default_rng(2)
    hot = rng.integers(0, 128, size=64)
    codes = rng.integers(0, 128, size=(int(off[-1]), 64))
    m = rng.random(codes.shape) < 0.6
    codes[m] = np.broadcast_to(hot, codes.shape)[m]
    q = rng.integers(0, 128, size=(16, 32, 64))
    qm = rng.random(q.shape) < 0.6
    q[qm] = np.broadcast_to(hot, q.shape)[qm]
    idx = _index_from_codes(codes, sizes, 64, 7)
    s, _ = d.score_matrix(idx, q)
    want = c_oracle.score(codes, off, q, O.sim_lut(7, 64))
    np.testing.assert_array_equal(s.cpu().numpy(), want)
    res = d.query_codes_batch(idx, q, 100)
    for r in range(16):
        assert res[r] == O.rank_topk(want[r], np.arange(20_000), 100)


def test_mq_variants_bit_exact():
    """m_q in {1, 7, 8, 31, 33, 64, 100, 128, 129, 200, 300} (one leaf, multi-slot, recursion)."""
    rng = np.random.default_rng(12)
    sizes = rng.integers(1, 90, size=300).astype(np.int64)
    off = np.concatenate([[0], np.cumsum(sizes)])
    codes = rng.integers(0, 8, size=(int(off[-1]), 32))
    idx = _index_from_codes(codes, sizes, 32, 3)
    lut = O.sim_lut(3, 32)
    for m_q in (1, 7, 8, 31, 33, 64, 100, 128, 129, 200, 300):
        q = rng.integers(0, 8, size=(9, m_q, 32))
        s, mc = d.score_matrix(idx, q, want_counts=True)
        want, wmc = c_oracle.score(codes, off, q, lut, want_counts=True)
        np.testing.assert_array_equal(s.cpu().numpy(), want, err_msg=f"m_q={m_q}")
        np.testing.assert_array_equal(mc.cpu().numpy().astype(np.uint16), wmc)
        s2, _ = d.score_matrix(idx, q[:2])
        np.testing.assert_array_equal(s2.cpu().numpy(), want[:2])


# ------------------------------------------------------- tensor-core prefilter
def _tc_prefilter_case(seed, n_docs, k, dup_noise=None):
    rng = np.random.default_rng(seed)
    docs = [rng.standard_normal((int(rng.integers(1, 12)), 128)) for _ in range(n_docs)]
    C = rng.standard_normal((k, 128))
    if dup_noise is not None:        # near-identical centroid pairs -> screen near-ties
        C[1::2] = C[0::2][: C[1::2].shape[0]] + dup_noise * rng.standard_normal(C[1::2].shape)
        C[5] = C[4]                   # an exact tie
    C /= np.linalg.norm(C, axis=1, keepdims=True)
    return rng, docs, C


@pytest.mark.parametrize("gemm2", ["0", "1"])  # chunk-max candidates / second screen GEMM
@pytest.mark.parametrize("seed,dup", [(1, None), (2, 1e-5), (3, 1e-3)])
def test_prefilter_tensor_core_screen_exact(seed, dup, gemm2, monkeypatch):
    monkeypatch.setenv("DSRT_SCREEN_GEMM2", gemm2)
    from paper_2210_15748_b200 import prefilter as pf
    rng, docs, C = _tc_prefilter_case(seed, 3000, 1000, dup)
    cents = d.Centroids(k=C.shape[0], seed=0, vectors=C)
    cindex = d.build_centroid_index(docs, cents)
    post = O.build_centroid_index(docs, C)
    for t in range(10):
        m_q = int(rng.choice([1, 7, 32, 64]))
        Q = rng.standard_normal((m_q, 128))
        if t % 3 == 0:
            Q[0] = C[4] * 2.5        # exact tie between centroids 4 and 5
        probe, kf = int(rng.integers(1, 9)), int(rng.choice([1, 50, 4096]))
        want = O.filter_candidates(post, len(docs), C, Q, probe, kf)
        Qd = torch.from_numpy(Q).to(DEV)
        cand, n_cand = pf.filter_candidates_device(cindex, cents, Qd, m_q, probe, kf, use_tc=True)
        got = cand[0, : int(n_cand[0])].cpu().numpy()
        np.testing.assert_array_equal(got, want, err_msg=f"case {t} probe {probe}")
    # batched: many query sets at once vs the exact SIMT kernel (2240 rows: two-row-tile
    # screen CTAs with a partial last tile)
    Qb = torch.from_numpy(rng.standard_normal((70 * 32, 128))).to(DEV)
    a, na = pf.filter_candidates_device(cindex, cents, Qb, 32, 4, 300, use_tc=True)
    b, nb = pf.filter_candidates_device(cindex, cents, Qb, 32, 4, 300, use_tc=False)
    assert torch.equal(na, nb) and torch.equal(a, b)


# ------------------------------------------------ native centroid assignment (K6)
@pytest.mark.parametrize("dtype", [torch.float16, torch.bfloat16, torch.float32, torch.float64])
def test_native_centroid_index_matches_oracle(dtype):
    rng = np.random.default_rng(40)
    k = 700
    C = rng.standard_normal((k, 128))
    C[1::2] = C[0::2] + 1e-4 * rng.standard_normal(C[0::2].shape)   # near-ties
    C[9] = C[8]                                                       # exact tie -> lower id
    C /= np.linalg.norm(C, axis=1, keepdims=True)
    docs = [rng.standard_normal((int(rng.integers(1, 40)), 128)) for _ in range(1500)]
    docs[3][0] = C[8] * 3.0                                           # lands exactly on the tie
    docs_t = [torch.from_numpy(x).to(dtype) for x in docs]
    exact = [x.to(torch.float64).numpy() for x in docs_t]             # values the device sees
    cents = d.Centroids(k=k, seed=0, vectors=C)
    got = d.build_centroid_index(docs_t, cents)
    want = O.build_centroid_index(exact, C)
    off = got.post_off.cpu().numpy()
    pd = got.post_docs.cpu().numpy()
    for c in range(k):
        np.testing.assert_array_equal(pd[off[c]:off[c + 1]], want[c], err_msg=f"centroid {c}")


def test_counting_sort_large_sets_and_keys():
    rng = np.random.default_rng(41)
    n_sets, n = 70_000, 600_000
    set_of = rng.integers(0, n_sets, size=n)
    set_of[:20_000] = 17                                              # one huge set (> 4096)
    rng.shuffle(set_of)
    so, perm = engine.counting_sort(torch.from_numpy(set_of).to(DEV), n_sets)
    np.testing.assert_array_equal(perm.cpu().numpy(), np.argsort(set_of, kind="stable"))
