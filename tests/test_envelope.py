"""The reference's full parameter envelope (golden fixture envelope.npz, generated
by running the reference: tests/golden/make_golden.py envelope).

* scoring shapes outside the register-blocked K3 kernels: C up to 24 and L > 128
  (lsh.py:17, 54-66) -- the general kernel K3g takes them, bit-exact;
* vectors -> build_index -> query at such shapes (index.py:131-167, 264-319);
* the prefilter with probe > 32 and k_filter > 16384 (prefilter.py:111-144).

CPU tests pin the oracle on the fixture; GPU tests run the product path.
"""

import os

import numpy as np
import pytest
import torch

from oracle import dessert_oracle as O

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "envelope.npz")


@pytest.fixture(scope="module")
def g():
    return np.load(GOLDEN, allow_pickle=False)


def _case(g, n):
    L, C, m_q = (int(x) for x in g[f"s{n}_shape"])
    sizes = g[f"s{n}_sizes"].astype(np.int64)
    return dict(L=L, C=C, m_q=m_q, sizes=sizes, off=np.concatenate([[0], np.cumsum(sizes)]),
                codes=g[f"s{n}_codes"], qcodes=g[f"s{n}_qcodes"], doc_ids=g[f"s{n}_doc_ids"],
                scores=g[f"s{n}_scores"])


def _postings(g):
    po, pd = g["pf_post_off"], g["pf_post_docs"]
    return [pd[po[c]:po[c + 1]] for c in range(len(po) - 1)]


# --------------------------------------------------------------------- CPU
def test_envelope_oracle_scores(g):
    for n in range(int(g["n_shapes"])):
        c = _case(g, n)
        for q in range(c["qcodes"].shape[0]):
            lut = O.sim_lut(c["C"], c["L"])
            dense = O.score_sets_dense(c["qcodes"][q], c["codes"], c["off"], lut)
            np.testing.assert_array_equal(dense, c["scores"][q], err_msg=f"shape {n}")


def test_envelope_oracle_prefilter(g):
    post = _postings(g)
    for t, (probe, kf) in enumerate(g["pf_cases"]):
        got = O.filter_candidates(post, int(g["pf_n_docs"]), g["pf_centroids"], g[f"pf_q{t}"],
                                  int(probe), int(kf))
        np.testing.assert_array_equal(got, g[f"pf_r{t}"], err_msg=f"case {t}")


# --------------------------------------------------------------------- GPU
@pytest.mark.gpu
def test_envelope_scores_gpu(g):
    import paper_2210_15748_b200 as d

    dev = torch.device("cuda")
    for n in range(int(g["n_shapes"])):
        c = _case(g, n)
        cfg = d.IndexConfig(d=4, C=c["C"], L=c["L"], filter=d.FilterConfig(enabled=False))
        cd = torch.from_numpy(np.ascontiguousarray(c["codes"]).astype(np.int32)).to(dev)
        idx = d.build_from_codes(cd, c["sizes"], c["doc_ids"], cfg)
        s, _ = d.score_matrix(idx, c["qcodes"])  # < 8 query sets: candidate windows
        np.testing.assert_array_equal(s.cpu().numpy(), c["scores"], err_msg=f"shape {n}")
        s8, _ = d.score_matrix(idx, np.concatenate([c["qcodes"]] * 3))  # exhaustive ranges
        np.testing.assert_array_equal(s8.cpu().numpy(), np.concatenate([c["scores"]] * 3))
        sets = np.stack([np.random.default_rng(n).permutation(len(c["sizes"]))] * 3)
        sc, _ = d.score_matrix(idx, c["qcodes"], sets=sets)
        np.testing.assert_array_equal(sc.cpu().numpy(), np.take_along_axis(c["scores"], sets, axis=1))
        for q in range(3):
            assert d.score_candidate(idx, int(sets[0, q]), c["qcodes"][q]) == c["scores"][q, sets[0, q]]
            got = d.query_codes_batch(idx, c["qcodes"][q:q + 1], 5)[0]
            assert got == O.rank_topk(c["scores"][q], c["doc_ids"], 5)


@pytest.mark.gpu
def test_envelope_end_to_end_gpu(g):
    import paper_2210_15748_b200 as d

    for n in range(2):
        dd, C, L, seed, top_k = (int(x) for x in g[f"e{n}_shape"])
        sizes = g[f"e{n}_sizes"]
        off = np.concatenate([[0], np.cumsum(sizes)])
        X, ids = g[f"e{n}_X"], g[f"e{n}_ids"]
        docs = [(int(ids[i]), X[off[i]:off[i + 1]]) for i in range(len(sizes))]
        idx = d.build_index(docs, d.IndexConfig(d=dd, C=C, L=L, seed=seed,
                                                filter=d.FilterConfig(enabled=False)))
        for q in range(2):
            r = d.query(idx, g[f"e{n}_Q"][q], top_k=top_k)
            assert [x for x, _ in r] == list(g[f"e{n}_top_ids"][q]), (n, q)
            assert [v for _, v in r] == list(g[f"e{n}_top_scores"][q]), (n, q)


@pytest.mark.gpu
def test_envelope_prefilter_gpu(g):
    import paper_2210_15748_b200 as d
    from paper_2210_15748_b200 import prefilter

    dev = torch.device("cuda")
    cents = d.Centroids(k=g["pf_centroids"].shape[0], seed=5, vectors=g["pf_centroids"])
    cindex = prefilter.CentroidIndex(n_docs=int(g["pf_n_docs"]),
                                     post_off=torch.from_numpy(g["pf_post_off"]).to(dev),
                                     post_docs=torch.from_numpy(g["pf_post_docs"]).to(dev))
    for t, (probe, kf) in enumerate(g["pf_cases"]):
        got = d.filter_candidates(cindex, cents, g[f"pf_q{t}"], int(probe), int(kf))
        np.testing.assert_array_equal(got, g[f"pf_r{t}"], err_msg=f"case {t}")
