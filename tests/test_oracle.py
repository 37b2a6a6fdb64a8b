"""Pin the CPU oracle (test infrastructure) to the reference.

Golden vectors in tests/golden/ were produced by running the reference package
itself (tests/golden/make_golden.py); the known-answer cases below restate the
reference's own unit tests (pkg/tests/test_sketch.py, test_lsh.py,
test_prefilter.py).  No GPU needed.
"""

import numpy as np
import pytest

from conftest import small_case
from oracle import c_oracle
from oracle import dessert_oracle as O


# ------------------------------------------------- known-answer tests (reference)
def test_lut_examples():  # pkg/tests/test_lsh.py:117-131
    np.testing.assert_allclose(O.sim_lut(2, 4), [0.0, 0.5, 0.70710678, 0.8660254, 1.0], atol=1e-8)
    np.testing.assert_allclose(O.sim_lut(1, 8), np.arange(9) / 8.0)
    np.testing.assert_allclose(O.sim_lut(3, 1), [0.0, 1.0])


def test_tinytable_hand_traced():  # pkg/tests/test_sketch.py:37-40
    t = O.build_tiny_table(np.array([[2], [0], [2]]), L=1, r=4)
    np.testing.assert_array_equal(t.offsets[0], [0, 1, 1, 3, 3])
    np.testing.assert_array_equal(t.ids[0], [1, 0, 2])


def test_collision_counts_hand_traced():  # pkg/tests/test_sketch.py:93-113
    codes = np.array([[2, 1], [0, 1], [2, 0]])
    t = O.build_tiny_table(codes, L=2, r=4)
    np.testing.assert_array_equal(O.accumulate_collisions_batch(t, codes[:1])[0], [2, 1, 1])
    np.testing.assert_array_equal(O.accumulate_collisions_batch(t, codes[1:2])[0], [1, 2, 0])
    np.testing.assert_array_equal(O.accumulate_collisions_batch(t, np.array([[3, 3]]))[0], [0, 0, 0])


def test_width_escalation():  # pkg/tests/test_sketch.py:58-65
    assert O.build_tiny_table(np.zeros((255, 1), int), 1, 2).offsets.dtype == np.uint8
    e = O.build_tiny_table(np.zeros((256, 1), int), 1, 2)
    assert e.offsets.dtype == np.uint16 and e.ids.dtype == np.uint8
    w = O.build_tiny_table(np.zeros((257, 1), int), 1, 2)
    assert w.ids.dtype == np.uint16


def test_sign_semantics():  # pkg/tests/test_lsh.py:62-73
    planes = np.array([[1.0, 0.0]])
    assert O.hash_matrix(planes, 1, 1, np.array([[3.0, -1.0]]))[0, 0] == 1
    assert O.hash_matrix(planes, 1, 1, np.array([[-3.0, -1.0]]))[0, 0] == 0
    P = O.sample_planes(16, 5, 10, 4)
    u = np.random.default_rng(5).standard_normal((1, 16))
    np.testing.assert_array_equal(O.hash_matrix(P, 10, 5, -u), 31 - O.hash_matrix(P, 10, 5, u))


def test_errors():
    with pytest.raises(ValueError, match="invalid parameter"):
        O.sample_planes(4, 25, 1, 0)
    with pytest.raises(ValueError, match="zero vector"):
        O.hash_matrix(O.sample_planes(3, 1, 1, 0), 1, 1, np.zeros((1, 3)))
    with pytest.raises(ValueError, match="out of range"):
        O.build_tiny_table(np.array([[4]]), L=1, r=4)
    with pytest.raises(ValueError, match="empty set"):
        O.build_tiny_table(np.zeros((0, 2), int), L=2, r=4)


# --------------------------------------------------------------- pairwise sum
@pytest.mark.parametrize("n", list(range(1, 140)) + [255, 256, 300, 1000, 4097, 9000])
def test_pairwise_sum_matches_numpy_mean(n):
    rng = np.random.default_rng(n)
    for _ in range(5):
        a = rng.random(n) ** 3
        assert O.pairwise_sum(a) / n == float(np.mean(a))
        assert c_oracle.pairwise_sum(a) == O.pairwise_sum(a)


def test_sequential_sum_is_not_numpy_order():
    """The order matters: a naive left-to-right sum disagrees often."""
    rng = np.random.default_rng(0)
    lut = O.sim_lut(6, 32)
    diff = 0
    for _ in range(2000):
        a = lut[rng.integers(0, 33, size=32)]
        seq = 0.0
        for v in a:
            seq += v
        diff += (seq / 32) != float(np.mean(a))
    assert diff > 100


# --------------------------------------------------------------- golden: lsh
def test_planes_and_hash_golden(golden_lsh):
    g = golden_lsh
    np.testing.assert_array_equal(O.sample_planes(128, 6, 32, 0), g["planes"])
    np.testing.assert_array_equal(O.sample_planes(16, 3, 5, 9), g["fam2_planes"])
    np.testing.assert_array_equal(O.hash_matrix(g["planes"], 32, 6, g["X"]), g["codes"])
    for key in g.files:
        if key.startswith("lut_"):
            _, C, L = key.split("_")
            np.testing.assert_array_equal(O.sim_lut(int(C), int(L)), g[key])


# ---------------------------------------------------- golden: scoring shapes
def test_small_golden_port_and_dense(golden_small):
    g = golden_small
    for n in range(int(g["n_shapes"])):
        c = small_case(g, n)
        r = 1 << c["C"]
        tables = [O.build_tiny_table(c["codes"][c["off"][i]:c["off"][i + 1]], c["L"], r)
                  for i in range(len(c["sizes"]))]
        for i in range(3):
            np.testing.assert_array_equal(tables[i].offsets, g[f"s{n}_tt{i}_offsets"])
            np.testing.assert_array_equal(tables[i].ids, g[f"s{n}_tt{i}_ids"])
        for q in range(c["qcodes"].shape[0]):
            qc = c["qcodes"][q]
            port = np.array([O.score_port(t, qc, c["lut"]) for t in tables])
            dense = O.score_sets_dense(qc, c["codes"], c["off"], c["lut"])
            np.testing.assert_array_equal(port, c["scores"][q])       # bit-exact
            np.testing.assert_array_equal(dense, c["scores"][q])
            mc = np.stack([O.max_counts(qc, c["codes"][c["off"][i]:c["off"][i + 1]])
                           for i in range(len(c["sizes"]))])
            np.testing.assert_array_equal(mc, c["maxcounts"][q])


def test_agg_golden_port_and_dense(golden_agg):
    """Row f3: every Scorer kind (max+weights, avg-phi x 3 phis, +-weights) bit-exact
    against the reference's _score_chunk, by the port and the dense restatement."""
    from conftest import agg_case
    from paper_2210_15748_b200 import scoring
    g = golden_agg
    names = [str(x) for x in g["scorers"]]
    assert len(names) == 7
    long_rows = 0
    for n in range(int(g["n_shapes"])):
        c = agg_case(g, n)
        r = 1 << c["C"]
        tables = [O.build_tiny_table(c["codes"][c["off"][i]:c["off"][i + 1]], c["L"], r)
                  for i in range(len(c["sizes"]))]
        for name in names:
            sc = agg_scorer_for(name, c["weights"])
            table = scoring.table_for(c["lut"], sc)
            kind = sc.inner.kind
            w = sc.weights
            want = g[f"a{n}_{name}"]
            for q in range(c["qcodes"].shape[0]):
                qc = c["qcodes"][q]
                port = np.array([O.score_port(t, qc, table, kind, w) for t in tables])
                np.testing.assert_array_equal(port, want[q], err_msg=f"{n} {name}")
                dense = O.score_sets_dense_agg(qc, c["codes"], c["off"], table, kind, w)
                np.testing.assert_array_equal(dense, want[q], err_msg=f"{n} {name}")
        # the long-row case really exercises > 128 non-zero counts per query row
        x = c["codes"][c["off"][0]:c["off"][1]]
        nz = ((c["qcodes"][0][:, None, :] == x[None, :, :]).sum(axis=2) > 0).sum(axis=1)
        long_rows += int((nz > 129).sum())
    assert long_rows > 0


def agg_scorer_for(name, weights):
    from conftest import agg_scorer
    return agg_scorer(name, weights)


def test_kmeans_golden_oracle(golden_kmeans):
    """Row f4: the oracle's train_centroids restatement equals the reference's output."""
    import kmeans_inputs as KI
    g = golden_kmeans
    for c, (n, d, k, iters, seed, _) in enumerate(KI.SPECS):
        got = O.train_centroids(KI.samples(c), k, iters, seed)
        np.testing.assert_array_equal(got, g[f"k{c}_C"], err_msg=f"case {c}")


def test_kmeans_oracle_errors():
    with pytest.raises(ValueError, match="zero vector"):
        O.train_centroids(np.zeros((3, 4)), 0, 1, 0)
    with pytest.raises(ValueError, match="k must be"):
        O.train_centroids(np.ones((3, 4)), 0, 1, 0)
    with pytest.raises(ValueError, match="too few samples"):
        O.train_centroids(np.ones((3, 4)), 4, 1, 0)
    with pytest.raises(ValueError, match="iters"):
        O.train_centroids(np.ones((3, 4)), 2, 0, 0)


def test_reduceat_restatement():
    rng = np.random.default_rng(11)
    for _ in range(500):
        n = int(rng.integers(1, 600))
        a = rng.random(n)
        cuts = np.unique(np.concatenate([[0], rng.integers(0, n, size=3)]))
        got = np.add.reduceat(a, cuts)
        b = list(cuts) + [n]
        for i in range(len(cuts)):
            assert O.reduceat_sum(a[b[i]:b[i + 1]]) == got[i]


def test_small_golden_c_oracle(golden_small):
    g = golden_small
    for n in range(int(g["n_shapes"])):
        c = small_case(g, n)
        s, mc = c_oracle.score(c["codes"], c["off"], c["qcodes"], c["lut"], want_counts=True)
        np.testing.assert_array_equal(s, c["scores"])
        np.testing.assert_array_equal(mc.astype(np.int32), c["maxcounts"])


def test_cfg0_golden_oracle(golden_cfg0):
    g = golden_cfg0
    off = np.concatenate([[0], np.cumsum(g["sizes"])])
    s, mc = c_oracle.score(g["codes"], off, g["qcodes"], g["lut"], want_counts=True)
    np.testing.assert_array_equal(s, g["scores"])
    np.testing.assert_array_equal(mc.transpose(0, 1, 2), g["maxcounts"])
    for q in range(g["qcodes"].shape[0]):
        top = O.rank_topk(s[q], np.arange(len(g["sizes"])), 10)
        assert [d for d, _ in top] == list(g["top_ids"][q])
        assert [v for _, v in top] == list(g["top_scores"][q])
    # the cfg0 generator reproduces the reference's codes
    from paper_2210_15748_b200 import workloads
    sizes, X, Q = workloads.cfg0_data(0)
    np.testing.assert_array_equal(sizes, g["sizes"])
    P = O.sample_planes(128, 6, 32, 0)
    np.testing.assert_array_equal(P[:8], g["planes_head"])
    np.testing.assert_array_equal(O.hash_matrix(P, 32, 6, X[:5000]), g["codes"][:5000])
    np.testing.assert_array_equal(O.hash_matrix(P, 32, 6, Q[3]), g["qcodes"][3])


def test_end_to_end_golden_oracle(golden_e2e):
    g = golden_e2e
    for n in range(int(g["n_cases"])):
        d, C, L, seed, top_k = (int(x) for x in g[f"e{n}_shape"])
        sizes = g[f"e{n}_sizes"]
        off = np.concatenate([[0], np.cumsum(sizes)])
        P = O.sample_planes(d, C, L, seed)
        codes = O.hash_matrix(P, L, C, g[f"e{n}_X"])
        np.testing.assert_array_equal(codes, g[f"e{n}_codes"])
        lut = O.sim_lut(C, L)
        for q in range(2):
            qc = O.hash_matrix(P, L, C, g[f"e{n}_Q"][q])
            s = O.score_sets_dense(qc, codes, off, lut)
            top = O.rank_topk(s, g[f"e{n}_ids"], top_k)
            assert [x for x, _ in top] == list(g[f"e{n}_top_ids"][q])
            assert [v for _, v in top] == list(g[f"e{n}_top_scores"][q])


# ----------------------------------------------------------- golden: prefilter
def test_prefilter_golden_oracle(golden_prefilter):
    g = golden_prefilter
    sizes = g["doc_sizes"]
    off = np.concatenate([[0], np.cumsum(sizes)])
    docs = [g["docs"][off[i]:off[i + 1]] for i in range(len(sizes))]
    post = O.build_centroid_index(docs, g["centroids"])
    po = g["post_off"]
    for c in range(len(po) - 1):
        np.testing.assert_array_equal(post[c], g["post_docs"][po[c]:po[c + 1]])
    for t, (probe, kf) in enumerate(g["cases"]):
        got = O.filter_candidates(post, len(sizes), g["centroids"], g[f"q{t}"], int(probe), int(kf))
        np.testing.assert_array_equal(got, g[f"r{t}"])
