"""TinyTable accessors: bucket, accumulate_collisions(_batch).

Restates pkg/tests/test_sketch.py:74-145 (hand-traced buckets, known collision
counts, reusable buffers, batch == single rows, random instances against a naive
map-of-lists).  bucket() and argument validation are host-only; the counts run
on the device (dsrt_collision_counts) and are marked gpu.
"""

import numpy as np
import pytest

import paper_2210_15748_b200 as d
from oracle import dessert_oracle as O


def _table(codes, L, r):
    """A TinyTable built by the oracle's counting sort (host, test-only)."""
    t = O.build_tiny_table(np.asarray(codes), L, r)
    return d.TinyTable(m=t.m, L=t.L, r=t.r, offsets=t.offsets, ids=t.ids)


def _naive_counts(codes, query):
    codes = np.asarray(codes)
    return np.array([sum(int(codes[j, t]) == int(query[t]) for t in range(codes.shape[1]))
                     for j in range(codes.shape[0])])


def test_bucket_hand_traced():
    table = _table([[2], [0], [2]], 1, 4)
    np.testing.assert_array_equal(d.bucket(table, 0, 2), [0, 2])
    np.testing.assert_array_equal(d.bucket(table, 0, 1), [])
    with pytest.raises(IndexError):
        d.bucket(table, 0, 4)
    with pytest.raises(IndexError):
        d.bucket(table, 1, 0)
    assert d.bucket(_table([[1], [1], [1]], 1, 2), 0, 1).base is not None


def test_bucket_random_against_naive_map():
    rng = np.random.default_rng(2)
    for _ in range(20):
        m, L, r = int(rng.integers(1, 120)), int(rng.integers(1, 16)), 1 << int(rng.integers(1, 7))
        codes = rng.integers(0, r, size=(m, L))
        table = _table(codes, L, r)
        for t in range(L):
            for h in range(r):
                np.testing.assert_array_equal(d.bucket(table, t, h), np.flatnonzero(codes[:, t] == h))


def test_accumulate_validation_is_host_side():
    table = _table([[2], [0]], 1, 4)
    with pytest.raises(ValueError, match="out of range"):
        d.accumulate_collisions(table, np.array([4]))
    with pytest.raises(ValueError, match="expected 1 query codes"):
        d.accumulate_collisions(table, np.array([1, 2]))
    with pytest.raises(ValueError, match=r"expected \(m_q, 1\) code matrix"):
        d.accumulate_collisions_batch(table, np.array([1, 2]))
    with pytest.raises(ValueError, match="out of range"):
        d.accumulate_collisions_batch(table, np.array([[1], [-1]]))


# ------------------------------------------------------------------ GPU
@pytest.mark.gpu
def test_accumulate_known_answers():
    codes = np.array([[2, 1], [0, 1], [2, 0]])
    table = d.build_tiny_table(codes, L=2, r=4)
    np.testing.assert_array_equal(d.accumulate_collisions(table, codes[0]), [2, 1, 1])
    np.testing.assert_array_equal(d.accumulate_collisions(table, np.array([3, 3])), [0, 0, 0])
    buf = np.full(10, 99, dtype=np.int32)
    out = d.accumulate_collisions(table, codes[1], out=buf)
    np.testing.assert_array_equal(out, [1, 2, 0])
    assert out.base is buf
    np.testing.assert_array_equal(buf[3:], 99)


@pytest.mark.gpu
def test_accumulate_batch_matches_single_and_naive():
    rng = np.random.default_rng(1)
    for m, L, r, m_q in [(19, 6, 8, 7), (300, 64, 128, 40), (1, 3, 2, 5), (257, 16, 16, 33)]:
        codes = rng.integers(0, r, size=(m, L))
        table = d.build_tiny_table(codes, L=L, r=r)
        queries = rng.integers(0, r, size=(m_q, L))
        queries[0] = codes[0]  # one row with a guaranteed full collision
        batch = d.accumulate_collisions_batch(table, queries)
        assert batch.shape == (m_q, m) and batch.dtype == np.int32
        for q in range(m_q):
            want = _naive_counts(codes, queries[q])
            np.testing.assert_array_equal(batch[q], want)
            np.testing.assert_array_equal(d.accumulate_collisions(table, queries[q]), want)
        buf = np.full((m_q + 2, m + 3), -7, dtype=np.int32)
        got = d.accumulate_collisions_batch(table, queries, out=buf)
        np.testing.assert_array_equal(got, batch)
        assert got.base is buf and (buf[m_q:] == -7).all() and (buf[:, m:] == -7).all()


@pytest.mark.gpu
def test_accumulate_on_index_sketches():
    """pkg/tests/test_index.py:136-145: the counts behind a set's score come from
    the set's own sketch."""
    rng = np.random.default_rng(5)
    docs = [(i, rng.standard_normal((int(rng.integers(1, 30)), 16))) for i in range(6)]
    idx = d.build_index(docs, d.IndexConfig(d=16, C=3, L=12, seed=1,
                                            filter=d.FilterConfig(enabled=False)))
    Q = rng.standard_normal((4, 16))
    qc = d.hash_matrix(idx.family, Q)
    for i, (_, X) in enumerate(docs):
        xc = d.hash_matrix(idx.family, X)
        got = d.accumulate_collisions_batch(idx.sketches[i], qc)
        for q in range(Q.shape[0]):
            np.testing.assert_array_equal(got[q], _naive_counts(xc, qc[q]))
