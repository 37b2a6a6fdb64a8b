"""Host-side API semantics that need no GPU: configs, profiles, validation order."""

import numpy as np
import pytest

import paper_2210_15748_b200 as d


def test_profiles_match_reference():  # pkg/tests/test_index.py:67-83
    assert set(d.PROFILES) == {"msmarco-k10-fast", "msmarco-k10-slow", "msmarco-k1000-fast",
                               "msmarco-k1000-slow"}
    cfg = d.apply_profile(d.IndexConfig(d=16), "msmarco-k10-fast")
    assert (cfg.C, cfg.L) == (7, 32)
    assert (cfg.filter.probe, cfg.filter.k_filter) == (1, 4096)
    with pytest.raises(ValueError, match="profile"):
        d.apply_profile(d.IndexConfig(d=16), "nope")


def test_config_defaults_match_reference():  # index.py:35-62
    c = d.IndexConfig(d=8)
    assert (c.C, c.L, c.seed, c.inner_kind, c.phi) == (7, 32, 0, "max", None)
    assert c.filter == d.FilterConfig(enabled=True, centroids=0, iters=10, probe=1, k_filter=4096)
    assert c.code_range == 128


def test_build_validation_errors_before_device_work():  # pkg/tests/test_index.py:41-65
    nf = dict(filter=d.FilterConfig(enabled=False))
    with pytest.raises(ValueError, match="empty collection"):
        d.build_index([], d.IndexConfig(d=4, **nf))
    with pytest.raises(ValueError, match="empty set"):
        d.build_index([(0, np.ones((0, 4)))], d.IndexConfig(d=4, **nf))
    with pytest.raises(ValueError, match="dimension"):
        d.build_index([(0, np.ones((2, 4))), (1, np.ones((2, 5)))], d.IndexConfig(d=4, **nf))
    with pytest.raises(ValueError, match="duplicate"):
        d.build_index([(3, np.ones((1, 2))), (3, np.ones((1, 2)))], d.IndexConfig(d=2, **nf))


def test_family_and_lut_are_reference_bytes(golden_lsh):
    fam = d.sample_srp_family(128, 6, 32, 0)
    np.testing.assert_array_equal(fam.planes, golden_lsh["planes"])
    for C in (1, 2, 3, 6, 7, 8, 12, 24):
        for L in (1, 4, 8, 16, 32, 33, 64, 128):
            np.testing.assert_array_equal(d.build_sim_lookup(C, L).table,
                                          golden_lsh[f"lut_{C}_{L}"])
    with pytest.raises(ValueError, match="invalid parameter"):
        d.sample_srp_family(4, 25, 1, 0)
    with pytest.raises(ValueError):
        d.sample_srp_family(0, 1, 1, 0)


def test_tiny_table_bytes():  # pkg/tests/test_sketch.py:149-155
    assert d.tiny_table_bytes(m=100, r=128, L=64) == 14_680
    assert d.tiny_table_bytes(m=1, r=2, L=1) == 28


def test_unsupported_scorer_is_loud():
    from paper_2210_15748_b200.scoring import InnerAggregation, Scorer, require_device_scorer
    with pytest.raises(NotImplementedError):
        require_device_scorer(Scorer(inner=InnerAggregation("avg", 1, 1, "identity")))
    require_device_scorer(d.default_scorer())
