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


# ---------------------------------------------- scoring descriptors (f3)
# behaviour of pkg/tests/test_scoring.py, restated


def test_sigma_max_and_bounds():
    assert d.sigma_max([0.2, 0.9, 0.5]) == pytest.approx(0.9)
    with pytest.raises(ValueError, match="empty"):
        d.sigma_max([])
    agg = d.max_aggregation()
    assert (agg.alpha, agg.beta, agg.beta_for(17)) == (1.0, 1.0, 1.0)


def test_sigma_avg_phi_kinds():
    assert d.sigma_avg_phi([0.5, 0.1], "identity") == pytest.approx(0.3)
    v = d.sigma_avg_phi([1.0, 1.0], "exp-minus-one")
    assert v == pytest.approx(np.e - 1.0)
    agg = d.avg_phi_aggregation("exp-minus-one")
    assert agg.beta_for(2) - 1e-12 <= v <= agg.alpha + 1e-12
    assert d.sigma_avg_phi([0.0, 0.0, 0.0], "debiased-sigmoid") == pytest.approx(0.0)
    ds = d.avg_phi_aggregation("debiased-sigmoid")
    assert ds.alpha == pytest.approx(0.25)
    assert ds.beta == pytest.approx(1.0 / (1.0 + np.exp(-1.0)) - 0.5, abs=1e-6)
    with pytest.raises(ValueError, match="range"):
        d.sigma_avg_phi([0.5, 1.2], "identity")
    with pytest.raises(ValueError, match="empty"):
        d.sigma_avg_phi([], "identity")
    with pytest.raises(ValueError, match="phi"):
        d.sigma_avg_phi([0.5], "cubic")
    with pytest.raises(ValueError, match="phi"):
        d.avg_phi_aggregation("cubic")


def test_outer_aggregate():
    assert d.outer_aggregate([0.4, 0.8], [1, 1]) == pytest.approx(0.6)
    assert d.outer_aggregate([0.4, 0.8], [0, 1]) == pytest.approx(0.4)
    with pytest.raises(ValueError, match="mismatch"):
        d.outer_aggregate([0.4, 0.8], [1.0])
    with pytest.raises(ValueError, match="range"):
        d.outer_aggregate([0.5], [1.5])


def test_maximality_sandwich():
    rng = np.random.default_rng(0)
    for agg in [d.max_aggregation()] + [d.avg_phi_aggregation(p) for p in d.PHI_KINDS]:
        for _ in range(100):
            m = int(rng.integers(1, 65))
            x = rng.uniform(0.0, 1.0, size=m)
            got = agg.apply(x)
            assert agg.beta_for(m) * x.max() - 1e-12 <= got <= agg.alpha * x.max() + 1e-12
            np.testing.assert_allclose(agg.apply_rows(x[None, :])[0], got, rtol=1e-15)


def test_score_plan_resolution():
    from paper_2210_15748_b200 import scoring
    assert scoring.is_default(None) and scoring.is_default(d.default_scorer())
    s = d.Scorer(inner=d.avg_phi_aggregation("identity"))
    assert not scoring.is_default(s) and scoring.inner_kind_code(s) == 1
    lut = np.linspace(0.0, 1.0, 9)
    np.testing.assert_array_equal(scoring.table_for(lut, s), lut)
    e = d.Scorer(inner=d.avg_phi_aggregation("exp-minus-one"))
    np.testing.assert_array_equal(scoring.table_for(lut, e), np.expm1(lut))
    with pytest.raises(ValueError, match="mismatch"):
        scoring.resolve_weights(d.Scorer(d.max_aggregation(), np.ones(3)), 4)
    with pytest.raises(ValueError, match="range"):
        scoring.resolve_weights(d.Scorer(d.max_aggregation(), np.full(4, 2.0)), 4)
    cfg = d.IndexConfig(d=8, inner_kind="avg-phi", phi="debiased-sigmoid")
    assert cfg.scorer().inner == d.avg_phi_aggregation("debiased-sigmoid")
