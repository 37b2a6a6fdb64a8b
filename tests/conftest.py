import os
import sys

import numpy as np
import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if REPO not in sys.path:
    sys.path.insert(0, REPO)
GOLDEN = os.path.join(REPO, "tests", "golden")
if GOLDEN not in sys.path:
    sys.path.insert(0, GOLDEN)  # kmeans_inputs (seeded golden inputs)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")


def pytest_collection_modifyitems(config, items):
    # GPU tests must fail loudly (not skip) when selected without a GPU.
    pass


def load_golden(name):
    return np.load(os.path.join(GOLDEN, name), allow_pickle=False)


@pytest.fixture(scope="session")
def golden_small():
    return load_golden("small.npz")


@pytest.fixture(scope="session")
def golden_cfg0():
    return load_golden("cfg0.npz")


@pytest.fixture(scope="session")
def golden_lsh():
    return load_golden("lsh.npz")


@pytest.fixture(scope="session")
def golden_prefilter():
    return load_golden("prefilter.npz")


@pytest.fixture(scope="session")
def golden_e2e():
    return load_golden("end_to_end.npz")


@pytest.fixture(scope="session")
def golden_kmeans():
    return load_golden("kmeans.npz")


@pytest.fixture(scope="session")
def golden_agg():
    return load_golden("agg.npz")


def agg_case(g, n):
    L, C, m_q = (int(x) for x in g[f"a{n}_shape"])
    sizes = g[f"a{n}_sizes"].astype(np.int64)
    return dict(L=L, C=C, m_q=m_q, sizes=sizes,
                off=np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64),
                codes=g[f"a{n}_codes"], qcodes=g[f"a{n}_qcodes"], weights=g[f"a{n}_weights"],
                lut=g[f"a{n}_lut"])


def agg_scorer(name, weights):
    """Scorer for a golden scorer name: max_w, <phi>, <phi>_w."""
    import paper_2210_15748_b200 as d
    base, _, wt = name.rpartition("_") if name.endswith("_w") else (name, "", "")
    inner = d.max_aggregation() if base == "max" else d.avg_phi_aggregation(base)
    return d.Scorer(inner=inner, weights=weights if wt == "w" else None)


def small_case(g, n):
    L, C, m_q = (int(x) for x in g[f"s{n}_shape"])
    sizes = g[f"s{n}_sizes"].astype(np.int64)
    return dict(L=L, C=C, m_q=m_q, sizes=sizes,
                off=np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64),
                codes=g[f"s{n}_codes"], qcodes=g[f"s{n}_qcodes"], doc_ids=g[f"s{n}_doc_ids"],
                scores=g[f"s{n}_scores"], maxcounts=g[f"s{n}_maxcounts"], lut=g[f"s{n}_lut"])
