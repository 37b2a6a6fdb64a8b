"""Differential fuzz: random small collections through the public API of this
package and of the UNMODIFIED reference (baseline/_ref), results required to be
identical (doc ids and float64 scores with ==, or the same exception type).

  python tools/fuzz_vs_reference.py [--cases 300] [--seed 0] [--verbose]

Covers build_index -> query / query_batch / score_candidate / add_sets with
random d, C, L, set sizes, m_q, top_k, scorers (max / avg-phi, weights),
prefilter settings, float32/float64 inputs and large uint64 doc ids.  Test
infrastructure (like oracle/): needs a GPU and baseline/_ref.
"""
import argparse
import hashlib
import os
import sys
import tempfile
import time
import traceback

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
sys.path.insert(0, os.path.join(REPO, "baseline", "_ref"))

import dessert as ref  # noqa: E402  (the reference package)

import paper_2210_15748_b200 as d  # noqa: E402

PHI = ["identity", "exp-minus-one", "debiased-sigmoid"]


def unit(x):
    n = np.linalg.norm(x, axis=1, keepdims=True)
    n[n == 0] = 1.0
    return x / n


def make_case(seed):
    rng = np.random.default_rng([seed, 0xF022])
    big = rng.random() < 0.15
    dim = int(rng.choice([2, 3, 8, 16, 31, 64, 100, 128, 130, 200]))
    C = int(rng.integers(1, 13)) if rng.random() < 0.9 else int(rng.integers(13, 17))
    L = int(rng.integers(1, 65)) if rng.random() < 0.8 else int(rng.integers(65, 201))
    if C > 12:
        L = min(L, 8)
    n_sets = int(rng.integers(1, 12)) if C > 12 else int(rng.integers(1, 300 if big else 80))
    if C <= 8 and L <= 64 and rng.random() < 0.04:
        n_sets = int(rng.integers(1000, 6000))  # several score chunks / prefilter chunks
    hi = 300 if (big and rng.random() < 0.3) else 40
    sizes = rng.integers(1, hi + 1, size=n_sets)
    dtype = np.float32 if rng.random() < 0.5 else np.float64
    # clustered data so the prefilter and the scores have structure
    n_cent = int(rng.integers(1, 20))
    cents = unit(rng.standard_normal((n_cent, dim)))
    docs = []
    ids = rng.choice(np.arange(1, 10 * n_sets + 10), size=n_sets, replace=False).astype(np.uint64)
    if rng.random() < 0.2:
        ids = ids + np.uint64(1 << 63)
    for i in range(n_sets):
        c = cents[rng.integers(0, n_cent, size=sizes[i])]
        X = unit(c + 0.3 * rng.standard_normal((sizes[i], dim))).astype(dtype)
        docs.append((int(ids[i]), X))
    m_q = int(rng.integers(1, 41)) if rng.random() < 0.9 else int(rng.integers(129, 260))
    nq = int(rng.integers(1, 5))
    Qs = []
    for _ in range(nq):
        src = docs[rng.integers(0, n_sets)][1]
        q = src[rng.integers(0, src.shape[0], size=m_q)] + 0.1 * rng.standard_normal((m_q, dim))
        Qs.append(unit(q).astype(dtype))
    inner = "max" if rng.random() < 0.6 else "avg-phi"
    phi = None if inner == "max" else str(rng.choice(PHI))
    weights = None
    if rng.random() < 0.3:
        weights = rng.random(m_q)
        if rng.random() < 0.3:
            weights[rng.integers(0, m_q)] = 0.0
    filt_on = rng.random() < 0.5
    total = int(sizes.sum())
    fc = dict(enabled=filt_on,
              centroids=0 if rng.random() < 0.4 else int(rng.integers(1, min(64, total) + 1)),
              iters=int(rng.integers(1, 5)), probe=int(rng.integers(1, 7)),
              k_filter=int(rng.integers(1, n_sets + 10)))
    top_k = int(rng.integers(1, n_sets + 6))
    q_probe = None if rng.random() < 0.6 else int(rng.integers(1, 40))
    q_kf = None if rng.random() < 0.6 else int(rng.integers(1, 2 * n_sets + 2))
    return dict(seed=seed, d=dim, C=C, L=L, docs=docs, Qs=Qs, m_q=m_q, inner=inner, phi=phi,
                weights=weights, filter=fc, top_k=top_k, probe=q_probe, k_filter=q_kf,
                cfg_seed=int(rng.integers(0, 1000)), add_split=int(rng.integers(0, n_sets + 1)),
                cand_ix=rng.integers(0, n_sets, size=min(3, n_sets)))


def run_side(mod, case, ours):
    """Everything the case asks of one implementation -> a comparable structure."""
    out = {}
    cfg = mod.IndexConfig(d=case["d"], C=case["C"], L=case["L"], seed=case["cfg_seed"],
                          inner_kind=case["inner"], phi=case["phi"],
                          filter=mod.FilterConfig(**case["filter"]))
    idx = mod.build_index(case["docs"], cfg)
    scorer = None
    if case["weights"] is not None:
        inner = mod.max_aggregation() if case["inner"] == "max" else mod.avg_phi_aggregation(case["phi"])
        scorer = mod.Scorer(inner=inner, weights=case["weights"])
    kw = dict(probe=case["probe"], k_filter=case["k_filter"], scorer=scorer)
    out["query"] = [mod.query(idx, Q, case["top_k"], **kw) for Q in case["Qs"]]
    fam = idx.family
    qc = mod.hash_matrix(fam, case["Qs"][0])
    out["codes"] = np.asarray(qc).astype(np.int64).tolist()
    out["cand"] = [float(mod.score_candidate(idx, int(i), qc, scorer=scorer)) for i in case["cand_ix"]]
    # index file bytes (C <= 12: the device writer's envelope) and a load -> query round trip
    if case["C"] <= 12:
        with tempfile.TemporaryDirectory() as td:
            path = os.path.join(td, "x.dsri")
            mod.save_index(path, idx)
            blob = open(path, "rb").read()
            out["file"] = hashlib.sha256(blob).hexdigest()
            idx2 = mod.load_index(path)
            out["loaded"] = mod.query(idx2, case["Qs"][0], case["top_k"], **kw)
    # the prefilter entry points on their own
    if idx.filter is not None:
        cents, cindex = idx.filter
        fc = mod.filter_candidates(cindex, cents, case["Qs"][0], case["filter"]["probe"], case["filter"]["k_filter"])
        out["filter_candidates"] = np.asarray(fc).astype(np.int64).tolist()
        out["centroids"] = hashlib.sha256(np.ascontiguousarray(np.asarray(cents.vectors, dtype=np.float64)).tobytes()).hexdigest()
    if ours:
        out["batch"] = mod.query_batch(idx, np.stack(case["Qs"]), case["top_k"], **kw)
        # add-set path: build the first part, add the rest; the scoring side must equal a full build
        k = case["add_split"]
        if 0 < k < len(case["docs"]) and not case["filter"]["enabled"]:
            part = mod.build_index(case["docs"][:k], cfg)
            part = mod.add_sets(part, case["docs"][k:])
            out["added"] = [mod.query(part, Q, case["top_k"], **kw) for Q in case["Qs"]]
    return out


def compare(case, a, b):
    errs = []
    if a["codes"] != b["codes"]:
        errs.append("query codes differ")
    if a["query"] != b["query"]:
        errs.append(f"query results differ: ref {a['query'][0][:3]} ours {b['query'][0][:3]}")
    for key in ("file", "loaded", "filter_candidates", "centroids"):
        if a.get(key) != b.get(key):
            errs.append(f"{key} differs")
    if a["cand"] != b["cand"]:
        errs.append(f"score_candidate differs: ref {a['cand']} ours {b['cand']}")
    if b.get("batch") is not None and b["batch"] != a["query"]:
        errs.append("query_batch differs from per-query reference results")
    if b.get("added") is not None and b["added"] != a["query"]:
        errs.append("add_sets index differs from the reference's full build")
    return errs


def make_case_fp16(seed):
    """d = 128, C <= 8, >= 4096 fp16 vectors: build_index hashes them on the tcgen05 hi/lo
    path, whose bits may differ from float64 inside the 1e-4 band only."""
    rng = np.random.default_rng([seed, 0xF16])
    if True:
        case = make_case(int(rng.integers(0, 1 << 30)))
        rs = np.random.default_rng([seed, 1])
        n_sets = int(rs.integers(210, 400))  # x >= 20 vectors: at least 4096 rows -> tcgen05 hash
        sizes = rs.integers(20, 60, size=n_sets)
        cents = unit(rs.standard_normal((int(rs.integers(2, 30)), 128)))
        ids = rs.choice(np.arange(1, 10 * n_sets), size=n_sets, replace=False)
        docs = []
        for i in range(n_sets):
            c = cents[rs.integers(0, cents.shape[0], size=sizes[i])]
            docs.append((int(ids[i]), unit(c + 0.3 * rs.standard_normal((sizes[i], 128))).astype(np.float16)))
        m_q = int(rs.integers(1, 41))
        Qs = []
        for _ in range(int(rs.integers(1, 4))):
            src = docs[rs.integers(0, n_sets)][1].astype(np.float64)
            q = src[rs.integers(0, src.shape[0], size=m_q)] + 0.1 * rs.standard_normal((m_q, 128))
            Qs.append(unit(q).astype(np.float16))
        case.update(d=128, C=int(rs.integers(1, 9)), L=int(rs.integers(1, 129)), docs=docs, Qs=Qs, m_q=m_q,
                    top_k=int(rs.integers(1, n_sets + 5)), cand_ix=rs.integers(0, n_sets, size=3),
                    add_split=0)
        if case["weights"] is not None:
            case["weights"] = rs.random(m_q)
        case["filter"]["k_filter"] = int(rs.integers(1, n_sets + 10))
        case["filter"]["centroids"] = 0 if rs.random() < 0.4 else int(rs.integers(1, 65))
    return case


def run_fp16_case(case):
    """Ours first (tensor-core hash of the fp16 documents); then the reference built on OUR
    codes (its hash_matrix patched for the build only) -- identical codes in, identical
    scores, rankings, file bytes and prefilter out.  Also counts the bits that differ from
    the reference's own float64 hash (they must sit inside the band; tests assert that)."""
    import dessert.index as ref_index

    rb = run_side(d, case, True)
    cfg = d.IndexConfig(d=128, C=case["C"], L=case["L"], seed=case["cfg_seed"], inner_kind=case["inner"],
                        phi=case["phi"], filter=d.FilterConfig(**case["filter"]))
    idx = d.build_index(case["docs"], cfg)
    codes = idx.codes.cpu().numpy().astype(np.int64)
    off = np.concatenate([[0], np.cumsum([X.shape[0] for _, X in case["docs"]])])
    queue = [codes[off[i]:off[i + 1]] for i in range(len(case["docs"]))]
    orig = ref_index.hash_matrix
    flips = 0

    def patched(fam, X):
        nonlocal flips
        if queue:
            mine = queue.pop(0)
            flips += int(np.count_nonzero(np.asarray(orig(fam, X)) != mine))
            return mine
        return orig(fam, X)

    ref_index.hash_matrix = patched
    try:
        ra = run_side(ref, case, False)
    finally:
        ref_index.hash_matrix = orig
    return ra, rb, flips


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cases", type=int, default=300)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--verbose", action="store_true")
    ap.add_argument("--fp16", action="store_true",
                    help="fp16 collections hashed on the tensor-core path; the reference is built on our codes")
    a = ap.parse_args()
    if a.fp16:
        return main_fp16(a)
    bad = 0
    t0 = time.time()
    for s in range(a.seed, a.seed + a.cases):
        case = make_case(s)
        desc = (f"seed={s} d={case['d']} C={case['C']} L={case['L']} sets={len(case['docs'])} "
                f"m_q={case['m_q']} inner={case['inner']}/{case['phi']} w={case['weights'] is not None} "
                f"filter={case['filter']} top_k={case['top_k']} probe={case['probe']} kf={case['k_filter']}")
        try:
            ra, ea = run_side(ref, case, False), None
        except Exception as e:  # noqa: BLE001
            ra, ea = None, e
        try:
            rb, eb = run_side(d, case, True), None
        except Exception as e:  # noqa: BLE001
            rb, eb = None, e
            tb = traceback.format_exc()
        if ea is not None or eb is not None:
            if type(ea) is type(eb) and str(ea) == str(eb):
                if a.verbose:
                    print("same error:", desc, "|", ea)
                continue
            bad += 1
            print("MISMATCH (exception):", desc, "| ref:", repr(ea), "| ours:", repr(eb))
            if eb is not None and ea is None:
                print(tb)
            continue
        errs = compare(case, ra, rb)
        if errs:
            bad += 1
            print("MISMATCH:", desc, "|", "; ".join(errs))
        elif a.verbose:
            print("ok:", desc)
    print(f"fuzz: {a.cases} cases, {bad} mismatches, {time.time() - t0:.0f} s")
    return 1 if bad else 0


def main_fp16(a):
    bad = flips = 0
    t0 = time.time()
    for s in range(a.seed, a.seed + a.cases):
        case = make_case_fp16(s)
        desc = (f"seed={s} C={case['C']} L={case['L']} sets={len(case['docs'])} m_q={case['m_q']} "
                f"inner={case['inner']}/{case['phi']} filter={case['filter']} top_k={case['top_k']}")
        try:
            ra, rb, f = run_fp16_case(case)
        except Exception:  # noqa: BLE001
            bad += 1
            print("MISMATCH (exception):", desc)
            print(traceback.format_exc())
            continue
        flips += f
        errs = compare(case, ra, rb)
        if errs:
            bad += 1
            print("MISMATCH:", desc, "|", "; ".join(errs))
        elif a.verbose:
            print("ok:", desc, "flipped code entries:", f)
    print(f"fuzz fp16: {a.cases} cases, {bad} mismatches, {flips} code entries differ from the float64 hash, "
          f"{time.time() - t0:.0f} s")
    return 1 if bad else 0


if __name__ == "__main__":
    sys.exit(main())
