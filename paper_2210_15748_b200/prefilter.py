"""Centroid prefilter -- drop-in for dessert.prefilter (reference: pkg/src/dessert/prefilter.py).

``filter_candidates`` (prefilter.py:111-144) runs on the GPU (K5,
csrc/prefilter.cu).  Centroid training (prefilter.py:47-82, row f4) is K7
(csrc/kmeans.cu) and the centroid->document postings (prefilter.py:85-108,
row f1) are K6 (csrc/prefilter.cu assignment + csrc/postings.cu radix
postings): native kernels following the reference's algorithm and tie rules
step by step; torch tensors are only the buffers.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch

from . import engine

MAX_TRAIN_SAMPLES = 1 << 20


@dataclass(frozen=True)
class Centroids:
    """k unit-norm centroid directions (prefilter.py:20-26)."""

    k: int
    seed: int
    vectors: np.ndarray
    _dev: dict = field(default_factory=dict, repr=False, compare=False)

    def device_vectors(self, device) -> torch.Tensor:
        key = str(device)
        t = self._dev.get(key)
        if t is None:
            t = torch.from_numpy(np.ascontiguousarray(self.vectors, dtype=np.float64)).to(device)
            self._dev[key] = t
        return t

    def device_lowp(self, device, bf16: bool):
        """fp16 / bf16 copy of vectors / max_norm (the screen's B operand)."""
        key = ("bf16" if bf16 else "f16", str(device))
        t = self._dev.get(key)
        if t is None:
            mx = self.max_norm()
            dv = self.device_vectors(device)
            t = engine.to_bf16_rows(dv, 1.0 / mx) if bf16 else engine.to_f16_rows(dv, 1.0 / mx)
            self._dev[key] = t
        return t

    def max_norm(self) -> float:
        mx = self._dev.get("max_norm")
        if mx is None:
            mx = float(np.linalg.norm(self.vectors, axis=1).max())
            self._dev["max_norm"] = mx
        return mx

    def device_f16(self, device):
        """(fp16 copy of vectors / max_norm, max_norm) for the tensor-core screen."""
        return self.device_lowp(device, bf16=False), self.max_norm()


@dataclass
class CentroidIndex:
    """Per-centroid postings of ascending, deduplicated doc indices (prefilter.py:29-34),
    held on the device as CSR (post_off (k+1), post_docs)."""

    n_docs: int
    post_off: torch.Tensor
    post_docs: torch.Tensor
    _cache: dict = field(default_factory=dict, repr=False, compare=False)

    def chunk_bounds(self, m_q: int, probe: int) -> torch.Tensor:
        """Posting chunk boundaries for the counting pass, computed once per counter
        width (the index is immutable)."""
        k_c = self.post_off.shape[0] - 1
        key = 8 if m_q * min(probe, k_c) <= 255 else 16
        t = self._cache.get(key)
        if t is None:
            t = engine.posting_chunk_bounds(self.post_off, self.post_docs, self.n_docs, m_q, probe)
            self._cache[key] = t
        return t

    @property
    def postings(self) -> list[np.ndarray]:
        off = self.post_off.cpu().numpy()
        docs = self.post_docs.cpu().numpy()
        return [docs[off[c]:off[c + 1]] for c in range(len(off) - 1)]


def _as_dev(X, device="cuda") -> torch.Tensor:
    if isinstance(X, torch.Tensor):
        return X.to(device)
    return torch.from_numpy(np.ascontiguousarray(np.asarray(X, dtype=np.float64))).to(device)


def train_centroids(samples, k: int, iters: int, seed: int, device="cuda") -> Centroids:
    """Spherical Lloyd iterations (prefilter.py:47-82) -- K7, native and deterministic.

    The init indices come from the reference's own rng call
    (np.random.default_rng(seed).choice(n, k, replace=False)); everything
    else runs in dsrt_train_centroids in float64, in numpy's operation order.
    """
    X = _as_dev(samples, device)
    if X.dim() != 2 or X.shape[0] == 0:
        raise ValueError(f"samples must be a non-empty (n, d) matrix, got shape {tuple(X.shape)}")
    X = X.to(torch.float64).contiguous()
    n = X.shape[0]
    init = None
    if 1 <= k <= n and iters >= 1:
        init = np.random.default_rng(seed).choice(n, size=k, replace=False)
    cents = engine.train_centroids(X, k, iters, init)
    return Centroids(k=k, seed=seed, vectors=cents.cpu().numpy())


def _check_nonzero_rows(X: torch.Tensor, off: torch.Tensor, chunk: int = 1 << 22) -> None:
    """prefilter.py:37-44 error ("zero vector in document i"), chunked (no float64 copy)."""
    for lo in range(0, X.shape[0], chunk):
        blk = X[lo:lo + chunk]
        z = (blk == 0).all(dim=1)
        if bool(z.any()):
            row = lo + int(torch.nonzero(z)[0].item())
            doc = int(torch.searchsorted(off, torch.tensor([row], device=off.device), right=True)[0]) - 1
            raise ValueError(f"zero vector in document {doc}: cannot assign to a centroid")


def build_centroid_index(docs, centroids: Centroids, set_off: torch.Tensor | None = None,
                         n_docs: int | None = None, device="cuda") -> CentroidIndex:
    """Invert centroid assignment (prefilter.py:85-108): posting c = docs with a
    vector whose argmax-dot centroid is c, each doc once, ascending.

    ``docs`` is either a list of (m_i, d) arrays or one device matrix of all
    vectors grouped by set with ``set_off``.
    """
    if isinstance(docs, torch.Tensor) and set_off is not None:
        X = docs
        off = set_off
        N = int(n_docs)
    else:
        mats = [np.asarray(S, dtype=np.float64) if not isinstance(S, torch.Tensor) else S
                for S in docs]
        if not mats:
            raise ValueError("empty collection: nothing to index")
        for i, S in enumerate(mats):
            if S.ndim != 2 or S.shape[1] != centroids.vectors.shape[1]:
                raise ValueError(
                    f"dimension mismatch: document {i} has d={S.shape[1]}, "
                    f"centroids have d={centroids.vectors.shape[1]}")
        sizes = np.array([S.shape[0] for S in mats], dtype=np.int64)
        X = torch.cat([_as_dev(S, device).to(torch.float64) for S in mats])
        off = torch.from_numpy(np.concatenate([[0], np.cumsum(sizes)])).to(X.device)
        N = len(mats)
    _check_nonzero_rows(X, off)
    return build_centroid_index_native(X, centroids, off, N)


def build_centroid_index_native(X: torch.Tensor, centroids: Centroids, set_off: torch.Tensor,
                                n_docs: int) -> CentroidIndex:
    """K6 on the device: exact argmax assignment (d = 128: tcgen05 screen + float64
    re-rank; other d: float64 SIMT scan; np.argmax tie rule) and postings by stable
    radix counting sort."""
    if X.dtype not in (torch.float16, torch.bfloat16, torch.float32, torch.float64):
        X = X.to(torch.float64)
    cvec = centroids.device_vectors(X.device)
    lowp = (centroids.device_lowp(X.device, bf16=X.dtype == torch.bfloat16)
            if X.shape[1] == 128 else None)
    assign = engine.assign_centroids(X, cvec, lowp)
    post_off, post_docs = engine.postings_from_assign(assign, set_off.contiguous(), n_docs,
                                                      centroids.k)
    return CentroidIndex(n_docs=n_docs, post_off=post_off, post_docs=post_docs)


def extend_centroid_index(cindex: CentroidIndex, X: torch.Tensor, centroids: Centroids,
                          sizes: np.ndarray) -> CentroidIndex:
    """Add postings for new docs (appended after the existing n_docs): K6 on the
    new vectors, then each posting = old posting + new docs (ids all larger)."""
    sizes = np.asarray(sizes, np.int64)
    off = torch.from_numpy(np.concatenate([[0], np.cumsum(sizes)])).to(X.device)
    add = build_centroid_index_native(X, centroids, off, len(sizes))
    add_docs = add.post_docs + cindex.n_docs
    post_off, post_docs = engine.merge_postings(cindex.post_off, cindex.post_docs, add.post_off,
                                                add_docs)
    return CentroidIndex(n_docs=cindex.n_docs + len(sizes), post_off=post_off, post_docs=post_docs)


def filter_candidates_device(cindex: CentroidIndex, centroids: Centroids, Q: torch.Tensor,
                             m_q: int, probe: int, k_filter: int, use_tc: bool = True):
    """K5 on the device: Q (n_qsets*m_q, d) -> (cand (n_qsets, k_filter), n_cand)."""
    if probe < 1:
        raise ValueError(f"invalid parameter: probe must be >= 1, got {probe}")
    if k_filter < 1:
        raise ValueError(f"invalid parameter: k_filter must be >= 1, got {k_filter}")
    Qd = Q.to(torch.float64).contiguous()
    if Qd.shape[1] != centroids.vectors.shape[1]:
        raise ValueError(f"dimension mismatch: Q has d={Qd.shape[1]}, "
                         f"centroids have d={centroids.vectors.shape[1]}")
    P = min(probe, centroids.k)
    if Qd.shape[1] == 128 and P <= 12 and use_tc:
        c16, mx = centroids.device_f16(Qd.device)
        return engine.prefilter_tc(Qd, m_q, centroids.device_vectors(Qd.device), c16, mx,
                                   cindex.post_off, cindex.post_docs, cindex.n_docs, probe,
                                   k_filter, chunk_bounds=cindex.chunk_bounds(m_q, probe))
    return engine.prefilter(Qd, m_q, centroids.device_vectors(Qd.device), cindex.post_off,
                            cindex.post_docs, cindex.n_docs, probe, k_filter,
                            chunk_bounds=cindex.chunk_bounds(m_q, probe))


def filter_candidates(index: CentroidIndex, centroids: Centroids, Q, probe: int,
                      k_filter: int) -> np.ndarray:
    """Drop-in for prefilter.filter_candidates: ordered doc indices (count desc, index asc)."""
    if probe < 1:
        raise ValueError(f"invalid parameter: probe must be >= 1, got {probe}")
    if k_filter < 1:
        raise ValueError(f"invalid parameter: k_filter must be >= 1, got {k_filter}")
    Qa = Q if isinstance(Q, torch.Tensor) else np.asarray(Q, dtype=np.float64)
    if Qa.ndim != 2 or Qa.shape[0] == 0:
        raise ValueError(f"Q must be a non-empty (m_q, d) matrix, got shape {tuple(Qa.shape)}")
    if Qa.shape[1] != centroids.vectors.shape[1]:
        raise ValueError(f"dimension mismatch: Q has d={Qa.shape[1]}, "
                         f"centroids have d={centroids.vectors.shape[1]}")
    Qd = _as_dev(Qa, index.post_off.device)
    cand, n_cand = filter_candidates_device(index, centroids, Qd, Qd.shape[0], probe, k_filter)
    n = int(n_cand[0].item())
    return cand[0, :n].cpu().numpy().astype(np.int64)
