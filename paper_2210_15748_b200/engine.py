"""Thin typed wrappers over the C ABI, taking torch CUDA tensors as buffers.

Each function checks shapes/dtypes/devices, passes ``data_ptr()`` and the
current CUDA stream to the library, and returns freshly allocated output
tensors.  torch is used only for device memory and streams; every
computation happens in the library's sm_100a kernels.
"""

from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import _lib

_DT = {torch.float32: _lib.F32, torch.float64: _lib.F64, torch.float16: _lib.F16,
       torch.bfloat16: _lib.BF16}


def _ptr(t):
    return ctypes.c_void_p(t.data_ptr()) if t is not None else None


def _stream():
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def _need(t, dtype, name):
    if not t.is_cuda:
        raise ValueError(f"invalid parameter: {name} must be a CUDA tensor")
    if t.dtype != dtype:
        raise ValueError(f"invalid parameter: {name} must be {dtype}, got {t.dtype}")
    if not t.is_contiguous():
        raise ValueError(f"invalid parameter: {name} must be contiguous")


def code_dtype(C: int):
    return torch.uint8 if C <= 8 else (torch.int16 if C <= 16 else torch.int32)


def code_bytes(C: int) -> int:
    return 1 if C <= 8 else (2 if C <= 16 else 4)


def record_words(L: int, C: int) -> int:
    r = _lib.lib().dsrt_record_words(L, C)
    if r <= 0:
        raise ValueError(f"invalid parameter: L={L} C={C}")
    return r


def device_info():
    sms, ma, mi, fr = ctypes.c_int(), ctypes.c_int(), ctypes.c_int(), ctypes.c_size_t()
    _lib.call("dsrt_device_info", ctypes.byref(sms), ctypes.byref(ma), ctypes.byref(mi),
              ctypes.byref(fr))
    return {"sm_count": sms.value, "cc": (ma.value, mi.value), "free_bytes": fr.value}


def copy_async(dst: torch.Tensor, src: torch.Tensor):
    """Stream-ordered copy between a device tensor and a pinned host tensor (or two
    device tensors) of equal dtype and shape, on the current stream (dsrt_copy_async:
    capturable, no allocator bookkeeping)."""
    if dst.shape != src.shape or dst.dtype != src.dtype:
        raise ValueError("invalid parameter: copy_async needs equal shapes and dtypes")
    if not (dst.is_contiguous() and src.is_contiguous()):
        raise ValueError("invalid parameter: copy_async needs contiguous tensors")
    for t in (dst, src):
        if not t.is_cuda and not t.is_pinned():
            raise ValueError("invalid parameter: host side of copy_async must be page-locked")
    _lib.call("dsrt_copy_async", _ptr(dst), _ptr(src), ctypes.c_size_t(dst.numel() * dst.element_size()),
              _stream())


def pack_layout(tensors):
    """(offsets, total bytes) of dsrt_pack4_async's destination for up to four tensors
    (None = absent): each segment starts at the next 16-byte boundary."""
    offs, off = [], 0
    for t in tensors:
        offs.append(off)
        if t is not None:
            off += (t.numel() * t.element_size() + 15) & ~15
    return offs, max(off, 16)


def pack4(dst: torch.Tensor, tensors):
    """Concatenate up to four small contiguous CUDA tensors into ``dst`` (uint8; device or
    pinned host memory) with one kernel on the current stream (dsrt_pack4_async)."""
    ts = list(tensors) + [None] * (4 - len(tensors))
    if len(ts) != 4:
        raise ValueError("invalid parameter: pack4 takes at most four tensors")
    args = []
    for t in ts:
        if t is not None and not (t.is_cuda and t.is_contiguous()):
            raise ValueError("invalid parameter: pack4 sources must be contiguous CUDA tensors")
        args += [_ptr(t), ctypes.c_size_t(0 if t is None else t.numel() * t.element_size())]
    if not dst.is_cuda and not dst.is_pinned():
        raise ValueError("invalid parameter: host side of pack4 must be page-locked")
    if dst.numel() * dst.element_size() < pack_layout(ts)[1]:
        raise ValueError("invalid parameter: pack4 destination too small")
    _lib.call("dsrt_pack4_async", _ptr(dst), *args, _stream())


# ------------------------------------------------------------------- K1
def hash_vectors(X: torch.Tensor, planes: torch.Tensor, mode: int, L: int, C: int,
                 want_codes: bool = True, want_records: bool = True, check_zero: bool = True):
    """X (n, d) CUDA tensor -> (codes (n, L) or None, records (n, R) or None, n_zero_rows)."""
    if X.dim() != 2:
        raise ValueError(f"dimension mismatch: expected (n, d) matrix, got shape {tuple(X.shape)}")
    if X.dtype not in _DT:
        raise ValueError(f"invalid parameter: unsupported vector dtype {X.dtype}")
    X = X.contiguous()
    n, d = X.shape
    codes = torch.empty((n, L), dtype=code_dtype(C), device=X.device) if want_codes else None
    recs = (torch.empty((n, record_words(L, C)), dtype=torch.int32, device=X.device)
            if want_records else None)
    zero = torch.zeros(1, dtype=torch.int32, device=X.device) if check_zero else None
    _lib.call("dsrt_hash", _ptr(X), _DT[X.dtype], n, d, _ptr(planes), mode, L, C, _ptr(codes),
              _ptr(recs), _ptr(zero), _stream())
    return codes, recs, zero


# ------------------------------------------------------------------- K2
def codes_to_records(codes: torch.Tensor, L: int, C: int, check: bool = True):
    if codes.dim() != 2 or codes.shape[1] != L:
        raise ValueError(f"expected (m, {L}) code matrix, got shape {tuple(codes.shape)}")
    codes = codes.contiguous()
    cb = codes.element_size()
    n = codes.shape[0]
    recs = torch.empty((n, record_words(L, C)), dtype=torch.int32, device=codes.device)
    bad = torch.zeros(1, dtype=torch.int32, device=codes.device) if check else None
    _lib.call("dsrt_codes_to_records", _ptr(codes), cb, n, L, C, _ptr(recs), _ptr(bad), _stream())
    return recs, bad


def sizes_to_offsets(sizes: torch.Tensor):
    _need(sizes, torch.int64, "sizes")
    n = sizes.shape[0]
    out = torch.empty(n + 1, dtype=torch.int64, device=sizes.device)
    ws_bytes = _lib.lib().dsrt_scan_workspace(n)
    ws = torch.empty(max(ws_bytes, 8), dtype=torch.uint8, device=sizes.device)
    bad = torch.zeros(1, dtype=torch.int32, device=sizes.device)
    _lib.call("dsrt_sizes_to_offsets", _ptr(sizes), n, _ptr(out), _ptr(bad), _ptr(ws), ws_bytes,
              _stream())
    return out, bad


def counting_sort(set_of_vec: torch.Tensor, n_sets: int):
    """Vectors tagged by set id -> (set_off (N+1), stable perm (n))."""
    _need(set_of_vec, torch.int64, "set_of_vec")
    n = set_of_vec.shape[0]
    set_off = torch.empty(n_sets + 1, dtype=torch.int64, device=set_of_vec.device)
    perm = torch.empty(n, dtype=torch.int64, device=set_of_vec.device)
    ws_bytes = _lib.lib().dsrt_counting_sort_workspace(n, n_sets)
    ws = torch.empty(ws_bytes, dtype=torch.uint8, device=set_of_vec.device)
    _lib.call("dsrt_counting_sort", _ptr(set_of_vec), n, n_sets, _ptr(set_off), _ptr(perm),
              _ptr(ws), ws_bytes, _stream())
    return set_off, perm


def gather_rows(src: torch.Tensor, perm: torch.Tensor):
    _need(perm, torch.int64, "perm")
    src = src.contiguous()
    row_bytes = src[0].numel() * src.element_size() if src.shape[0] else 4
    dst = torch.empty((perm.shape[0],) + tuple(src.shape[1:]), dtype=src.dtype, device=src.device)
    _lib.call("dsrt_gather_rows", _ptr(src), row_bytes, _ptr(perm), perm.shape[0], _ptr(dst),
              _stream())
    return dst


def tinytable(codes: torch.Tensor, set_off: torch.Tensor, s: int, m: int, L: int, C: int):
    r = 1 << C
    offsets = torch.empty((L, r + 1), dtype=torch.int32, device=codes.device)
    ids = torch.empty((L, m), dtype=torch.int32, device=codes.device)
    _lib.call("dsrt_tinytable", _ptr(codes), codes.element_size(), _ptr(set_off), s, L, C,
              _ptr(offsets), _ptr(ids), _stream())
    return offsets, ids


# ------------------------------------------------------------------- K3
def score_all(records, set_off, qrecords, m_q: int, L: int, C: int, lut, set_begin=0,
              set_end=None, scores=None, ld=None, want_counts=False):
    n_sets = set_off.shape[0] - 1
    set_end = n_sets if set_end is None else set_end
    n_q = qrecords.shape[0] // m_q if qrecords.dim() == 2 else qrecords.shape[0]
    width = set_end - set_begin
    if scores is None:
        ld = width if ld is None else ld
        scores = torch.empty((n_q, ld), dtype=torch.float64, device=records.device)
    ld = scores.shape[1] if ld is None else ld
    mc = (torch.empty((n_q, ld, m_q), dtype=torch.int16, device=records.device)
          if want_counts else None)
    _lib.call("dsrt_score_all", _ptr(records), _ptr(set_off), set_begin, set_end, _ptr(qrecords),
              n_q, m_q, L, C, _ptr(lut), _ptr(scores), ld, _ptr(mc), _stream())
    return scores, mc


def score_candidates(records, set_off, qrecords, m_q: int, L: int, C: int, lut, cand=None,
                     n_cand=None, cand_ld=None, n_qsets=None, want_counts=False):
    n_sets = set_off.shape[0] - 1
    n_q = n_qsets if n_qsets is not None else (qrecords.shape[0] // m_q)
    if cand is not None:
        _need(cand, torch.int64, "cand")
        cand_ld = cand.shape[-1]
    elif cand_ld is None:
        cand_ld = n_sets
    if n_cand is not None:
        _need(n_cand, torch.int32, "n_cand")
    scores = torch.empty((n_q, cand_ld), dtype=torch.float64, device=records.device)
    mc = (torch.empty((n_q, cand_ld, m_q), dtype=torch.int16, device=records.device)
          if want_counts else None)
    _lib.call("dsrt_score_candidates", _ptr(records), _ptr(set_off), n_sets, _ptr(cand),
              _ptr(n_cand), cand_ld, _ptr(qrecords), n_q, m_q, L, C, _ptr(lut), _ptr(scores),
              _ptr(mc), _stream())
    return scores, mc


def score_agg(records, set_off, qrecords, m_q: int, L: int, C: int, table, inner_kind: int,
              weights=None, m_cap: int = 0, cand=None, n_cand=None, cand_ld=None, n_qsets=None):
    """General aggregation scores (sigma max / avg-phi, optional weights): (n_qsets, cand_ld)."""
    _need(table, torch.float64, "table")
    n_sets = set_off.shape[0] - 1
    n_q = n_qsets if n_qsets is not None else (qrecords.shape[0] // m_q)
    if cand is not None:
        _need(cand, torch.int64, "cand")
        cand_ld = cand.shape[-1]
    elif cand_ld is None:
        cand_ld = n_sets
    if n_cand is not None:
        _need(n_cand, torch.int32, "n_cand")
    if weights is not None:
        _need(weights, torch.float64, "weights")
        if weights.numel() != m_q:
            raise ValueError(f"length mismatch: {weights.numel()} weights for {m_q} query vectors")
    scores = torch.empty((n_q, cand_ld), dtype=torch.float64, device=records.device)
    ws_bytes = _lib.lib().dsrt_score_agg_workspace(n_q, cand_ld, m_q, m_cap)
    ws = torch.empty(max(ws_bytes, 1), dtype=torch.uint8, device=records.device)
    _lib.call("dsrt_score_agg", _ptr(records), _ptr(set_off), n_sets, _ptr(cand), _ptr(n_cand),
              cand_ld, _ptr(qrecords), n_q, m_q, L, C, inner_kind, _ptr(table), _ptr(weights),
              m_cap, _ptr(scores), _ptr(ws), ws_bytes, _stream())
    return scores


def train_centroids(samples: torch.Tensor, k: int, iters: int, init_idx):
    """K7: spherical k-means on float64 samples (n, d) -> centroids (k, d) float64."""
    _need(samples, torch.float64, "samples")
    n, d = samples.shape
    init = None
    if init_idx is not None:
        init = torch.as_tensor(np.asarray(init_idx, dtype=np.int64)).to(samples.device)
    out = torch.empty((max(k, 1), d), dtype=torch.float64, device=samples.device)
    ws_bytes = _lib.lib().dsrt_train_centroids_workspace(n, d, k)
    ws = torch.empty(max(ws_bytes, 1), dtype=torch.uint8, device=samples.device)
    _lib.call("dsrt_train_centroids", _ptr(samples), n, d, k, iters, _ptr(init), _ptr(out),
              _ptr(ws), ws_bytes, _stream())
    return out


def collision_counts(offsets, ids, L: int, r: int, m: int, qcodes, out):
    """TinyTable bucket gather: out (m_q, m) int32 collision counts."""
    _lib.call("dsrt_collision_counts", _ptr(offsets), _ptr(ids), L, r, m, _ptr(qcodes),
              qcodes.shape[0], _ptr(out), _stream())
    return out


# ------------------------------------------------------------------- K4
def topk(scores: torch.Tensor, k: int, ids: torch.Tensor | None = None, n_valid=None, n=None,
         id_index: torch.Tensor | None = None):
    """Row-wise top-k by (score desc, id asc); ids shared (1-D) or per row (2-D).

    ``scores`` may be a row-strided view (unit column stride), e.g. the first
    columns of a wider score buffer; the kernel reads rows at stride ld.
    ``id_index`` (rows, n) int64: element i of row r has id ids[id_index[r, i]]
    (candidate lists; 1-D ids), read in the kernel."""
    if not scores.is_cuda or scores.dtype != torch.float64:
        raise ValueError("invalid parameter: scores must be a float64 CUDA tensor")
    if scores.dim() != 2 or (scores.shape[1] > 1 and scores.stride(1) != 1):
        raise ValueError("invalid parameter: scores must be 2-D with unit column stride")
    rows, width = scores.shape
    ld = scores.stride(0) if rows > 1 else width
    n = width if n is None else n
    ids_ld = 0
    if ids is not None:
        if ids.dtype not in (torch.int64, torch.uint64):
            raise ValueError("invalid parameter: ids must be 64-bit")
        ids = ids.contiguous()
        ids_ld = ids.shape[1] if ids.dim() == 2 else 0
    if n_valid is not None:
        _need(n_valid, torch.int32, "n_valid")
    out_s = torch.empty((rows, k), dtype=torch.float64, device=scores.device)
    out_i = torch.empty((rows, k), dtype=torch.int64, device=scores.device)
    out_p = torch.empty((rows, k), dtype=torch.int64, device=scores.device)
    if id_index is not None:
        _need(id_index, torch.int64, "id_index")
        if ids is None or ids.dim() != 1 or id_index.dim() != 2 or id_index.shape[0] != rows:
            raise ValueError("invalid parameter: id_index needs 1-D ids and one index row per score row")
        _lib.call("dsrt_topk_indexed", _ptr(scores), ld, _ptr(ids), _ptr(id_index), id_index.stride(0),
                  _ptr(n_valid), n, rows, k, _ptr(out_s), _ptr(out_i), _ptr(out_p), _stream())
        return out_s, out_i, out_p
    _lib.call("dsrt_topk", _ptr(scores), ld, _ptr(ids), ids_ld, _ptr(n_valid), n, rows, k,
              _ptr(out_s), _ptr(out_i), _ptr(out_p), _stream())
    return out_s, out_i, out_p


def topk_max_k() -> int:
    """Largest k of the shared-memory selector; larger k runs the global-merge kernel."""
    return _lib.lib().dsrt_topk_max_k()


def search_all(records, set_off, doc_ids, qrecords, m_q: int, L: int, C: int, lut, k: int,
               weights=None, mode: int = 0, score_buffer_bytes: int = 4 << 30):
    """Exhaustive top-k of every query set over all sets (K3 + K4 fused, dsrt_search_all).

    Returns (scores (n_q, k) f64, doc ids (n_q, k) int64, overflow (1,) int32 device flag).
    mode 0 may set ``overflow`` (survivor list too small): the caller reruns with mode 1."""
    _need(set_off, torch.int64, "set_off")
    _need(doc_ids, torch.int64, "doc_ids")
    n_sets = set_off.shape[0] - 1
    n_q = qrecords.shape[0] // m_q
    if weights is not None:
        _need(weights, torch.float64, "weights")
    out_s = torch.empty((n_q, k), dtype=torch.float64, device=records.device)
    out_i = torch.empty((n_q, k), dtype=torch.int64, device=records.device)
    ovf = torch.empty(1, dtype=torch.int32, device=records.device)
    ws_bytes = _lib.lib().dsrt_search_all_workspace(n_sets, n_q, m_q, k, mode, score_buffer_bytes)
    ws = torch.empty(max(ws_bytes, 256), dtype=torch.uint8, device=records.device)
    _lib.call("dsrt_search_all", _ptr(records), _ptr(set_off), n_sets, _ptr(doc_ids), _ptr(qrecords),
              n_q, m_q, L, C, _ptr(lut), _ptr(weights), k, mode, score_buffer_bytes, _ptr(out_s),
              _ptr(out_i), _ptr(ovf), _ptr(ws), ws_bytes, _stream())
    return out_s, out_i, ovf


def search_profile(enable: bool) -> None:
    """Bracket every dsrt_search_all launch with CUDA events (measurement hook)."""
    _lib.lib().dsrt_search_profile(1 if enable else 0)


def search_profile_read() -> dict:
    """Summed ms of the scoring and top-k/list launches since the last read (syncs)."""
    a, b, n = ctypes.c_double(), ctypes.c_double(), ctypes.c_int64()
    _lib.call("dsrt_search_profile_read", ctypes.byref(a), ctypes.byref(b), ctypes.byref(n))
    return {"score_ms": a.value, "other_ms": b.value, "launches": n.value}


# ------------------------------------------------------------------- K5
def posting_chunk_bounds(post_off, post_docs, n_docs: int, m_q: int, probe: int):
    """Chunk boundaries of every posting for the counting pass (cache per index)."""
    k_c = post_off.shape[0] - 1
    n = _lib.lib().dsrt_posting_chunk_bounds_size(k_c, n_docs, m_q, probe)
    out = torch.empty(max(n, 1), dtype=torch.int64, device=post_off.device)
    _lib.call("dsrt_posting_chunk_bounds", _ptr(post_off), _ptr(post_docs), k_c, n_docs, m_q, probe,
              _ptr(out), _stream())
    return out


def prefilter(Q, m_q: int, centroids, post_off, post_docs, n_docs: int, probe: int,
              k_filter: int, chunk_bounds=None):
    """Q (n_qsets*m_q, d) float64 -> (cand (n_qsets, k_filter) int64, n_cand (n_qsets) int32)."""
    _need(Q, torch.float64, "Q")
    _need(centroids, torch.float64, "centroids")
    n_q = Q.shape[0] // m_q
    k_c, d = centroids.shape
    cand = torch.empty((n_q, k_filter), dtype=torch.int64, device=Q.device)
    n_cand = torch.empty(n_q, dtype=torch.int32, device=Q.device)
    ws_bytes = _lib.lib().dsrt_prefilter_workspace(n_q, m_q, k_c, n_docs, probe)
    ws = torch.empty(max(ws_bytes, 8), dtype=torch.uint8, device=Q.device)
    _lib.call("dsrt_prefilter", _ptr(Q), n_q, m_q, d, _ptr(centroids), k_c, _ptr(post_off),
              _ptr(post_docs), n_docs, _ptr(chunk_bounds), probe, k_filter, _ptr(cand),
              _ptr(n_cand), _ptr(ws), ws_bytes, _stream())
    return cand, n_cand


def tc_selftest(A: torch.Tensor, B: torch.Tensor) -> torch.Tensor:
    """D = A . B^T (K = 128) through the tcgen05 path (diagnostic)."""
    M, N = A.shape[0], B.shape[0]
    D = torch.empty((M, N), dtype=torch.float32, device=A.device)
    _lib.call("dsrt_tc_selftest", _ptr(A.contiguous()), int(A.dtype == torch.bfloat16),
              _ptr(B.contiguous()), int(B.dtype == torch.bfloat16), _ptr(D), M, N, _stream())
    return D


def to_f16_rows(src: torch.Tensor, scale: float) -> torch.Tensor:
    _need(src, torch.float64, "src")
    dst = torch.empty(src.shape, dtype=torch.float16, device=src.device)
    _lib.call("dsrt_to_f16_rows", _ptr(src), src.shape[0], src.shape[1], float(scale), _ptr(dst),
              _stream())
    return dst


def prefilter_tc(Q, m_q: int, centroids, cents_f16, cent_max_norm: float, post_off, post_docs,
                 n_docs: int, probe: int, k_filter: int, chunk_bounds=None):
    """Tensor-core screened prefilter (exact results); Q (n_qsets*m_q, 128) float64."""
    _need(Q, torch.float64, "Q")
    _need(centroids, torch.float64, "centroids")
    n_q = Q.shape[0] // m_q
    k_c, d = centroids.shape
    cand = torch.empty((n_q, k_filter), dtype=torch.int64, device=Q.device)
    n_cand = torch.empty(n_q, dtype=torch.int32, device=Q.device)
    ws_bytes = _lib.lib().dsrt_prefilter_tc_workspace(n_q, m_q, k_c, n_docs, probe)
    ws = torch.empty(max(ws_bytes, 8), dtype=torch.uint8, device=Q.device)
    _lib.call("dsrt_prefilter_tc", _ptr(Q), n_q, m_q, d, _ptr(centroids), _ptr(cents_f16),
              float(cent_max_norm), k_c, _ptr(post_off), _ptr(post_docs), n_docs,
              _ptr(chunk_bounds), probe, k_filter, _ptr(cand), _ptr(n_cand), _ptr(ws), ws_bytes,
              _stream())
    return cand, n_cand


def to_bf16_rows(src: torch.Tensor, scale: float) -> torch.Tensor:
    _need(src, torch.float64, "src")
    dst = torch.empty(src.shape, dtype=torch.bfloat16, device=src.device)
    _lib.call("dsrt_to_bf16_rows", _ptr(src), src.shape[0], src.shape[1], float(scale), _ptr(dst),
              _stream())
    return dst


def assign_centroids(X: torch.Tensor, centroids: torch.Tensor, cents_lp: torch.Tensor | None):
    """Exact argmax centroid per row of X (n, d) -> int32 (n,); cents_lp only for d = 128."""
    if X.dtype not in _DT:
        raise ValueError(f"invalid parameter: unsupported vector dtype {X.dtype}")
    X = X.contiguous()
    _need(centroids, torch.float64, "centroids")
    n, d = X.shape
    out = torch.empty(n, dtype=torch.int32, device=X.device)
    ws_bytes = _lib.lib().dsrt_assign_centroids_workspace(n, d, centroids.shape[0])
    ws = torch.empty(max(ws_bytes, 8), dtype=torch.uint8, device=X.device)
    _lib.call("dsrt_assign_centroids", _ptr(X), _DT[X.dtype], n, d, _ptr(centroids),
              _ptr(cents_lp), centroids.shape[0], _ptr(out), _ptr(ws), ws_bytes, _stream())
    return out


def postings_from_assign(assign: torch.Tensor, set_off: torch.Tensor, n_docs: int, k_c: int):
    """-> (post_off (k_c+1) int64, post_docs int64) with deduplicated ascending docs."""
    _need(assign, torch.int32, "assign")
    _need(set_off, torch.int64, "set_off")
    n = assign.shape[0]
    post_off = torch.empty(k_c + 1, dtype=torch.int64, device=assign.device)
    post_docs = torch.empty(n, dtype=torch.int64, device=assign.device)
    n_post = torch.zeros(1, dtype=torch.int64, device=assign.device)
    ws_bytes = _lib.lib().dsrt_postings_workspace(n, k_c)
    ws = torch.empty(ws_bytes, dtype=torch.uint8, device=assign.device)
    _lib.call("dsrt_postings_from_assign", _ptr(assign), n, _ptr(set_off), n_docs, k_c,
              _ptr(post_off), _ptr(post_docs), _ptr(n_post), _ptr(ws), ws_bytes, _stream())
    return post_off, post_docs[: int(n_post.item())].clone()


def merge_postings(old_off: torch.Tensor, old_docs: torch.Tensor, add_off: torch.Tensor,
                   add_docs: torch.Tensor):
    """Posting c = old posting c + added posting c (added doc ids all newer)."""
    for t, name in ((old_off, "old_off"), (old_docs, "old_docs"), (add_off, "add_off"),
                    (add_docs, "add_docs")):
        _need(t, torch.int64, name)
    k = old_off.shape[0] - 1
    new_off = torch.empty(k + 1, dtype=torch.int64, device=old_off.device)
    new_docs = torch.empty(old_docs.shape[0] + add_docs.shape[0], dtype=torch.int64,
                           device=old_off.device)
    _lib.call("dsrt_merge_postings", _ptr(old_off), _ptr(old_docs), _ptr(add_off), _ptr(add_docs),
              k, _ptr(new_off), _ptr(new_docs), _stream())
    return new_off, new_docs


def microbench_int() -> dict:
    out = (ctypes.c_double * 4)()
    _lib.call("dsrt_microbench_int", out, _stream())
    return {"lop3_ops_per_s": out[0], "popc_ops_per_s": out[1], "imnmx_ops_per_s": out[2],
            "mix_compares_per_s": out[3]}


