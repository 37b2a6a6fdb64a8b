"""Index files (.dsri) -- drop-in for dessert.storage save_index / load_index
(storage.py:130-260), byte-identical to the reference's format, produced from
and loaded into the device layout.

* ``save_index``: the header is packed here; the sets section (doc id +
  TinyTable per set) is written on the device by dsrt_dsri_write_sets (a
  stable per-(set, table) counting sort over the plane records, equal to
  build_tiny_table), the prefilter postings are varint-encoded by
  dsrt_postings_to_varints.
* ``load_index``: dsrt_dsri_scan_sets walks the set headers (host, native),
  dsrt_dsri_decode_sets validates every TinyTable and decodes the codes on
  the device, dsrt_varints_to_postings rebuilds the postings CSR.  Errors are
  the reference's exception types and messages, raised for the same (first)
  offending set.
"""

from __future__ import annotations

import ctypes
import struct
from pathlib import Path

import numpy as np
import torch

from . import _lib, engine
from .index import DessertIndex, FilterConfig, IndexConfig, build_from_codes
from .prefilter import CentroidIndex, Centroids
from .scoring import PHI_KINDS

INDEX_MAGIC = b"DSRI"
FORMAT_VERSION = 1
_HEADER = struct.Struct("<IIIIQBBBBIIII")
_TT_HEADER = 24


class StorageError(Exception):
    """Base class for file format failures."""


class BadMagicError(StorageError):
    pass


class VersionMismatchError(StorageError):
    pass


class TruncatedFileError(StorageError):
    pass


class CorruptSketchError(StorageError):
    pass


def _set_bytes(sizes: np.ndarray, L: int, r: int) -> np.ndarray:
    """Bytes of (doc id + TinyTable) per set (sketch.py:180-189 + 8)."""
    ow = np.where(sizes <= 255, 1, 2)
    iw = np.where(sizes <= 256, 1, 2)
    return 8 + _TT_HEADER + L * ((r + 1) * ow + sizes * iw)


def _ptr(t):
    return ctypes.c_void_p(t.data_ptr()) if t is not None else None


def _stream():
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def _sets_section(index: DessertIndex) -> np.ndarray:
    cfg = index.config
    r = 1 << cfg.C
    sizes = index.sizes.astype(np.int64)
    nbytes = _set_bytes(sizes, cfg.L, r)
    rec_off = np.zeros(len(sizes), dtype=np.int64)
    np.cumsum(nbytes[:-1], out=rec_off[1:])
    total = int(nbytes.sum())
    dev = index.device
    out = torch.empty(total, dtype=torch.uint8, device=dev)
    off_dev = torch.from_numpy(rec_off).to(dev)
    _lib.call("dsrt_dsri_write_sets", _ptr(index.records), _ptr(index.set_off),
              _ptr(index.doc_ids_dev), index.n_docs, cfg.L, cfg.C, _ptr(off_dev), _ptr(out),
              _stream())
    return out.cpu().numpy()


def _postings_varints(cindex: CentroidIndex) -> bytes:
    k = cindex.post_off.shape[0] - 1
    total = int(cindex.post_docs.shape[0])
    ws_bytes = _lib.lib().dsrt_varint_workspace(k + total)
    dev = cindex.post_off.device
    ws = torch.empty(max(ws_bytes, 1), dtype=torch.uint8, device=dev)
    n = ctypes.c_int64(0)
    _lib.call("dsrt_postings_to_varints", _ptr(cindex.post_off), _ptr(cindex.post_docs), k,
              total, None, ctypes.byref(n), _ptr(ws), ws_bytes, _stream())
    out = torch.empty(max(n.value, 1), dtype=torch.uint8, device=dev)
    _lib.call("dsrt_postings_to_varints", _ptr(cindex.post_off), _ptr(cindex.post_docs), k,
              total, _ptr(out), ctypes.byref(n), _ptr(ws), ws_bytes, _stream())
    return out[: n.value].cpu().numpy().tobytes()


def save_index(path, index: DessertIndex) -> None:
    """Serialize an index (storage.py:130-173). Equal indexes produce equal bytes."""
    cfg = index.config
    phi_code = 0 if cfg.phi is None else PHI_KINDS.index(cfg.phi) + 1
    parts = [
        INDEX_MAGIC,
        _HEADER.pack(FORMAT_VERSION, cfg.d, cfg.C, cfg.L, cfg.seed,
                     0 if cfg.inner_kind == "max" else 1, phi_code,
                     1 if cfg.filter.enabled else 0, 0, cfg.filter.centroids, cfg.filter.iters,
                     cfg.filter.probe, cfg.filter.k_filter),
        struct.pack("<Q", index.n_docs),
        _sets_section(index),
    ]
    if index.filter is not None:
        centroids, cindex = index.filter
        parts.append(struct.pack("<IIQ", centroids.k, cfg.d, cindex.n_docs))
        parts.append(np.ascontiguousarray(centroids.vectors, dtype="<f8").tobytes())
        parts.append(_postings_varints(cindex))
    with open(path, "wb") as f:  # buffers written as they are (no joined copy)
        for part in parts:
            f.write(memoryview(part))


class _Reader:
    def __init__(self, buf: bytes, path):
        self.buf, self.pos, self.path = buf, 0, path

    def take(self, n: int) -> bytes:
        if self.pos + n > len(self.buf):
            raise TruncatedFileError(f"{self.path}: truncated (needed {n} more bytes)")
        out = self.buf[self.pos:self.pos + n]
        self.pos += n
        return out

    def unpack(self, fmt: str):
        return struct.unpack("<" + fmt, self.take(struct.calcsize("<" + fmt)))


def _payload_error(buf: bytes, pos: int, m: int, L: int, r: int, flags: int):
    """The reference's payload checks for one TinyTable (sketch.py:224-238), host-side;
    only used to order errors for a set whose shape differs from the config."""
    ow = 2 if flags & 1 else 1
    iw = 2 if flags & 2 else 1
    p = pos + _TT_HEADER
    off = np.frombuffer(buf, dtype="<u2" if ow == 2 else "u1", count=L * (r + 1), offset=p)
    off = off.astype(np.int64).reshape(L, r + 1)
    ids = np.frombuffer(buf, dtype="<u2" if iw == 2 else "u1", count=L * m,
                        offset=p + L * (r + 1) * ow).astype(np.int64).reshape(L, m)
    if np.any(off[:, 0] != 0) or np.any(off[:, -1] != m):
        return "corrupt sketch: offsets do not span 0..m"
    if np.any(np.diff(off, axis=1) < 0):
        return "corrupt sketch: offsets not monotone"
    if not np.array_equal(np.sort(ids, axis=1), np.broadcast_to(np.arange(m), (L, m))):
        return "corrupt sketch: ids are not a permutation per table"
    return None


_DEVICE_ERRORS = {1: "corrupt sketch: offsets do not span 0..m",
                  2: "corrupt sketch: offsets not monotone",
                  3: "corrupt sketch: ids are not a permutation per table"}


def load_index(path, device="cuda") -> DessertIndex:
    """Load an index (storage.py:176-260) straight into the device layout."""
    buf = Path(path).read_bytes()
    r = _Reader(buf, path)
    magic = r.take(4)
    if magic != INDEX_MAGIC:
        raise BadMagicError(f"{path}: bad magic {magic!r}, expected {INDEX_MAGIC!r}")
    (version, d, C, L, seed, inner_code, phi_code, filter_enabled, _pad, f_centroids, f_iters,
     f_probe, f_kfilter) = r.unpack("IIIIQBBBBIIII")
    if version != FORMAT_VERSION:
        raise VersionMismatchError(f"{path}: format version {version}, expected {FORMAT_VERSION}")
    config = IndexConfig(
        d=d, C=C, L=L, seed=seed, inner_kind="max" if inner_code == 0 else "avg-phi",
        phi=None if phi_code == 0 else PHI_KINDS[phi_code - 1],
        filter=FilterConfig(enabled=bool(filter_enabled), centroids=f_centroids, iters=f_iters,
                            probe=f_probe, k_filter=f_kfilter))
    (n_docs,) = r.unpack("Q")
    if n_docs < 1:
        raise TruncatedFileError(f"{path}: index declares zero sets")

    # ---- sets: host header walk, device validation + decode
    doc_ids = np.zeros(n_docs, dtype=np.uint64)
    sizes = np.zeros(n_docs, dtype=np.int64)
    tt_off = np.zeros(n_docs, dtype=np.int64)
    hdr = np.zeros(4, dtype=np.uint32)
    err = ctypes.c_int(0)
    end = ctypes.c_size_t(0)
    raw = np.frombuffer(buf, dtype=np.uint8)
    lib = _lib.lib()
    n_ok = lib.dsrt_dsri_scan_sets(raw.ctypes.data_as(ctypes.c_void_p), len(buf), r.pos, n_docs,
                                   L, C, doc_ids.ctypes.data_as(ctypes.c_void_p),
                                   sizes.ctypes.data_as(ctypes.c_void_p),
                                   tt_off.ctypes.data_as(ctypes.c_void_p),
                                   hdr.ctypes.data_as(ctypes.c_void_p), ctypes.byref(err),
                                   ctypes.byref(end))
    dev = torch.device(device)
    code_dtype = engine.code_dtype(C)
    n_vec = int(sizes[:n_ok].sum())
    set_off_h = np.zeros(n_ok + 1, dtype=np.int64)
    np.cumsum(sizes[:n_ok], out=set_off_h[1:])
    codes = torch.empty((max(n_vec, 1), L), dtype=code_dtype, device=dev)
    first_bad = ctypes.c_int64(-1)
    if n_ok > 0:
        # bytes through the last parsed TinyTable (tt_off points at its header)
        hi = int(tt_off[n_ok - 1]) + int(_set_bytes(sizes[n_ok - 1:n_ok], L, 1 << C)[0]) - 8
        # keep every device temporary referenced until the call returns
        buf_dev = torch.from_numpy(raw[:hi].copy()).to(dev)
        tt_dev = torch.from_numpy(tt_off[:n_ok].copy()).to(dev)
        off_dev = torch.from_numpy(set_off_h).to(dev)
        _lib.call("dsrt_dsri_decode_sets", _ptr(buf_dev), _ptr(tt_dev), _ptr(off_dev), n_ok, L, C,
                  int(sizes[:n_ok].max()), _ptr(codes), codes.element_size(),
                  ctypes.byref(first_bad), _stream())
        del buf_dev, tt_dev, off_dev
    if first_bad.value >= 0:
        s, kind = first_bad.value >> 2, first_bad.value & 3
        raise CorruptSketchError(f"{path}: set {doc_ids[s]}: {_DEVICE_ERRORS[kind]}")
    if err.value:
        s = n_ok
        m, l_f, r_f, flags = (int(x) for x in hdr)
        if err.value == 1:
            raise TruncatedFileError(f"{path}: truncated (needed 8 more bytes)")
        if err.value == 2:
            raise TruncatedFileError(f"{path}: truncated sketch: missing header")
        if err.value == 3:
            raise TruncatedFileError(f"{path}: truncated sketch: missing payload")
        if err.value == 4:
            raise CorruptSketchError(f"{path}: set {doc_ids[s]}: corrupt sketch: bad dimensions "
                                     f"m={m}, L={l_f}, r={r_f}")
        if err.value == 5:
            raise CorruptSketchError(f"{path}: set {doc_ids[s]}: corrupt sketch: width flags "
                                     f"{flags} inconsistent with m={m}")
        msg = _payload_error(buf, end.value, m, l_f, r_f, flags)
        if msg is not None:
            raise CorruptSketchError(f"{path}: set {doc_ids[s]}: {msg}")
        raise CorruptSketchError(f"{path}: set {doc_ids[s]}: sketch shape (L={l_f}, r={r_f}) "
                                 f"does not match config (L={L}, r={1 << C})")
    r.pos = end.value

    # ---- prefilter block
    filt = None
    if filter_enabled:
        k, cd, fn_docs = r.unpack("IIQ")
        if cd != d or fn_docs != n_docs:
            raise CorruptSketchError(f"{path}: prefilter block inconsistent with index")
        vectors = np.frombuffer(r.take(8 * k * d), dtype="<f8", count=k * d)
        vectors = vectors.astype(np.float64).reshape(k, d)
        tail = raw[r.pos:]
        n_bytes = int(tail.shape[0])
        ws_bytes = lib.dsrt_varint_workspace(n_bytes) + (k + 2) * 8
        ws = torch.empty(ws_bytes, dtype=torch.uint8, device=dev)
        tail_dev = torch.from_numpy(tail.copy() if n_bytes else np.zeros(1, np.uint8)).to(dev)
        post_off = torch.empty(k + 1, dtype=torch.int64, device=dev)
        post_docs = torch.empty(max(n_bytes, 1), dtype=torch.int64, device=dev)
        total = ctypes.c_int64(0)
        try:
            _lib.call("dsrt_varints_to_postings", _ptr(tail_dev), n_bytes, k, _ptr(post_off),
                      _ptr(post_docs), ctypes.byref(total), _ptr(ws), ws_bytes, _stream())
        except IndexError:
            raise TruncatedFileError(f"{path}: truncated (needed 1 more bytes)") from None
        filt = (Centroids(k=k, seed=seed, vectors=vectors),
                CentroidIndex(n_docs=n_docs, post_off=post_off,
                              post_docs=post_docs[: total.value].clone()))

    index = build_from_codes(codes[:n_vec], sizes, doc_ids, config, filt=filt)
    return index


__all__ = ["save_index", "load_index", "StorageError", "BadMagicError", "VersionMismatchError",
           "TruncatedFileError", "CorruptSketchError", "INDEX_MAGIC", "FORMAT_VERSION"]
