"""TinyTable view of the device layout -- drop-in subset of dessert.sketch.

The device never materialises TinyTables on the query path (scoring compares
codes directly; see csrc/score_kernels.cuh).  For callers that inspect
``index.sketches[i]`` or call ``build_tiny_table`` the per-(set, table)
counting sort runs on the GPU (dsrt_tinytable) and returns the reference's
exact offsets/ids arrays (sketch.py:51-80: u8 offsets when m <= 255, u8 ids
when m <= 256, else u16).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import engine

HEADER_BYTES = 24
MAX_SET_SIZE = 65535


def _offset_dtype(m: int):
    return np.dtype(np.uint8) if m <= 255 else np.dtype(np.uint16)


def _id_dtype(m: int):
    return np.dtype(np.uint8) if m <= 256 else np.dtype(np.uint16)


@dataclass(frozen=True)
class TinyTable:
    m: int
    L: int
    r: int
    offsets: np.ndarray
    ids: np.ndarray


def tiny_table_bytes(m: int, r: int, L: int) -> int:
    """sketch.py:181-189."""
    return HEADER_BYTES + L * (_id_dtype(m).itemsize * m + _offset_dtype(m).itemsize * (r + 1))


def export_tiny_table(codes: torch.Tensor, set_off: torch.Tensor, s: int, m: int, L: int,
                      C: int) -> TinyTable:
    offsets, ids = engine.tinytable(codes, set_off, s, m, L, C)
    return TinyTable(m=m, L=L, r=1 << C, offsets=offsets.cpu().numpy().astype(_offset_dtype(m)),
                     ids=ids.cpu().numpy().astype(_id_dtype(m)))


def build_tiny_table(codes_per_vector, L: int, r: int, device="cuda") -> TinyTable:
    """Drop-in for sketch.build_tiny_table (sketch.py:51-80), computed on the GPU."""
    codes = np.asarray(codes_per_vector)
    if codes.ndim != 2:
        raise ValueError(f"expected (m, L) code matrix, got shape {codes.shape}")
    m = codes.shape[0]
    if m == 0:
        raise ValueError("empty set: cannot sketch zero vectors")
    if m > MAX_SET_SIZE:
        raise ValueError(f"set too large: m must be <= {MAX_SET_SIZE}, got {m}")
    if codes.shape[1] != L:
        raise ValueError(f"expected {L} codes per vector, got {codes.shape[1]}")
    if r < 1:
        raise ValueError(f"invalid parameter: r must be >= 1, got {r}")
    if codes.min() < 0 or codes.max() >= r:
        raise ValueError(f"code out of range: codes must lie in [0, {r})")
    C = max(1, int(r - 1).bit_length())
    dev = torch.from_numpy(codes.astype(np.int32)).to(device)
    set_off = torch.tensor([0, m], dtype=torch.int64, device=device)
    offsets, ids = engine.tinytable(dev, set_off, 0, m, L, C)
    off = offsets.cpu().numpy()[:, : r + 1]
    return TinyTable(m=m, L=L, r=r, offsets=off.astype(_offset_dtype(m)),
                     ids=ids.cpu().numpy().astype(_id_dtype(m)))


def bucket(table: TinyTable, t: int, h: int) -> np.ndarray:
    """sketch.py:83-89: the vector ids stored in bucket (t, h), a zero-copy view."""
    if not 0 <= t < table.L:
        raise IndexError(f"table index out of range: t={t}, L={table.L}")
    if not 0 <= h < table.r:
        raise IndexError(f"hash value out of range: h={h}, r={table.r}")
    return table.ids[t, int(table.offsets[t, h]): int(table.offsets[t, h + 1])]


def _collision_counts(table: TinyTable, codes: np.ndarray, device="cuda") -> np.ndarray:
    """counts[q, j] on the device (dsrt_collision_counts): bucket gather per (q, t)."""
    off = torch.from_numpy(np.ascontiguousarray(table.offsets, dtype=np.int32)).to(device)
    ids = torch.from_numpy(np.ascontiguousarray(table.ids, dtype=np.int32)).to(device)
    q = torch.from_numpy(np.ascontiguousarray(codes, dtype=np.int32)).to(device)
    out = torch.empty((codes.shape[0], table.m), dtype=torch.int32, device=device)
    engine.collision_counts(off, ids, table.L, table.r, table.m, q, out)
    return out.cpu().numpy()


def accumulate_collisions(table: TinyTable, query_codes, out: np.ndarray | None = None) -> np.ndarray:
    """sketch.py:92-115: per stored vector, the number of tables colliding with one
    query vector's L codes; ``out`` may supply a buffer of length >= m."""
    codes = np.asarray(query_codes)
    if codes.shape != (table.L,):
        raise ValueError(f"expected {table.L} query codes, got shape {codes.shape}")
    if codes.min() < 0 or codes.max() >= table.r:
        raise ValueError(f"code out of range: codes must lie in [0, {table.r})")
    counts = _collision_counts(table, codes[None, :])[0]
    if out is None:
        return counts
    out[: table.m] = counts
    return out[: table.m]


def accumulate_collisions_batch(table: TinyTable, query_codes, out: np.ndarray | None = None) -> np.ndarray:
    """sketch.py:118-153: row q = accumulate_collisions(table, query_codes[q]);
    ``out`` may supply a (>= m_q, >= m) buffer."""
    codes = np.asarray(query_codes)
    if codes.ndim != 2 or codes.shape[1] != table.L:
        raise ValueError(f"expected (m_q, {table.L}) code matrix, got shape {codes.shape}")
    if codes.min() < 0 or codes.max() >= table.r:  # empty input raises here, as numpy does
        raise ValueError(f"code out of range: codes must lie in [0, {table.r})")
    counts = _collision_counts(table, codes)
    if out is None:
        return counts
    out[: codes.shape[0], : table.m] = counts
    return out[: codes.shape[0], : table.m]


class SketchView:
    """Lazy ``index.sketches``: len() and [i] -> TinyTable exported from the device."""

    def __init__(self, index):
        self._index = index

    def __len__(self):
        return self._index.n_docs

    def __getitem__(self, i):
        idx = self._index
        if not 0 <= i < idx.n_docs:
            raise IndexError(f"set index out of range: {i} (N={idx.n_docs})")
        if idx.codes is None:
            raise RuntimeError("index was built with keep_codes=False; no TinyTable export")
        m = int(idx.sizes[i])
        return export_tiny_table(idx.codes, idx.set_off, i, m, idx.config.L, idx.config.C)
