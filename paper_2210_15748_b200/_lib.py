"""ctypes binding of the C ABI declared in include/dessert_b200.h.

The shared library is built in-tree (``paper_2210_15748_b200/csrc/
libdessert_b200.so``, see ``__graft_entry__.build``).  There is no fallback:
if the library is missing or fails to load, every entry point raises.
Status codes map onto the reference's exception types (ValueError /
IndexError) with the C side's message, whose prefixes follow the reference
("invalid parameter", "dimension mismatch", "zero vector", ...).
"""

from __future__ import annotations

import ctypes
import os
import re

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("DSRT_LIB") or os.path.join(_HERE, "csrc", "libdessert_b200.so")
HEADER_PATH = os.path.join(os.path.dirname(_HERE), "include", "dessert_b200.h")

OK, EINVAL, ECUDA, EUNSUPPORTED, ERANGE = 0, 1, 2, 3, 4
F32, F64, F16, BF16 = 0, 1, 2, 3
HASH_F64, HASH_F32, HASH_TC_FIX, HASH_TC_BF16X2, HASH_TC_F16X2 = 0, 1, 2, 3, 4

_vp = ctypes.c_void_p
_i64 = ctypes.c_int64
_i32 = ctypes.c_int
_sz = ctypes.c_size_t

# name -> (restype, argtypes); must cover every function in the header.
SIGNATURES = {
    "dsrt_last_error": (ctypes.c_char_p, []),
    "dsrt_version": (_i32, []),
    "dsrt_record_words": (_i32, [_i32, _i32]),
    "dsrt_device_info": (_i32, [_vp, _vp, _vp, _vp]),
    "dsrt_copy_async": (_i32, [_vp, _vp, _sz, _vp]),
    "dsrt_pack4_async": (_i32, [_vp, _vp, _sz, _vp, _sz, _vp, _sz, _vp, _sz, _vp]),
    "dsrt_hash": (_i32, [_vp, _i32, _i64, _i32, _vp, _i32, _i32, _i32, _vp, _vp, _vp, _vp]),
    "dsrt_codes_to_records": (_i32, [_vp, _i32, _i64, _i32, _i32, _vp, _vp, _vp]),
    "dsrt_sizes_to_offsets": (_i32, [_vp, _i64, _vp, _vp, _vp, _sz, _vp]),
    "dsrt_scan_workspace": (_sz, [_i64]),
    "dsrt_counting_sort": (_i32, [_vp, _i64, _i64, _vp, _vp, _vp, _sz, _vp]),
    "dsrt_counting_sort_workspace": (_sz, [_i64, _i64]),
    "dsrt_gather_rows": (_i32, [_vp, _i64, _vp, _i64, _vp, _vp]),
    "dsrt_score_all": (_i32, [_vp, _vp, _i64, _i64, _vp, _i64, _i32, _i32, _i32, _vp, _vp, _i64,
                              _vp, _vp]),
    "dsrt_score_candidates": (_i32, [_vp, _vp, _i64, _vp, _vp, _i64, _vp, _i64, _i32, _i32, _i32,
                                     _vp, _vp, _vp, _vp]),
    "dsrt_score_agg_workspace": (_sz, [_i64, _i64, _i32, _i64]),
    "dsrt_score_agg": (_i32, [_vp, _vp, _i64, _vp, _vp, _i64, _vp, _i64, _i32, _i32, _i32, _i32,
                              _vp, _vp, _i64, _vp, _vp, _sz, _vp]),
    "dsrt_train_centroids_workspace": (_sz, [_i64, _i32, _i64]),
    "dsrt_train_centroids": (_i32, [_vp, _i64, _i32, _i64, _i32, _vp, _vp, _vp, _sz, _vp]),
    "dsrt_dsri_write_sets": (_i32, [_vp, _vp, _vp, _i64, _i32, _i32, _vp, _vp, _vp]),
    "dsrt_varint_workspace": (_sz, [_i64]),
    "dsrt_postings_to_varints": (_i32, [_vp, _vp, _i64, _i64, _vp, _vp, _vp, _sz, _vp]),
    "dsrt_dsri_scan_sets": (_i64, [_vp, _sz, _sz, _i64, _i32, _i32, _vp, _vp, _vp, _vp, _vp, _vp]),
    "dsrt_dsri_decode_sets": (_i32, [_vp, _vp, _vp, _i64, _i32, _i32, _i64, _vp, _i32, _vp, _vp]),
    "dsrt_varints_to_postings": (_i32, [_vp, _i64, _i64, _vp, _vp, _vp, _vp, _sz, _vp]),
    "dsrt_collision_counts": (_i32, [_vp, _vp, _i32, _i32, _i32, _vp, _i32, _vp, _vp]),
    "dsrt_topk": (_i32, [_vp, _i64, _vp, _i64, _vp, _i64, _i64, _i32, _vp, _vp, _vp, _vp]),
    "dsrt_topk_max_k": (_i32, []),
    "dsrt_search_all_workspace": (_sz, [_i64, _i64, _i32, _i32, _i32, _sz]),
    "dsrt_search_profile": (None, [_i32]),
    "dsrt_search_profile_read": (_i32, [_vp, _vp, _vp]),
    "dsrt_search_all": (_i32, [_vp, _vp, _i64, _vp, _vp, _i64, _i32, _i32, _i32, _vp, _vp, _i32,
                               _i32, _sz, _vp, _vp, _vp, _vp, _sz, _vp]),
    "dsrt_topk_indexed": (_i32, [_vp, _i64, _vp, _vp, _i64, _vp, _i64, _i64, _i32, _vp, _vp, _vp, _vp]),
    "dsrt_prefilter": (_i32, [_vp, _i64, _i32, _i32, _vp, _i64, _vp, _vp, _i64, _vp, _i32, _i32,
                              _vp, _vp, _vp, _sz, _vp]),
    "dsrt_prefilter_workspace": (_sz, [_i64, _i32, _i64, _i64, _i32]),
    "dsrt_prefilter_tc": (_i32, [_vp, _i64, _i32, _i32, _vp, _vp, ctypes.c_double, _i64, _vp, _vp,
                                 _i64, _vp, _i32, _i32, _vp, _vp, _vp, _sz, _vp]),
    "dsrt_posting_chunk_bounds_size": (_i64, [_i64, _i64, _i32, _i32]),
    "dsrt_posting_chunk_bounds": (_i32, [_vp, _vp, _i64, _i64, _i32, _i32, _vp, _vp]),
    "dsrt_prefilter_tc_workspace": (_sz, [_i64, _i32, _i64, _i64, _i32]),
    "dsrt_to_f16_rows": (_i32, [_vp, _i64, _i32, ctypes.c_double, _vp, _vp]),
    "dsrt_to_bf16_rows": (_i32, [_vp, _i64, _i32, ctypes.c_double, _vp, _vp]),
    "dsrt_assign_centroids": (_i32, [_vp, _i32, _i64, _i32, _vp, _vp, _i64, _vp, _vp, _sz, _vp]),
    "dsrt_assign_centroids_workspace": (_sz, [_i64, _i32, _i64]),
    "dsrt_merge_postings": (_i32, [_vp, _vp, _vp, _vp, _i64, _vp, _vp, _vp]),
    "dsrt_postings_from_assign": (_i32, [_vp, _i64, _vp, _i64, _i64, _vp, _vp, _vp, _vp, _sz, _vp]),
    "dsrt_postings_workspace": (_sz, [_i64, _i64]),
    "dsrt_tinytable": (_i32, [_vp, _i32, _vp, _i64, _i32, _i32, _vp, _vp, _vp]),
    "dsrt_microbench_int": (_i32, [_vp, _vp]),
    "dsrt_tc_selftest": (_i32, [_vp, _i32, _vp, _i32, _vp, _i32, _i32, _vp]),
}

_LIB = None


class LibraryMissing(RuntimeError):
    pass


def header_functions() -> list[str]:
    """Function names declared in include/dessert_b200.h."""
    with open(HEADER_PATH) as f:
        text = f.read()
    return sorted(set(re.findall(r"\b(dsrt_[a-z0-9_]+)\s*\(", text)))


def lib():
    global _LIB
    if _LIB is None:
        if not os.path.exists(LIB_PATH):
            raise LibraryMissing(
                f"{LIB_PATH} not built: run `python -c 'import __graft_entry__ as g; g.build()'`"
                " (no CPU fallback exists)")
        handle = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(handle, name)
            fn.restype = res
            fn.argtypes = args
        _LIB = handle
    return _LIB


def last_error() -> str:
    msg = lib().dsrt_last_error()
    return msg.decode() if msg else ""


def check(rc: int) -> None:
    if rc == OK:
        return
    msg = last_error()
    if rc == EINVAL:
        raise ValueError(msg)
    if rc == ERANGE:
        raise IndexError(msg)
    if rc == EUNSUPPORTED:
        raise NotImplementedError(msg)
    raise RuntimeError(msg)


def call(name: str, *args) -> None:
    check(getattr(lib(), name)(*args))
