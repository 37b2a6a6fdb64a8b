"""ctypes loader for the C oracle (oracle/_build/liboracle.so) -- test infrastructure only."""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None


def build() -> str:
    subprocess.check_call(["make", "-s", "-C", _HERE])
    return os.path.join(_HERE, "_build", "liboracle.so")


def lib():
    global _LIB
    if _LIB is None:
        path = os.path.join(_HERE, "_build", "liboracle.so")
        if not os.path.exists(path):
            path = build()
        _LIB = ctypes.CDLL(path)
        _LIB.oracle_score.restype = ctypes.c_int
        _LIB.oracle_pairwise_sum.restype = ctypes.c_double
        _LIB.oracle_pairwise_sum.argtypes = [ctypes.c_void_p, ctypes.c_int64]
    return _LIB


def _p(a):
    return a.ctypes.data_as(ctypes.c_void_p) if a is not None else None


def pairwise_sum(a) -> float:
    a = np.ascontiguousarray(a, dtype=np.float64)
    return lib().oracle_pairwise_sum(_p(a), a.size)


def score(codes, set_off, qcodes, lut, sets=None, want_counts=False, threads=None):
    """Dense oracle scores: qcodes (n_qsets, m_q, L); sets (n_qsets, n_eval) or None."""
    codes = np.ascontiguousarray(codes, dtype=np.int32)
    set_off = np.ascontiguousarray(set_off, dtype=np.int64)
    qcodes = np.ascontiguousarray(qcodes, dtype=np.int32)
    lut = np.ascontiguousarray(lut, dtype=np.float64)
    n_qsets, m_q, L = qcodes.shape
    if sets is not None:
        sets = np.ascontiguousarray(sets, dtype=np.int64)
        n_eval = sets.shape[1]
    else:
        n_eval = len(set_off) - 1
    scores = np.zeros((n_qsets, n_eval), dtype=np.float64)
    counts = np.zeros((n_qsets, n_eval, m_q), dtype=np.uint16) if want_counts else None
    threads = threads or len(os.sched_getaffinity(0))
    lib().oracle_score(_p(codes), _p(set_off), _p(qcodes), _p(sets), _p(lut),
                       ctypes.c_int64(n_qsets), ctypes.c_int64(n_eval), ctypes.c_int64(m_q),
                       ctypes.c_int64(L), _p(scores), _p(counts), ctypes.c_int(threads))
    return (scores, counts) if want_counts else scores
