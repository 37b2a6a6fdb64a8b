"""SRP hashing -- drop-in for dessert.lsh (reference: pkg/src/dessert/lsh.py).

The family (seeded float64 Gaussian planes) and the count->similarity LUT are
host-side constants built exactly as the reference builds them
(lsh.py:54-66, :130-139) -- the LUT bytes are uploaded verbatim so device
scores are bit-identical.  ``hash_matrix`` runs the K1 kernel on the GPU.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib, engine

MAX_CONCAT_BITS = 24


@dataclass(frozen=True)
class SrpFamily:
    """L tables of C sign bits; planes (L*C, d) float64, row t*C + c (lsh.py:20-38)."""

    d: int
    C: int
    L: int
    seed: int
    planes: np.ndarray
    _dev: dict = field(default_factory=dict, repr=False, compare=False)

    @property
    def code_range(self) -> int:
        return 1 << self.C

    def device_planes(self, mode: int, device) -> torch.Tensor:
        """Planes converted for a hash mode, cached per (mode, device)."""
        key = (mode, str(device))
        t = self._dev.get(key)
        if t is None:
            p = torch.from_numpy(np.ascontiguousarray(self.planes))
            if mode in (_lib.HASH_F64, _lib.HASH_TC_FIX):  # TC_FIX splits them on the device
                t = p.to(device=device, dtype=torch.float64)
            elif mode == _lib.HASH_F32:
                t = p.to(device=device, dtype=torch.float32)
            elif mode in (_lib.HASH_TC_BF16X2, _lib.HASH_TC_F16X2):
                dt = torch.bfloat16 if mode == _lib.HASH_TC_BF16X2 else torch.float16
                hi = p.to(dt)
                lo = (p - hi.to(torch.float64)).to(dt)
                t = torch.stack([hi, lo]).contiguous().to(device)
            else:
                raise ValueError(f"invalid parameter: hash mode {mode}")
            self._dev[key] = t
        return t


@dataclass(frozen=True)
class SimLookup:
    """table[k] = (k/L)^(1/C), table[0] = 0 (lsh.py:41-51)."""

    C: int
    L: int
    table: np.ndarray


def sample_srp_family(d: int, C: int, L: int, seed: int) -> SrpFamily:
    """lsh.py:54-66 -- same RNG stream, so planes are bit-identical to the reference."""
    if d < 1:
        raise ValueError(f"invalid parameter: d must be >= 1, got {d}")
    if C < 1 or C > MAX_CONCAT_BITS:
        raise ValueError(f"invalid parameter: C must be in [1, {MAX_CONCAT_BITS}], got {C}")
    if L < 1:
        raise ValueError(f"invalid parameter: L must be >= 1, got {L}")
    planes = np.random.default_rng(seed).standard_normal((L * C, d))
    return SrpFamily(d=d, C=C, L=L, seed=seed, planes=planes)


def build_sim_lookup(C: int, L: int) -> SimLookup:
    """lsh.py:130-139 (numpy power, so the bytes match the reference exactly)."""
    if C < 1:
        raise ValueError(f"invalid parameter: C must be >= 1, got {C}")
    if L < 1:
        raise ValueError(f"invalid parameter: L must be >= 1, got {L}")
    k = np.arange(L + 1, dtype=np.float64)
    table = (k / L) ** (1.0 / C)
    table[0] = 0.0
    return SimLookup(C=C, L=L, table=table)


def default_mode(dtype, d: int = 128, C: int = 7, n: int = 0, L: int = 64) -> int:
    """Hash arithmetic per input dtype (K1).

    float32/float64 inputs hash in float64 against the float64 planes (exact).
    fp16 / bf16 inputs with d = 128, C <= 8 use the tcgen05 kernel with hi/lo
    split planes (two MMA passes; operand rounding <= 2^-17 relative, far inside
    the 1e-4 band).  HASH_TC_FIX (one fp16 MMA pass + an exact fix-up of the
    bits near zero) gives the same guarantee but measured slower (its epilogue,
    not the tensor pipe, is the bound: DESIGN.md K1), so it is opt-in.  Small
    batches (< 4096 rows) use float64 SIMT.
    """
    if d == 128 and C <= 8 and n >= 4096:
        if dtype == torch.bfloat16:
            return _lib.HASH_TC_BF16X2
        if dtype == torch.float16:
            return _lib.HASH_TC_F16X2
    return _lib.HASH_F64


def to_device_matrix(X, d: int, device="cuda") -> torch.Tensor:
    if isinstance(X, torch.Tensor):
        t = X if X.is_cuda else X.to(device)
        if t.dtype not in (torch.float32, torch.float64, torch.float16, torch.bfloat16):
            t = t.to(torch.float64)
    else:
        a = np.asarray(X)
        if a.dtype not in (np.float32, np.float64, np.float16):
            a = a.astype(np.float64)
        t = torch.from_numpy(np.ascontiguousarray(a)).to(device)
    if t.dim() != 2 or t.shape[1] != d:
        raise ValueError(
            f"dimension mismatch: expected (n, {d}) matrix, got shape {tuple(t.shape)}")
    return t.contiguous()


def hash_device(family: SrpFamily, X: torch.Tensor, mode: int | None = None, want_codes=True,
                want_records=True, check_zero=True):
    """Hash a CUDA matrix; raises the reference's 'zero vector' error."""
    mode = (default_mode(X.dtype, X.shape[1], family.C, X.shape[0], family.L) if mode is None
            else mode)
    planes = family.device_planes(mode, X.device)
    codes, recs, zero = engine.hash_vectors(X, planes, mode, family.L, family.C, want_codes,
                                            want_records, check_zero)
    if check_zero and int(zero.item()) != 0:
        raise ValueError("zero vector cannot be hashed (sign of zero projection undefined)")
    return codes, recs


def hash_matrix(family: SrpFamily, X) -> np.ndarray:
    """Drop-in for lsh.hash_matrix (lsh.py:90-106): (n, d) -> (n, L) int64 codes."""
    t = to_device_matrix(X, family.d)
    codes, _ = hash_device(family, t, want_records=False)
    out = codes.cpu().numpy()
    if out.dtype != np.uint8:
        out = out.view(np.uint16 if out.dtype == np.int16 else np.uint32)
    return out.astype(np.int64)


def hash_vector(family: SrpFamily, v) -> np.ndarray:
    """lsh.py:80-87."""
    v = np.asarray(v, dtype=np.float64)
    if v.shape != (family.d,):
        raise ValueError(
            f"dimension mismatch: expected vector of dim {family.d}, got shape {v.shape}")
    if not np.any(v):
        raise ValueError("zero vector cannot be hashed (sign of zero projection undefined)")
    return hash_matrix(family, v[None, :])[0]
