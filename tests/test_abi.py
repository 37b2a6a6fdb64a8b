"""The C-ABI library loads on CPU and exports exactly what include/dessert_b200.h declares."""

import ctypes
import subprocess

from paper_2210_15748_b200 import _lib


def test_library_loads_and_exports_every_header_symbol():
    lib = _lib.lib()
    declared = _lib.header_functions()
    assert len(declared) >= 15
    for name in declared:
        assert hasattr(lib, name), name
    assert sorted(_lib.SIGNATURES) == declared
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True,
                         text=True, check=True).stdout
    exported = {line.split()[-1] for line in out.splitlines() if " T " in line}
    assert set(declared) <= exported


def test_host_only_entry_points():
    lib = _lib.lib()
    assert lib.dsrt_version() == 100
    assert lib.dsrt_record_words(32, 8) == 8      # 8 planes x 1 word
    assert lib.dsrt_record_words(64, 7) == 16     # 7 x 2 = 14 -> 16 (16-byte records)
    assert lib.dsrt_record_words(32, 7) == 8
    assert lib.dsrt_record_words(32, 6) == 8
    assert lib.dsrt_record_words(8, 2) == 4
    assert lib.dsrt_record_words(0, 2) == 0
    assert lib.dsrt_topk_max_k() == 4096
    assert lib.dsrt_scan_workspace(10) >= 8
    assert lib.dsrt_prefilter_workspace(256, 32, 65536, 1_000_000, 4) > 0


def test_errors_map_to_reference_exceptions():
    import pytest
    lib = _lib.lib()
    rc = lib.dsrt_topk(None, 0, None, 0, None, 0, 1, 0, None, None, None, None)
    assert rc == _lib.EINVAL
    assert _lib.last_error().startswith("invalid parameter")
    with pytest.raises(ValueError, match="invalid parameter"):
        _lib.check(rc)
    rc = lib.dsrt_hash(None, 0, 1, 0, None, 0, 1, 1, None, None, None, None)
    assert rc == _lib.EINVAL and "d must be >= 1" in _lib.last_error()
    rc = lib.dsrt_prefilter(None, 1, 1, 4, None, 4, None, None, 1, None, 0, 5, None, None, None, 0,
                            None)
    assert rc == _lib.EINVAL and _lib.last_error().startswith("invalid parameter: probe")
    assert ctypes.sizeof(ctypes.c_void_p) == 8
