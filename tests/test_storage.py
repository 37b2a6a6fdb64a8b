""".dsri index files (row f2): byte-identical save, load -> query parity against
files written by the reference (tests/golden/storage.npz), corruption handling
as pkg/tests/test_storage.py:70-135 specifies.

The host header walk (dsrt_dsri_scan_sets) runs without a GPU; everything else
is marked gpu."""

import ctypes
import struct

import numpy as np
import pytest

import storage_inputs as SI
from conftest import load_golden
from paper_2210_15748_b200 import _lib

G = load_golden("storage.npz")
HEADER = struct.Struct("<IIIIQBBBBIIII")


def _scan(raw: bytes, n_docs=None):
    """Run the native host walk over the sets section of a .dsri file."""
    hdr = HEADER.unpack_from(raw, 4)
    C, L = hdr[2], hdr[3]
    pos = 4 + HEADER.size
    (n,) = struct.unpack_from("<Q", raw, pos)
    n = n if n_docs is None else n_docs
    pos += 8
    buf = np.frombuffer(raw, dtype=np.uint8)
    ids = np.zeros(n, np.uint64)
    sizes = np.zeros(n, np.int64)
    tt = np.zeros(n, np.int64)
    bad = np.zeros(4, np.uint32)
    err = ctypes.c_int(0)
    end = ctypes.c_size_t(0)
    k = _lib.lib().dsrt_dsri_scan_sets(buf.ctypes.data_as(ctypes.c_void_p), len(raw), pos, n, L, C,
                                       ids.ctypes.data_as(ctypes.c_void_p),
                                       sizes.ctypes.data_as(ctypes.c_void_p),
                                       tt.ctypes.data_as(ctypes.c_void_p),
                                       bad.ctypes.data_as(ctypes.c_void_p), ctypes.byref(err),
                                       ctypes.byref(end))
    return k, err.value, ids, sizes, tt, bad, end.value


def _file(name) -> bytes:
    return G[f"{name}_file"].tobytes()


@pytest.mark.parametrize("name", list(SI.CASES))
def test_host_walk_reads_reference_files(name):
    raw = _file(name)
    docs = SI.docs(name)
    k, err, ids, sizes, tt, _, end = _scan(raw)
    assert err == 0 and k == len(docs)
    assert list(ids) == [i for i, _ in docs]
    assert list(sizes) == [x.shape[0] for _, x in docs]
    # the TinyTable at tt[0] starts right after the first doc id
    assert tt[0] == 4 + HEADER.size + 8 + 8
    if SI.CASES[name][6] is None:
        assert end == len(raw)  # no prefilter block: the sets section ends the file


def test_host_walk_errors():
    raw = _file("wide")
    L, C = 8, 4
    base = 4 + HEADER.size + 8
    # truncated inside the first doc id / header / payload
    assert _scan(raw[: base + 4])[1] == 1
    assert _scan(raw[: base + 8 + 10])[1] == 2
    assert _scan(raw[: base + 8 + 24 + 5])[1] == 3
    # bad dimensions (m = 0), width flags, shape differing from the config
    for field, value, kind in [(0, 0, 4), (3, 3, 5), (1, L + 1, 6)]:
        b = bytearray(raw)
        struct.pack_into("<I", b, base + 8 + 4 * field, value)
        k, err, *_ = _scan(bytes(b))
        assert (k, err) == (0, kind)
    del C


# ------------------------------------------------------------------ GPU
@pytest.mark.gpu
@pytest.mark.parametrize("name", list(SI.CASES))
def test_save_is_byte_identical_to_reference(name, tmp_path):
    import paper_2210_15748_b200 as d
    dd, C, L, seed, inner, phi, fkw, _ = SI.CASES[name]
    filt = d.FilterConfig(enabled=fkw is not None, **(fkw or {}))
    cfg = d.IndexConfig(d=dd, C=C, L=L, seed=seed, inner_kind=inner, phi=phi, filter=filt)
    idx = d.build_index(SI.docs(name), cfg)
    path = tmp_path / "x.dsri"
    d.save_index(path, idx)
    got = path.read_bytes()
    want = _file(name)
    assert len(got) == len(want)
    assert got == want
    d.save_index(tmp_path / "y.dsri", idx)  # deterministic
    assert (tmp_path / "y.dsri").read_bytes() == got


@pytest.mark.gpu
@pytest.mark.parametrize("name", list(SI.CASES))
def test_load_reference_file_and_query(name, tmp_path):
    import paper_2210_15748_b200 as d
    path = tmp_path / "ref.dsri"
    path.write_bytes(_file(name))
    idx = d.load_index(path)
    dd, C, L, seed, inner, phi, fkw, _ = SI.CASES[name]
    assert idx.config == d.IndexConfig(
        d=dd, C=C, L=L, seed=seed, inner_kind=inner, phi=phi,
        filter=d.FilterConfig(enabled=fkw is not None, **(fkw or {})))
    for q, Q in enumerate(SI.queries(name)):
        res = d.query(idx, Q, top_k=5)
        assert [x for x, _ in res] == list(G[f"{name}_q{q}_ids"])
        assert [v for _, v in res] == list(G[f"{name}_q{q}_scores"])
    # round trip through our writer reproduces the file
    d.save_index(tmp_path / "again.dsri", idx)
    assert (tmp_path / "again.dsri").read_bytes() == _file(name)


@pytest.mark.gpu
def test_load_errors(tmp_path):
    import paper_2210_15748_b200 as d
    raw = _file("small_nofilter")
    p = tmp_path / "x.dsri"

    def load(b):
        p.write_bytes(bytes(b))
        return d.load_index(p)

    with pytest.raises(d.BadMagicError):
        load(b"WHAT" + b"\x00" * 64)
    b = bytearray(raw)
    b[4:8] = struct.pack("<I", 2)
    with pytest.raises(d.VersionMismatchError):
        load(b)
    # smash monotonicity of the first sketch's offsets (pkg/tests/test_storage.py:116-127)
    first_offsets = 48 + 8 + 8 + 24
    b = bytearray(raw)
    b[first_offsets + 1] = 200
    with pytest.raises(d.CorruptSketchError, match="monotone|span"):
        load(b)
    # offsets must span 0..m
    b = bytearray(raw)
    b[first_offsets] = 1
    with pytest.raises(d.CorruptSketchError, match="span"):
        load(b)
    # ids not a permutation: duplicate an id in the first table of the first set
    k, err, ids, sizes, tt, _, _ = _scan(raw)
    m0 = int(sizes[0])
    L, r = 16, 8
    id0 = int(tt[0]) + 24 + L * (r + 1)
    if m0 >= 2:
        b = bytearray(raw)
        b[id0 + 1] = b[id0]
        with pytest.raises(d.CorruptSketchError, match="permutation"):
            load(b)
    # the first failing set is reported: corrupt set 3's payload and set 5's header
    b = bytearray(raw)
    b[int(tt[3]) + 24 + 1] = 255          # offsets of set 3 out of order
    struct.pack_into("<I", b, int(tt[5]) + 4, L + 1)  # set 5: L differs from the config
    with pytest.raises(d.CorruptSketchError, match=f"set {ids[3]}"):
        load(b)
    # truncated files (pkg/tests/test_storage.py:129-135)
    filt = _file("small_filter")
    with pytest.raises(d.TruncatedFileError):
        load(filt[:-10])
    with pytest.raises(d.TruncatedFileError):
        load(raw[: int(tt[2]) + 10])
    with pytest.raises(d.TruncatedFileError, match="zero sets"):
        b = bytearray(raw[:48 + 8])
        struct.pack_into("<Q", b, 48, 0)
        load(b)
