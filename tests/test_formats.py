"""Wire / on-disk formats: APLR and MP lowrank serialization
(mixedprec.cpp:254-342) and the HCMX file.  Host-only (CPU)."""
import os
import struct

import numpy as np
import pytest


def _cb(b):
    from paper_2308_10960_b200.codec import CompressedBuffer, FormatDescriptor, Scheme
    return CompressedBuffer(FormatDescriptor(Scheme(b.scheme), b.e, b.m, b.scale), b.count, b.payload)


def test_aplr_serialization_layout(oracle, ref):
    """u32 rank, u8 scheme, 3 zero bytes, f64 sigma, then every W and X column in the
    reference codec's own wire format"""
    from paper_2308_10960_b200.formats import deserialize_aplr, serialize_aplr
    rng = np.random.default_rng(8)
    W, X = rng.standard_normal((40, 5)), rng.standard_normal((56, 5))
    sigma = np.array([3.0, 1.0, 0.2, 1e-3, 1e-5])
    bufs = oracle.aplr_compress(W, X, sigma, 1e-6, 1)
    wc, xc = [_cb(b) for b in bufs[:5]], [_cb(b) for b in bufs[5:]]
    got = serialize_aplr(sigma, 1, wc, xc)
    exp = struct.pack("<IB3x", 5, 1) + sigma.astype("<f8").tobytes() + b"".join(ref.serialize(b) for b in bufs)
    assert got == exp
    s2, sch, w2, x2, off = deserialize_aplr(got + b"tail", 0)
    assert off == len(got) and (s2 == sigma).all() and int(sch) == 1
    assert [b.payload for b in w2 + x2] == [b.payload for b in bufs]
    from paper_2308_10960_b200.codec import CorruptBufferError
    with pytest.raises(CorruptBufferError):
        deserialize_aplr(got[:-3])
    bad = bytearray(got)
    bad[4] = 9
    with pytest.raises(CorruptBufferError):
        deserialize_aplr(bytes(bad))


def test_mp_serialization_roundtrip(oracle):
    from paper_2308_10960_b200.formats import deserialize_mp, serialize_mp
    rng = np.random.default_rng(9)
    W, X = rng.standard_normal(30 * 4), rng.standard_normal(20 * 4)
    sigma = np.array([1.0, 0.1, 1e-4, 1e-5])
    groups = [(4, 1, oracle.pack_raw(W[:30], 4), oracle.pack_raw(X[:20], 4)),
              (5, 2, oracle.pack_raw(W[30:90], 5), oracle.pack_raw(X[20:60], 5)),
              (6, 1, oracle.pack_raw(W[90:], 6), oracle.pack_raw(X[60:], 6))]
    data = serialize_mp(sigma, groups)
    assert len(data) == 4 + 32 + 4 + 3 * 5 + (8 + 2 * 4 + 2) * 30 + (8 + 2 * 4 + 2) * 20
    s2, g2, off = deserialize_mp(data, 0, 30, 20)
    assert off == len(data) and (s2 == sigma).all() and g2 == groups


@pytest.mark.parametrize("mode,scheme", [("aplr", 0), ("aplr", 3), ("codec", 1), ("mp", 0), ("fp64", 0)])
def test_hcmx_file_roundtrip(oracle, tmp_path, mode, scheme):
    """save -> load keeps every leaf, buffer and byte; the product is unchanged"""
    from cpu_hmatrix import build_small_flat
    from paper_2308_10960_b200.formats import load_hcmx, save_hcmx
    f, x = build_small_flat(n=768, eps=1e-6, scheme=scheme, mode=mode)
    fp = f.to_product()
    path = os.path.join(tmp_path, "m.hcmx")
    save_hcmx(fp, path)
    g = load_hcmx(path)
    for k in ("row0", "row1", "col0", "col1", "kind", "rank", "count"):
        assert (getattr(g, k) == getattr(fp, k)).all(), k
    assert (g.desc == fp.desc).all()
    for b in range(fp.count.size):
        assert g.blob[g.poff[b]: g.poff[b] + g.plen[b]].tobytes() == \
            fp.blob[fp.poff[b]: fp.poff[b] + fp.plen[b]].tobytes(), b
    y0 = oracle.hmat_matvec(fp, 1.0, x, 0.0, np.zeros(768), threads=2)
    y1 = oracle.hmat_matvec(g, 1.0, x, 0.0, np.zeros(768), threads=2)
    assert (y0 == y1).all()


def test_hcmx_rejects_bad_files(tmp_path):
    from paper_2308_10960_b200.codec import CorruptBufferError
    from paper_2308_10960_b200.formats import load_hcmx
    p = os.path.join(tmp_path, "bad.hcmx")
    open(p, "wb").write(b"NOPE" + b"\0" * 40)
    with pytest.raises(CorruptBufferError):
        load_hcmx(p)
    open(p, "wb").write(b"HCMX" + struct.pack("<IQQQ", 1, 64, 64, 1) + b"\0\0")
    with pytest.raises(CorruptBufferError):
        load_hcmx(p)
