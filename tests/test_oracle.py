"""The CPU oracle (oracle/hcmx_oracle.c) pinned against the reference codec:
the committed golden fixtures (always) and the live reference build
oracle/_ref (where /root/reference exists)."""
import numpy as np
import pytest

from conftest import golden_cases, sha


def test_oracle_matches_golden_codec(oracle, codec_golden):
    n = 0
    for v, eps, s, e, m, scale, payload, dsha in golden_cases(codec_golden):
        b = oracle.compress(v, eps, s)
        assert (b.e, b.m) == (e, m), (eps, s)
        assert b.scale == scale or (np.isnan(b.scale) and np.isnan(scale))
        assert b.payload == payload, (eps, s, len(v))
        assert sha(oracle.decompress(b)) == dsha
        n += 1
    assert n > 300


def test_oracle_scalar_anchors(oracle, codec_golden):
    z = codec_golden
    for eps, m in zip(z["mbits_eps"], z["mbits"]):
        assert oracle.mantissa_bits_for(float(eps)) == m
    for (a, b, c), e in zip(z["ebits_stats"], z["ebits"]):
        assert oracle.exponent_bits_for_stats(a, b, int(c)) == e


def test_oracle_aplr_matches_golden(oracle, codec_golden):
    z = codec_golden
    meta, pay = z["aplr_meta"], z["aplr_payload"]
    po, mi, t = 0, 0, 0
    while f"aplr{t}_cfg" in z:
        rows, cols, k, s = (int(v) for v in z[f"aplr{t}_cfg"])
        W = z[f"aplr{t}_W"].reshape(k, rows).T
        X = z[f"aplr{t}_X"].reshape(k, cols).T
        bufs = oracle.aplr_compress(W, X, z[f"aplr{t}_sigma"], float(z[f"aplr{t}_eps"][0]), s)
        for b in bufs:
            r = meta[mi]
            assert (b.e, b.m, b.scale) == (r["e"], r["m"], r["scale"])
            n = int(r["plen"])
            assert b.payload == pay[po: po + n].tobytes()
            po += n
            mi += 1
        t += 1
    assert mi == len(meta)


def test_oracle_matvec_matches_golden(oracle, hmat_golden):
    from cpu_hmatrix import Flat
    f = Flat.from_npz(hmat_golden)
    x = hmat_golden["x"]
    y = oracle.hmat_matvec(f, 1.0, x, 0.0, np.zeros(f.n_rows))
    ref = hmat_golden["y"]
    assert np.linalg.norm(y - ref) <= 1e-14 * np.linalg.norm(ref)
    y2 = oracle.hmat_matvec(f, -0.5, x, 2.0, ref, threads=3)
    assert np.linalg.norm(y2 - hmat_golden["y2"]) <= 1e-14 * np.linalg.norm(hmat_golden["y2"])


def test_mt19937_64_pin(oracle, ref):
    assert oracle.mt64_raw(5489, 10000)[-1] == 9981545732273789042  # the C++ standard's check value
    for seed in (0, 1, 42, 2 ** 63 + 5):
        assert (oracle.mt64_raw(seed, 700) == ref.mt64_raw(seed, 700)).all()


@pytest.mark.parametrize("seed", range(6))
def test_oracle_vs_reference_random(oracle, ref, seed):
    rng = np.random.default_rng(seed)
    for trial in range(40):
        n = int(rng.integers(0, 600))
        lo, hi = sorted(rng.uniform(-300, 300, 2)) if trial % 5 == 0 else (-6, 0)
        v = np.sign(rng.standard_normal(n)) * 10 ** rng.uniform(lo, hi, n)
        if n > 4:
            v[rng.integers(0, n, 3)] = 0.0
            v[1] = -0.0
        for eps in (0.3, 1e-3, 1e-6, 1e-9, 1e-13, 1e-16):
            for s in range(4):
                a, b = oracle.compress(v, eps, s), ref.compress(v, eps, s)
                assert a == b, (n, eps, s)
                assert (oracle.decompress(a).view(np.uint64) == ref.decompress(b).view(np.uint64)).all()


def test_oracle_errors_match_reference(oracle, ref):
    for eps in (0.0, 1.0, -1e-4, float("nan")):
        with pytest.raises(ValueError):
            oracle.mantissa_bits_for(eps)
        with pytest.raises(ValueError):
            ref.mantissa_bits_for(eps)
    for bad in (np.array([1.0, np.nan]), np.array([np.inf, 1.0])):
        for o in (oracle, ref):
            with pytest.raises(ValueError):
                o.compress(bad, 1e-4, 0)
    from oracle import Buf, CorruptBufferError
    good = ref.compress(np.arange(1.0, 101.0), 1e-6, 1)
    short = Buf(good.scheme, good.e, good.m, good.scale, good.count, good.payload[:-3])
    for o in (oracle, ref):
        with pytest.raises(CorruptBufferError):
            o.decompress(short)


def test_oracle_matvec_vs_reference_glue(oracle, ref):
    from cpu_hmatrix import build_small_flat
    f, x = build_small_flat(n=640, eps=1e-6, scheme=2, use_ref=False, geometry="cube",
                            kernel="matern")
    y0 = np.random.default_rng(3).standard_normal(f.n_rows)
    for alpha, beta in ((1.0, 0.0), (0.7, -1.5), (0.0, 2.0)):
        a = oracle.hmat_matvec(f, alpha, x, beta, y0, threads=2)
        b = ref.hmat_matvec(f, alpha, x, beta, y0, threads=1)
        assert np.linalg.norm(a - b) <= 1e-13 * max(np.linalg.norm(b), 1e-300)


def test_half_conversions_match_reference(oracle, ref):
    """half.hpp float_to_half / half_to_float restated bit for bit (MP storage):
    every binary16 pattern, and floats around every rounding boundary"""
    import struct
    for h in range(0, 1 << 16, 7):
        a, b = oracle.half_to_float(h), ref.half_to_float(h)
        assert struct.pack("<f", a) == struct.pack("<f", b), h
    rng = np.random.default_rng(4)
    bits = np.concatenate([rng.integers(0, 1 << 32, 20000, dtype=np.uint64),
                           np.arange(0x33000000, 0x33800000, 997, dtype=np.uint64),   # denormal range
                           np.arange(0x477fe000, 0x47800100, 1, dtype=np.uint64)])   # overflow boundary
    for u in bits:
        f = struct.unpack("<f", struct.pack("<I", int(u)))[0]
        if f != f:  # NaN: both map it to inf; skip payload details
            continue
        assert oracle.float_to_half(f) == ref.float_to_half(f), hex(int(u))


def test_mp_partition_rule(oracle):
    """mixedprec.cpp:66-82 with the D-S-H roundoffs (mixedprec.hpp:23)"""
    delta = 1e-6
    sigma = np.array([1.0, 1e-3, 1e-5, 1.5e-6, 1e-6, 5e-7])
    # s*rho_i <= delta picks the cheapest group: 1.0 -> fp64 (6e-8 > 1e-6? no: 1*6e-8 <= 1e-6 -> fp32)
    r = oracle.mp_partition(sigma, delta)
    exp = [0, 0, 0]
    for s_ in sigma:
        if s_ <= delta:
            continue
        g = 2 if s_ * 4.9e-4 <= delta else (1 if s_ * 6.0e-8 <= delta else 0)
        exp[g] += 1
    assert list(r) == exp
