"""CUDA codec parity: packed bytes and decoded FP64 bits identical to the
reference codec (golden fixtures) and to the pinned oracle, at the BASELINE
config-2 size, plus the reference test_codec.cpp cases restated."""
import numpy as np
import pytest
import torch

from conftest import golden_cases, sha

pytestmark = pytest.mark.gpu


def test_golden_single_buffer_host_api(gpu, codec_golden):
    from paper_2308_10960_b200 import codec
    n = 0
    for v, eps, s, e, m, scale, payload, dsha in golden_cases(codec_golden):
        b = codec.compress(v, eps, s)
        assert (b.descriptor.exp_bits, b.descriptor.mant_bits) == (e, m)
        assert b.descriptor.scale == scale
        assert b.payload == payload, (len(v), eps, s)
        assert sha(codec.decompress(b)) == dsha
        n += 1
    assert n > 300


def test_golden_batched_device_api(gpu, codec_golden):
    """all golden cases of one (eps, scheme) as ONE batch through the HBM-resident API"""
    from paper_2308_10960_b200 import codec
    groups = {}
    for v, eps, s, e, m, scale, payload, dsha in golden_cases(codec_golden):
        groups.setdefault((eps, s), []).append((v, e, m, scale, payload, dsha))
    for (eps, s), items in groups.items():
        vals = np.concatenate([it[0] for it in items])
        counts = np.array([len(it[0]) for it in items], np.uint64)
        bb = codec.compress_batch(torch.as_tensor(vals).cuda(), counts, eps, s)
        host = bb.payload.cpu().numpy()
        dec = codec.decompress_batch(bb).cpu().numpy()
        o = 0
        for b, (v, e, m, scale, payload, dsha) in enumerate(items):
            got = bb.buffer(b, host)
            assert (got.descriptor.exp_bits, got.descriptor.mant_bits, got.descriptor.scale) == (e, m, scale)
            assert got.payload == payload
            assert sha(dec[o: o + len(v)]) == dsha
            o += len(v)


@pytest.mark.parametrize("eps", [1e-4, 1e-6, 1e-8])
def test_config2_full_size_bit_exact(gpu, oracle, eps):
    """BASELINE config 2: 4096 blocks of 64x64, sign * 10^U[-6,0], every scheme"""
    from paper_2308_10960_b200 import codec
    nb, bs = 4096, 4096
    vals = oracle.config2_values(2, nb * bs)
    d_vals = torch.as_tensor(vals).cuda()
    counts = np.full(nb, bs, np.uint64)
    for s in range(4):
        bb = codec.compress_batch(d_vals, counts, eps, s)
        e, m, sc, poff, blob = oracle.compress_batch(vals, counts, eps, s, threads=8)
        assert (bb.desc["exp_bits"] == e).all() and (bb.desc["mant_bits"] == m).all()
        assert (bb.desc["scale"] == sc).all()
        host = bb.payload.cpu().numpy()
        w = int(bb.desc["bit_width"][0])
        plen = (bs * w + 7) // 8
        assert (bb.desc["bit_width"] == w).all()
        got = host[(bb.poff[:, None] + np.arange(plen)[None, :]).astype(np.int64)]
        exp = blob[(poff[:, None] + np.arange(plen)[None, :]).astype(np.int64)]
        assert (got == exp).all(), (eps, s)
        dec = codec.decompress_batch(bb).cpu().numpy()
        ref = oracle.decompress_batch(blob, poff, counts, s, e, m, sc, threads=8)
        assert (dec.view(np.uint64) == ref.view(np.uint64)).all()


def test_random_ragged_batches(gpu, oracle):
    from paper_2308_10960_b200 import codec
    rng = np.random.default_rng(7)
    for trial in range(6):
        nb = int(rng.integers(1, 300))
        counts = rng.integers(0, 3000, nb).astype(np.uint64)
        counts[rng.integers(0, nb)] = 40000  # multi-job buffer
        n = int(counts.sum())
        lo, hi = sorted(rng.uniform(-200, 200, 2))
        v = np.sign(rng.standard_normal(n)) * 10 ** rng.uniform(lo, hi, n)
        v[rng.integers(0, max(n, 1), n // 50 + 1)] = 0.0
        for eps in (0.2, 1e-5, 1e-11, 1e-16):
            s = int(rng.integers(0, 4))
            bb = codec.compress_batch(torch.as_tensor(v).cuda(), counts, eps, s)
            host = bb.payload.cpu().numpy()
            dec = codec.decompress_batch(bb).cpu().numpy()
            o = 0
            for b in range(nb):
                c = int(counts[b])
                ob = oracle.compress(v[o: o + c], eps, s)
                g = bb.buffer(b, host)
                assert (g.descriptor.exp_bits, g.descriptor.mant_bits, g.descriptor.scale) == (ob.e, ob.m, ob.scale)
                assert g.payload == ob.payload
                assert (dec[o: o + c].view(np.uint64) == oracle.decompress(ob).view(np.uint64)).all()
                o += c


def test_pinned_layouts_and_saturation(gpu, oracle):
    """compress_block with fixed layouts: BFL/DFL saturation, subnormal scale, m=52"""
    from paper_2308_10960_b200 import codec
    rng = np.random.default_rng(3)
    v = np.sign(rng.standard_normal(999)) * 10 ** rng.uniform(-300, 300, 999)
    for s, e, m, scale in [(2, 8, 15, 1e-300), (3, 11, 52, 5e-324), (0, 3, 4, 1.0), (0, 11, 52, 1e-3),
                           (1, 2, 5, 7.0), (3, 11, 20, 1e-10), (0, 5, 40, 1e-200)]:
        d = codec.FormatDescriptor(codec.Scheme(s), e, m, scale)
        w = d.bit_width()
        if w > 64:
            continue
        g = codec.compress_block(v, d)
        assert g.payload == oracle.compress_block(v, s, e, m, scale), (s, e, m, scale)
        from oracle import Buf
        ref = oracle.decompress(Buf(s, e, m, scale, v.size, g.payload))
        assert (codec.decompress(g).view(np.uint64) == ref.view(np.uint64)).all()


def test_rejects_non_finite_and_bad_eps(gpu):
    from paper_2308_10960_b200 import codec
    with pytest.raises(ValueError):
        codec.compress(np.array([1.0, np.nan]), 1e-4, codec.Scheme.afl)
    with pytest.raises(ValueError):
        codec.compress(np.array([1.0, np.inf]), 1e-4, codec.Scheme.dfl)
    with pytest.raises(ValueError):
        codec.compress(np.array([1.0, 2.0]), 1.0, codec.Scheme.afl)
    with pytest.raises(ValueError):
        codec.compress_batch(torch.tensor([1.0, -np.inf, 3.0]).cuda(), [2, 1], 1e-6, 0)
    b = codec.compress(np.arange(1.0, 101.0), 1e-6, codec.Scheme.aflp)
    short = codec.CompressedBuffer(b.descriptor, b.count, b.payload[:-3])
    with pytest.raises(codec.CorruptBufferError):
        codec.decompress(short)


# ---- proj/tests/test_codec.cpp restated on the CUDA path ----------------
def test_constants_zeros_and_negative_zero(gpu):  # test_codec.cpp:62-78
    from paper_2308_10960_b200 import codec
    for s in codec.Scheme:
        out = codec.decompress(codec.compress([7.5] * 5, 1e-2, s))
        assert (out == 7.5).all()
        back = codec.decompress(codec.compress([0.0, -1.25, 1.25, -0.0, 0.0], 1e-4, s))
        assert back[0] == 0.0 and not np.signbit(back[0])
        assert np.signbit(back[1]) and np.signbit(back[3])
        assert back[2] == 1.25 and back[1] == -1.25


def test_empty_block(gpu):  # test_codec.cpp:80-86
    from paper_2308_10960_b200 import codec
    for s in codec.Scheme:
        b = codec.compress(np.zeros(0), 1e-4, s)
        assert b.count == 0 and codec.decompress(b).size == 0


def test_afl_equals_mask_mantissa(gpu, oracle):  # test_codec.cpp:88-103
    from paper_2308_10960_b200 import codec
    v = oracle.log_uniform_signed(42, 4096, 1.0, 1e4)
    eps = 1e-4
    m = codec.mantissa_bits_for(eps)
    b = codec.compress(v, eps, codec.Scheme.afl)
    out = codec.decompress(b)
    mn = codec.analyze(v).min_mag
    bound = 2.0 ** -(m + 1)

    def mask_mantissa(x):  # oracles.hpp:21-32 (divides by min_mag)
        if x == 0.0:
            return x
        u = np.float64(abs(x) / mn + 1.0).view(np.uint64)
        u = np.uint64(u + np.uint64(1 << (51 - m))) & ~np.uint64((1 << (52 - m)) - 1)
        back = (u.view(np.float64) - 1.0) * mn
        return -back if np.signbit(x) else back

    for i in range(v.size):
        assert out[i] == mask_mantissa(v[i])
        assert abs(out[i] - v[i]) <= bound * (abs(v[i]) + mn)


def test_error_bound_all_schemes(gpu, oracle):  # test_codec.cpp:105-119
    from paper_2308_10960_b200 import codec
    rng_seed = 7
    for eps in (1e-2, 1e-4, 1e-6, 1e-8):
        m = codec.mantissa_bits_for(eps)
        u = 2.0 ** -(m + 1)
        for s in codec.Scheme:
            rng_seed += 1
            v = oracle.log_uniform_signed(rng_seed, 512, 1e-3, 1e3)
            v[17] = 0.0
            mn = codec.analyze(v).min_mag
            out = codec.decompress(codec.compress(v, eps, s))
            assert (np.abs(out - v) <= u * (np.abs(v) + mn)).all()


def test_determinism(gpu, oracle):  # test_codec.cpp:167-176
    from paper_2308_10960_b200 import codec
    v = oracle.log_uniform_signed(3, 333, 1e-2, 1e5)
    for s in codec.Scheme:
        a, b = codec.compress(v, 1e-5, s), codec.compress(v, 1e-5, s)
        assert a.payload == b.payload and a.descriptor.scale == b.descriptor.scale


def test_analyze_matches_reference(gpu, oracle):
    from paper_2308_10960_b200 import codec
    rng = np.random.default_rng(0)
    for v in (np.zeros(7), rng.standard_normal(5000), np.array([0.0, -3.0, 1e-310, 2.0]),
              np.array([0.0, np.inf, 2.0])):
        st = codec.analyze(v)
        assert (st.min_mag, st.max_mag, st.all_zero) == oracle.analyze(v)


def test_large_buffers_unfused_path(gpu, oracle):
    """buffers above the fused kernel's 2^17 values go through device analyze +
    host layout selection + device pack; mixed with small ones in one batch"""
    from paper_2308_10960_b200 import codec
    rng = np.random.default_rng(11)
    counts = np.array([300000, 5, 140000, 0, 4096], np.uint64)
    n = int(counts.sum())
    v = np.sign(rng.standard_normal(n)) * 10 ** rng.uniform(-9, 3, n)
    v[::97] = 0.0
    for eps, s in ((1e-6, 0), (1e-9, 2), (1e-3, 3)):
        bb = codec.compress_batch(torch.as_tensor(v).cuda(), counts, eps, s)
        host = bb.payload.cpu().numpy()
        dec = codec.decompress_batch(bb).cpu().numpy()
        o = 0
        for b in range(counts.size):
            c = int(counts[b])
            ob = oracle.compress(v[o: o + c], eps, s)
            g = bb.buffer(b, host)
            assert (g.descriptor.exp_bits, g.descriptor.mant_bits) == (ob.e, ob.m), (eps, s, b)
            assert g.payload == ob.payload, (eps, s, b)
            assert (dec[o: o + c].view(np.uint64) == oracle.decompress(ob).view(np.uint64)).all()
            o += c


def test_exponent_width_thresholds(gpu, oracle):
    """exponent_bits_for (codec.cpp:69-79) flips only where log2(max) - log2(min) + 2
    crosses a power of two; blocks whose max / min sits exactly on (or one ulp
    either side of) 2^6, 2^14, 2^30, 2^62 take the device's ambiguity flag and the
    host re-decision (glibc log2, as the reference) -- descriptors and bytes must
    still equal the oracle's"""
    from paper_2308_10960_b200 import codec
    rng = np.random.default_rng(21)
    blocks = []
    for span in (6, 14, 30, 62):
        for lo in (1.0, 3.7, 1e-100, 2.0 ** -40):
            hi = lo * 2.0 ** span
            for top in (hi, np.nextafter(hi, 0.0), np.nextafter(hi, np.inf)):
                v = lo * 2.0 ** rng.uniform(0, span, 257)
                v[0], v[1] = lo, top
                v *= np.sign(rng.standard_normal(v.size))
                blocks.append(v)
    counts = np.array([b.size for b in blocks], np.uint64)
    vals = np.concatenate(blocks)
    for s in (0, 1):
        bb = codec.compress_batch(torch.as_tensor(vals).cuda(), counts, 1e-6, s)
        host = bb.payload.cpu().numpy()
        for i, v in enumerate(blocks):
            r = oracle.compress(v, 1e-6, s)
            got = bb.buffer(i, host)
            assert (got.descriptor.exp_bits, got.descriptor.mant_bits, got.descriptor.scale) == (r.e, r.m, r.scale), i
            assert got.payload == r.payload, i


def test_compress_device_api_bit_exact(gpu, oracle):
    """hcmx_gpu_codec_compress_device (no read-back) + the fix-up: the same bytes
    and descriptors as the oracle, including blocks on exponent thresholds (which
    the fix-up re-decides with the host rule) and an all-zero block"""
    from paper_2308_10960_b200 import codec
    rng = np.random.default_rng(5)
    blocks = [np.sign(rng.standard_normal(4096)) * 10 ** rng.uniform(-6, 0, 4096) for _ in range(40)]
    for span in (6, 14):
        v = 2.0 ** rng.uniform(0, span, 300)
        v[0], v[1] = 1.0, 2.0 ** span
        blocks.append(v)
    blocks.append(np.zeros(100))
    counts = np.array([b.size for b in blocks], np.uint64)
    vals = torch.as_tensor(np.concatenate(blocks)).cuda()
    for s in (0, 1, 3):
        db = codec.device_batch(vals, counts, 1e-6, s)
        codec.compress_device(vals, db)
        flags = db.d_flags.cpu().numpy()
        if s != 3:  # DFL fixes e = 11: nothing to decide
            assert (flags[-3:-1] & 1).all()
        assert not (flags[:40] & 1).any()
        bb, nfix = codec.compress_device_finish(vals, db)
        host = bb.payload.cpu().numpy()
        for i, v in enumerate(blocks):
            r = oracle.compress(v, 1e-6, s)
            got = bb.buffer(i, host)
            assert (got.descriptor.exp_bits, got.descriptor.mant_bits, got.descriptor.scale) == (r.e, r.m, r.scale), (s, i)
            assert got.payload == r.payload, (s, i)
    bad = vals.clone()
    bad[5] = float("nan")
    db = codec.device_batch(bad, counts, 1e-6, 0)
    codec.compress_device(bad, db)
    with pytest.raises(ValueError):
        codec.compress_device_finish(bad, db)
