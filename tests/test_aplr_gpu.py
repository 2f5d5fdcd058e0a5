"""APLR (mixedprec.cpp:155-187) on the GPU: per-column layouts and packed
bytes identical to the reference glue on given factors."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _gpu_aplr(cases, eps, scheme):
    """batched hcmx_gpu_aplr_compress over several leaves -> per leaf list of buffers"""
    import ctypes as C
    from paper_2308_10960_b200 import _lib
    from paper_2308_10960_b200._lib import DESC_DTYPE, check, lib, ptr, u64p
    rows = np.array([c[0].shape[0] for c in cases], np.uint64)
    cols = np.array([c[1].shape[0] for c in cases], np.uint64)
    ks = np.array([c[0].shape[1] for c in cases], np.uint64)
    W = np.concatenate([c[0].ravel(order="F") for c in cases] + [np.zeros(1)])
    X = np.concatenate([c[1].ravel(order="F") for c in cases] + [np.zeros(1)])
    S = np.concatenate([c[2] for c in cases] + [np.zeros(1)])
    wo = np.concatenate([[0], np.cumsum(rows * ks)[:-1]]).astype(np.uint64)
    xo = np.concatenate([[0], np.cumsum(cols * ks)[:-1]]).astype(np.uint64)
    so = np.concatenate([[0], np.cumsum(ks)[:-1]]).astype(np.uint64)
    bo = np.concatenate([[0], np.cumsum(2 * ks)[:-1]]).astype(np.uint64)
    nb = int(2 * ks.sum())
    dW, dX = torch.as_tensor(W).cuda(), torch.as_tensor(X).cuda()
    cap = 8 * (W.size + X.size) + 16 * nb + 64
    pay = torch.zeros(cap, dtype=torch.uint8, device="cuda")
    desc = np.zeros(max(nb, 1), DESC_DTYPE)
    poff = np.zeros(max(nb, 1), np.uint64)
    tot = C.c_uint64()
    check(lib().hcmx_gpu_aplr_compress(len(cases), u64p(rows), u64p(cols), u64p(ks), ptr(dW), u64p(wo),
                                       ptr(dX), u64p(xo), ptr(S), u64p(so), u64p(bo), eps, scheme,
                                       ptr(pay), cap, ptr(desc), u64p(poff), C.byref(tot),
                                       torch.cuda.current_stream().cuda_stream), "aplr")
    host = pay.cpu().numpy()
    out = []
    for j in range(len(cases)):
        bufs = []
        for i in range(int(2 * ks[j])):
            b = int(bo[j]) + i
            cnt = int(rows[j]) if i < ks[j] else int(cols[j])
            n = (cnt * int(desc["bit_width"][b]) + 7) // 8
            bufs.append((int(desc["exp_bits"][b]), int(desc["mant_bits"][b]), float(desc["scale"][b]),
                         host[int(poff[b]): int(poff[b]) + n].tobytes()))
        out.append(bufs)
    return out


def test_aplr_golden(gpu, codec_golden):
    z = codec_golden
    meta, pay = z["aplr_meta"], z["aplr_payload"]
    po = mi = t = 0
    while f"aplr{t}_cfg" in z:
        rows, cols, k, s = (int(v) for v in z[f"aplr{t}_cfg"])
        W = z[f"aplr{t}_W"].reshape(k, rows).T
        X = z[f"aplr{t}_X"].reshape(k, cols).T
        got = _gpu_aplr([(W, X, z[f"aplr{t}_sigma"])], float(z[f"aplr{t}_eps"][0]), s)[0]
        for e, m, scale, p in got:
            r = meta[mi]
            assert (e, m, scale) == (r["e"], r["m"], r["scale"])
            n = int(r["plen"])
            assert p == pay[po: po + n].tobytes()
            po += n
            mi += 1
        t += 1
    assert mi == len(meta)


def test_aplr_widths_follow_sigma(gpu):  # test_mixedprec.cpp:142-156
    rng = np.random.default_rng(5)
    W, _ = np.linalg.qr(rng.standard_normal((48, 3)))
    X, _ = np.linalg.qr(rng.standard_normal((40, 3)))
    got = _gpu_aplr([(W, X, np.array([1.0, 1e-2, 1e-3]))], 1e-8, 0)[0]
    assert got[0][1] == 26 and got[2][1] == 16
    assert got[0][1] >= got[1][1] >= got[2][1]


@pytest.mark.parametrize("scheme", [0, 1, 2, 3])
def test_aplr_batch_vs_oracle(gpu, oracle, scheme):
    rng = np.random.default_rng(scheme)
    cases = []
    for _ in range(40):
        rows, cols = int(rng.integers(1, 300)), int(rng.integers(1, 300))
        k = int(rng.integers(0, min(rows, cols, 20) + 1))
        W = rng.standard_normal((rows, k)) * 10 ** rng.uniform(-3, 3)
        X = rng.standard_normal((cols, k))
        sig = np.sort(10 ** rng.uniform(-9, 0, k))[::-1].copy()
        cases.append((W, X, sig))
    got = _gpu_aplr(cases, 1e-7, scheme)
    for (W, X, sig), g in zip(cases, got):
        exp = oracle.aplr_compress(W, X, sig, 1e-7, scheme) if W.shape[1] else []
        assert len(g) == len(exp)
        for (e, m, scale, p), ob in zip(g, exp):
            assert (e, m, scale) == (ob.e, ob.m, ob.scale)
            assert p == ob.payload
