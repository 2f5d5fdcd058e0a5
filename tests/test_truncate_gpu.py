"""Semi-on-the-fly truncation (Algorithm 4; SPEC.md:551-559
truncate_compressed): decompress -> QR / SVD -> rank rule -> APLR compress, on
the device.  Checked against the uncompressed truncation of the decompressed
factors (same ranks, Frobenius distance within the codec bound), idempotence,
zero factors and the sum of two blocks sharing a column space."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _blocks(B, m, n, k, decay, seed):
    rng = np.random.default_rng(seed)
    U = np.empty((B, m, k)); V = np.empty((B, n, k))
    for b in range(B):
        q1, _ = np.linalg.qr(rng.standard_normal((m, k)))
        q2, _ = np.linalg.qr(rng.standard_normal((n, k)))
        s = decay ** np.arange(k) * (1.0 + b)
        U[b] = q1 * s
        V[b] = q2
    return U, V


def _compress(F, eps):
    from paper_2308_10960_b200.codec import Scheme, compress_batch
    B, r, k = F.shape
    cm = np.ascontiguousarray(F.transpose(0, 2, 1)).reshape(-1)   # column-major per block
    return compress_batch(torch.as_tensor(cm).cuda(), np.full(B, r * k, np.uint64), eps, Scheme.afl)


def _host(bb, B, r, k):
    from paper_2308_10960_b200.codec import decompress_batch
    return decompress_batch(bb).cpu().numpy().reshape(B, k, r).transpose(0, 2, 1)


def _rank(s, eps):
    return int(np.sum(np.cumprod((s > eps * s[0]) & (s[0] > 0))))


@pytest.mark.parametrize("eps", [1e-4, 1e-6])
def test_truncate_matches_uncompressed(gpu, eps):
    from paper_2308_10960_b200.arith import truncate_compressed
    B, m, n, k = 6, 128, 96, 24
    U, V = _blocks(B, m, n, k, 0.3, 3)   # no singular value next to a threshold
    Uc, Vc = _compress(U, 1e-10), _compress(V, 1e-10)
    tb = truncate_compressed(Uc, Vc, m, n, k, eps)
    Ud, Vd = _host(Uc, B, m, k), _host(Vc, B, n, k)
    for b in range(B):
        M = Ud[b] @ Vd[b].T
        u, s, vt = np.linalg.svd(M)
        kr = _rank(s, eps)
        assert tb.rank[b] == kr, (b, tb.rank[b], kr)
        W, sig, X = tb.factors(b)
        best = (u[:, :kr] * s[:kr]) @ vt[:kr]
        # codec bound: each column within its APLR precision eps_i = eps s_0 / s_i
        assert np.linalg.norm((W * sig) @ X.T - best) <= 10 * kr * eps * s[0], b
        assert np.allclose(sig, s[:kr], rtol=1e-9, atol=0)


def test_truncate_idempotent_and_degenerate(gpu):
    from paper_2308_10960_b200.arith import truncate_compressed
    B, m, n, k, eps = 4, 64, 64, 16, 1e-6
    U, V = _blocks(B, m, n, k, 0.3, 5)
    tb = truncate_compressed(_compress(U, 1e-12), _compress(V, 1e-12), m, n, k, eps)
    k1 = int(tb.rank.max())
    assert (tb.rank == tb.rank[0]).all() and 0 < k1 < k
    # truncating the (decompressed) output again keeps every rank
    U2 = np.zeros((B, m, k1)); V2 = np.zeros((B, n, k1))
    for b in range(B):
        W, sig, X = tb.factors(b)
        U2[b], V2[b] = W * sig, X
    tb2 = truncate_compressed(_compress(U2, 1e-12), _compress(V2, 1e-12), m, n, k1, eps)
    assert (tb2.rank == tb.rank).all()
    # zero factors -> rank 0; U1 V1^T + (-U1) V1^T -> rank 0 (the sum cancels exactly)
    Z = np.zeros((2, m, 4))
    tz = truncate_compressed(_compress(Z, 1e-6), _compress(np.ones((2, n, 4)), 1e-6), m, n, 4, eps)
    assert (tz.rank == 0).all()
    # a sum of two blocks with one column space, U1 V1^T + U1 (2 V1)^T = 3 U1 V1^T
    # (the H-arithmetic update): the concatenated rank-8 factors truncate to 4
    Us = np.concatenate([U[:2, :, :4], U[:2, :, :4]], axis=2)
    Vs = np.concatenate([V[:2, :, :4], 2 * V[:2, :, :4]], axis=2)
    tc = truncate_compressed(_compress(Us, 1e-12), _compress(Vs, 1e-12), m, n, 8, eps)
    assert (tc.rank == 4).all()
    for b in range(2):
        W, sig, X = tc.factors(b)
        ref = 3 * U[b, :, :4] @ V[b, :, :4].T
        assert np.linalg.norm((W * sig) @ X.T - ref) <= 1e-5 * np.linalg.norm(ref)
