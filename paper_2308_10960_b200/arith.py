"""Semi-on-the-fly lowrank truncation (Algorithm 4;
SPEC.md:551-559 `truncate_compressed`) -- the building block of compressed
H-arithmetic, batched on the device:

    [U, V]   := decompress[U^c, V^c]          (the codec decompress kernel)
    [Q_U, R_U] := qr(U),  [Q_V, R_V] := qr(V) (cuSOLVER, batched)
    [U_s, S_s, V_s] := svd(R_U R_V^T)
    k := rank(S_s)                            (lowrank.cpp:14-21: S_k > eps S_0)
    W := Q_U U_s(:, 1:k),  X := Q_V V_s(:, 1:k)
    [W^c, X^c] := compress[W, X]              (APLR: per-column precision from S_s)

With APLR storage the multiplication by S_s is omitted: the representation keeps
Sigma separate.  The dense linear algebra is library code
(torch.linalg on cuSOLVER); the conversions are this package's kernels.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np
import torch

from ._lib import DESC_DTYPE, check, lib, ptr, u64p
from .assemble import rank_from_singular_values
from .codec import BatchBuffers, Scheme, decompress_batch


@dataclass
class TruncatedBatch:
    """APLR blocks W diag(sigma) X^T (mixedprec.hpp:68-82) for a batch of B blocks:
    block b owns buffers boff[b] .. boff[b] + 2 rank[b] (W columns, then X columns)"""
    m: int
    n: int
    rank: np.ndarray          # int64 [B]
    sigma: np.ndarray         # float64, concatenated per block
    sig_off: np.ndarray       # int64 [B]
    boff: np.ndarray          # int64 [B]
    buffers: BatchBuffers     # 2 sum(rank) per-column buffers

    def factors(self, b: int) -> tuple[np.ndarray, np.ndarray, np.ndarray]:
        """decompressed (W, sigma, X) of block b (host, for checks)"""
        k = int(self.rank[b])
        vals = decompress_batch(self.buffers).cpu().numpy()
        voff = np.concatenate([[0], np.cumsum(self.buffers.count.astype(np.int64))[:-1]])
        cols = []
        for j in range(2 * k):
            q = int(self.boff[b]) + j
            cols.append(vals[voff[q]: voff[q] + int(self.buffers.count[q])])
        W = np.stack(cols[:k], 1) if k else np.zeros((self.m, 0))
        X = np.stack(cols[k:], 1) if k else np.zeros((self.n, 0))
        s = self.sigma[self.sig_off[b]: self.sig_off[b] + k]
        return W, s, X


def truncate_compressed(Uc: BatchBuffers, Vc: BatchBuffers, m: int, n: int, k: int, eps: float,
                        scheme=Scheme.afl) -> TruncatedBatch:
    """Algorithm 4 over B blocks U V^T of one shape: Uc holds B column-major m x k
    buffers, Vc B column-major n x k buffers (CodecLowrank factors,
    hmatrix.hpp:46-49).  Returns the truncated blocks as APLR leaves."""
    B = len(Uc)
    if len(Vc) != B or (Uc.count != m * k).any() or (Vc.count != n * k).any():
        raise ValueError("truncate_compressed: factor buffers do not match the block shape")
    if not (0.0 < eps < 1.0):
        raise ValueError("truncate_compressed: eps must lie in (0, 1)")
    U = decompress_batch(Uc).view(B, k, m).transpose(1, 2)     # column-major buffers
    V = decompress_batch(Vc).view(B, k, n).transpose(1, 2)
    Qu, Ru = torch.linalg.qr(U)
    Qv, Rv = torch.linalg.qr(V)
    Us, S, Vsh = torch.linalg.svd(Ru @ Rv.transpose(1, 2))
    S = torch.where(torch.isfinite(S), S, torch.zeros_like(S))
    ks_t = rank_from_singular_values(S, eps)
    W = Qu @ Us                                                   # (B, m, k)
    X = Qv @ Vsh.transpose(1, 2)                                  # (B, n, k)
    keep = torch.arange(S.shape[1], device=S.device)[None, :] < ks_t[:, None]
    Wf = W.transpose(1, 2)[keep].reshape(-1).contiguous()        # columns of W, block by block
    Xf = X.transpose(1, 2)[keep].reshape(-1).contiguous()
    sig = S[keep].cpu().numpy().astype(np.float64)
    ks = ks_t.cpu().numpy().astype(np.int64)
    woff = np.concatenate([[0], np.cumsum(ks * m)[:-1]]).astype(np.uint64)
    xoff = np.concatenate([[0], np.cumsum(ks * n)[:-1]]).astype(np.uint64)
    soff = np.concatenate([[0], np.cumsum(ks)[:-1]]).astype(np.int64)
    boff = np.concatenate([[0], np.cumsum(2 * ks)[:-1]]).astype(np.int64)
    nbuf = int(2 * ks.sum())
    count = np.concatenate([np.concatenate([[m] * int(kb), [n] * int(kb)]) for kb in ks]).astype(np.uint64) \
        if nbuf else np.zeros(0, np.uint64)
    desc = np.zeros(nbuf, dtype=DESC_DTYPE)
    poff = np.zeros(nbuf, dtype=np.uint64)
    cap = int(8 * (Wf.numel() + Xf.numel()) + 16 * nbuf + 16)
    payload = torch.empty(max(cap, 16), dtype=torch.uint8, device="cuda")
    tot = C.c_uint64()
    if nbuf:
        # every array handed to the C-ABI stays referenced until the call returns
        rows_a, cols_a = np.full(B, m, np.uint64), np.full(B, n, np.uint64)
        k_a, soff_a, boff_a = ks.astype(np.uint64), soff.astype(np.uint64), boff.astype(np.uint64)
        check(lib().hcmx_gpu_aplr_compress(B, u64p(rows_a), u64p(cols_a), u64p(k_a), ptr(Wf), u64p(woff),
                                           ptr(Xf), u64p(xoff), ptr(sig), u64p(soff_a), u64p(boff_a), float(eps),
                                           int(scheme), ptr(payload), payload.numel(), ptr(desc), u64p(poff),
                                           C.byref(tot), torch.cuda.current_stream().cuda_stream), "aplr_compress")
    bb = BatchBuffers(desc, count, poff, payload, tot.value)
    return TruncatedBatch(m, n, ks, sig, soff, boff, bb)
