"""FP64 assembly of an H-matrix for the synthetic problems (host-driven setup,
runs once before the hot path; torch on the GPU when present).

Dense (inadmissible) leaves are evaluated entry by entry.  Admissible leaves
get W, sigma, X with A ~= W diag(sigma) X^T, W and X orthonormal, truncated by
the reference's rank rule sigma_k > eps * sigma_0 (lowrank.cpp:14-21) -- the
shape svd_factors produces (lowrank.cpp:76-93).  Blocks up to EXACT_SVD_MAX (32)
columns use a full SVD; larger blocks a randomized range finder whose sketch
is grown per block until the captured spectrum reaches 1e-3 * eps * sigma_0,
so the truncation sees the same leading singular values a full SVD would
(tests/test_assemble.py compares ranks and singular values with a full SVD).
"""
from __future__ import annotations

import os
import sys
import time
from dataclasses import dataclass

import numpy as np
import torch

from .problems import PointKernel
from .tree import BlockLeaves

EXACT_SVD_MAX = 32
_PROF = {}  # HCMX_VERBOSE: seconds per setup step (synchronised timers)


def _tick(name, t0):
    if os.environ.get("HCMX_VERBOSE"):
        if torch.cuda.is_available():
            torch.cuda.synchronize()
        _PROF[name] = _PROF.get(name, 0.0) + time.time() - t0
    return time.time()


@dataclass
class Assembled:
    n: int
    leaves: BlockLeaves
    kind: np.ndarray          # 0 dense, 1 lowrank
    rank: np.ndarray          # lowrank rank (0 for dense)
    dense: torch.Tensor       # FP64, dense leaves column-major, leaf order
    dense_off: np.ndarray     # per leaf (dense) value offset, -1 otherwise
    W: torch.Tensor           # FP64, per lowrank leaf rows*k column-major
    X: torch.Tensor
    w_off: np.ndarray         # per leaf offsets into W / X, -1 for dense
    x_off: np.ndarray
    sigma: np.ndarray         # concatenated singular values
    sig_off: np.ndarray


def rank_from_singular_values(s: torch.Tensor, eps: float) -> torch.Tensor:
    """lowrank.cpp:14-21, batched: number of leading sigma_k > eps * sigma_0"""
    s0 = s[..., :1]
    keep = (s > eps * s0) & (s0 > 0)
    return keep.cumprod(dim=-1).sum(dim=-1)


_POOL = None


def _svd_chunk(a):
    from threadpoolctl import threadpool_limits
    with threadpool_limits(1):
        return np.linalg.svd(a, full_matrices=False)


def _host_workers() -> int:
    """host workers for this process: the cores divided among the GPU ranks of the
    node (torchrun's LOCAL_WORLD_SIZE), so N ranks setting up at once do not
    oversubscribe the host"""
    local = max(1, int(os.environ.get("LOCAL_WORLD_SIZE", "1") or 1))
    return max(1, min(32, (os.cpu_count() or 1) // local))


def _pool():
    """worker processes for host LAPACK (numpy's batched SVD does not scale over
    threads: measured 1.4x on 16 threads vs 6.6x on 16 processes); forkserver
    workers never touch CUDA"""
    global _POOL
    if _POOL is None:
        import multiprocessing as mp
        from concurrent.futures import ProcessPoolExecutor
        _POOL = ProcessPoolExecutor(_host_workers(), mp_context=mp.get_context("forkserver"))
    return _POOL


def _cpu_svd(M: torch.Tensor):
    """batched SVD of small matrices on the host (LAPACK gesdd per matrix):
    cuSOLVER runs batched SVDs above 32x32 one matrix at a time.  Large batches
    go to a process pool, small ones run in this process."""
    from concurrent.futures import ThreadPoolExecutor
    a = M.detach().resolve_conj().cpu().numpy()
    if a.shape[0] >= 2048 and _host_workers() > 2:
        parts = np.array_split(a, 4 * _host_workers())
        res = list(_pool().map(_svd_chunk, parts))
        dev = M.device
        cat = lambda i: torch.from_numpy(np.concatenate([r[i] for r in res])).to(dev)
        return cat(0), cat(1), cat(2)
    B = a.shape[0]
    U = np.empty(a.shape[:-1] + (min(a.shape[-2:]),), a.dtype)
    S = np.empty((B, min(a.shape[-2:])))
    Vh = np.empty((B, min(a.shape[-2:]), a.shape[-1]), a.dtype)
    nt = _host_workers()
    cuts = np.linspace(0, B, nt + 1).astype(int)

    def work(i):
        lo, hi = cuts[i], cuts[i + 1]
        if hi > lo:
            U[lo:hi], S[lo:hi], Vh[lo:hi] = np.linalg.svd(a[lo:hi], full_matrices=False)

    # one BLAS thread per worker: numpy's LAPACK would otherwise start a full
    # OpenBLAS pool inside every worker thread (nt x cores threads thrashing)
    from threadpoolctl import threadpool_limits
    with threadpool_limits(1), ThreadPoolExecutor(nt) as ex:
        list(ex.map(work, range(nt)))
    dev = M.device
    return torch.from_numpy(U).to(dev), torch.from_numpy(S).to(dev), torch.from_numpy(Vh).to(dev)


def _orth(Y: torch.Tensor) -> torch.Tensor:
    """orthonormal basis of the columns of a batch of tall matrices: classical
    Gram-Schmidt applied twice per column (batched GEMVs, so it stays fast for
    many small blocks where the batched Householder QR launches per matrix).
    Numerically dependent columns become arbitrary orthonormal directions, which
    a range finder tolerates.  Few large blocks: Householder QR."""
    B, m, p = Y.shape
    if B <= 64 and m >= 2048:
        return torch.linalg.qr(Y)[0]
    Q = torch.empty_like(Y)
    for j in range(p):
        v = Y[:, :, j:j + 1]
        for _ in range(2):
            if j:
                Qj = Q[:, :, :j]
                v = v - Qj @ (Qj.mH @ v)
        Q[:, :, j:j + 1] = v / torch.clamp(v.norm(dim=1, keepdim=True), min=1e-300)
    return Q


def _core_svd(M: torch.Tensor):
    """SVD of a batch of small square cores: batched Jacobi on the GPU up to 32 x 32
    (cuSOLVER's batched gesvdj), host LAPACK beyond"""
    if M.is_cuda and M.shape[-1] <= 32:
        U, S, Vh = torch.linalg.svd(M, full_matrices=False)
        return U, S, Vh
    return _cpu_svd(M)


def _svd_batch(A: torch.Tensor, eps: float, p0: int = 32):
    """truncation-grade SVD of a batch of blocks: (U, S, Vh) holding at least every
    singular triple above 1e-3 * eps * sigma_0 (the rank rule then keeps sigma_k >
    eps * sigma_0, lowrank.cpp:14-21).  Blocks up to EXACT_SVD_MAX columns: full
    SVD.  Larger: a randomized range finder Q = orth(A Omega) with p columns and
    one power iteration, then the exact SVD of Q^H A through Z = A^H Q = Q2 R2
    (Q^H A = R2^H Q2^H, so R2^H is the p x p core).  p grows per block (32, 48,
    64, 128, ...) until the p-th singular value of Q^H A is below
    0.03 * eps * sigma_0, so the sketch spans the whole retained spectrum;
    blocks that miss are redone with the next p, the others keep their result
    (zero-padded to the batch's width)."""
    B, m, n = A.shape
    if min(m, n) <= EXACT_SVD_MAX:
        return _core_svd(A) if m == n else _cpu_svd(A)
    g = torch.Generator(device=A.device)
    g.manual_seed(1234 + m)
    k = min(m, n)
    p = min(k, p0)
    todo = torch.arange(B, device=A.device)
    U = S = Vh = None
    while True:
        t0 = time.time()
        Ab = A[todo] if todo.numel() < B else A
        nb = Ab.shape[0]
        omega = torch.randn(nb, n, p, dtype=A.dtype, device=A.device, generator=g)
        Y = Ab @ omega
        t0 = _tick(f"sketch p{p}", t0)
        Q = _orth(Y)                                       # range of A, m x p
        Q = _orth(Ab @ _orth(Ab.mH @ Q))                   # one power iteration (A A^H) Q
        Z = Ab.mH @ Q                                      # (Q^H A)^H, n x p
        Q2 = _orth(Z)
        R2 = Q2.mH @ Z                                     # Z = Q2 R2
        t0 = _tick(f"orth p{p}", t0)
        Ur, Sb, Vrh = _core_svd(R2.mH)                     # Q^H A = Ur Sb (Q2 Vrh^H)^H
        t0 = _tick(f"core svd p{p}", t0)
        Ub, Vb = Q @ Ur, Vrh @ Q2.mH
        if U is None:  # width p for now, zero-padded when a later round widens it
            U = torch.zeros(B, m, p, dtype=A.dtype, device=A.device)
            S = torch.zeros(B, p, dtype=Sb.dtype, device=A.device)
            Vh = torch.zeros(B, p, n, dtype=A.dtype, device=A.device)
        elif U.shape[2] < p:
            pad = p - U.shape[2]
            U = torch.nn.functional.pad(U, (0, pad))
            S = torch.nn.functional.pad(S, (0, pad))
            Vh = torch.nn.functional.pad(Vh, (0, 0, 0, pad))
        # with one power iteration the error of a captured sigma_i is ~
        # sigma_{p+1}^4 / sigma_i^3: at sigma_p <= 0.03 eps sigma_0 the values near
        # the cut eps sigma_0 are exact to ~1e-6 relative, as a full SVD decides them
        done = (Sb[:, -1] <= 0.03 * eps * Sb[:, 0]) | (p >= k)
        idx = todo[done]
        U[idx, :, :p] = Ub[done]
        S[idx, :p] = Sb[done]
        Vh[idx, :p, :] = Vb[done]
        todo = todo[~done]
        _PROF[f"blocks p{p}"] = _PROF.get(f"blocks p{p}", 0) + nb
        t0 = _tick(f"collect p{p}", t0)
        if todo.numel() == 0:
            break
        p = min(k, p + 16 if p < 64 else 2 * p)                # 32, 48, 64, 128, ...
    w = max(1, int((S > 0).sum(dim=1).max().item())) if B else 1
    return U[:, :, :w], S[:, :w], Vh[:, :w, :]


def assemble(points_internal: np.ndarray, leaves: BlockLeaves, kernel: PointKernel, eps: float,
             device: str | None = None, batch_bytes: int | None = None) -> Assembled:
    dev = torch.device(device or ("cuda" if torch.cuda.is_available() else "cpu"))
    if batch_bytes is None:
        batch_bytes = (16 << 30) if dev.type == "cuda" else (1 << 30)
    P = torch.as_tensor(np.ascontiguousarray(points_internal, dtype=np.float64), device=dev)
    L = len(leaves)
    kind = np.where(leaves.admissible, 1, 0).astype(np.int64)
    rows = (leaves.row1 - leaves.row0).astype(np.int64)
    cols = (leaves.col1 - leaves.col0).astype(np.int64)
    rank = np.zeros(L, np.int64)

    # ---- dense leaves (column-major, leaf order)
    dense_off = np.full(L, -1, np.int64)
    didx = np.nonzero(kind == 0)[0]
    sizes = rows[didx] * cols[didx]
    dense_off[didx] = np.concatenate([[0], np.cumsum(sizes)[:-1]]) if didx.size else []
    dense = torch.empty(int(sizes.sum()), dtype=torch.float64, device=dev)
    _fill_blocks(P, leaves, didx, kernel, dense, dense_off, batch_bytes)

    # ---- lowrank leaves: SVD per shape group; factors packed per chunk with
    # one masked gather (column-major W and X, leaf by leaf within a chunk)
    lidx = np.nonzero(kind == 1)[0]
    w_off = np.full(L, -1, np.int64)
    x_off = np.full(L, -1, np.int64)
    sig_off = np.full(L, -1, np.int64)
    wl, xl, sl = [], [], []
    wo = xo = so = 0
    shapes = {}
    for l in lidx:
        shapes.setdefault((int(rows[l]), int(cols[l])), []).append(int(l))
    verbose = os.environ.get("HCMX_VERBOSE")
    for (m, n), ids in shapes.items():
        t0 = time.time()
        per = max(1, batch_bytes // (8 * m * n * 3))
        for c0 in range(0, len(ids), per):
            chunk = np.array(ids[c0: c0 + per])
            t1 = time.time()
            A = _blocks(P, leaves, chunk, kernel, separated=True)  # admissible: separated clusters
            _tick("kernel blocks", t1)
            U, S, Vh = _svd_batch(A, eps)
            ks_t = rank_from_singular_values(S, eps)
            keep = torch.arange(S.shape[1], device=S.device)[None, :] < ks_t[:, None]   # (B, p)
            Wc = U.transpose(1, 2)[keep].reshape(-1)     # rows of U^T = columns of W
            Xc = Vh[keep].reshape(-1)
            Sc = S[keep].cpu().numpy()
            ks = ks_t.cpu().numpy().astype(np.int64)
            rank[chunk] = ks
            cw = np.concatenate([[0], np.cumsum(ks * m)[:-1]])
            cx = np.concatenate([[0], np.cumsum(ks * n)[:-1]])
            cs = np.concatenate([[0], np.cumsum(ks)[:-1]])
            w_off[chunk] = wo + cw
            x_off[chunk] = xo + cx
            sig_off[chunk] = so + cs
            wl.append(Wc); xl.append(Xc); sl.append(Sc)
            wo += Wc.numel(); xo += Xc.numel(); so += Sc.size
            del A, U, S, Vh
        if verbose:
            sys.stderr.write(f"[assemble] {len(ids)} blocks {m}x{n}: {time.time() - t0:.2f}s "
                             f"{ {k: round(v, 2) for k, v in _PROF.items()} }\n")
            _PROF.clear()
    W = torch.cat(wl) if wl else torch.zeros(0, dtype=torch.float64, device=dev)
    X = torch.cat(xl) if xl else torch.zeros(0, dtype=torch.float64, device=dev)
    sigma = np.concatenate(sl) if sl else np.zeros(0)
    return Assembled(points_internal.shape[0], leaves, kind, rank, dense, dense_off, W, X, w_off,
                     x_off, sigma, sig_off)


def _blocks(P, leaves, ids, kernel, separated=False):
    r0 = torch.as_tensor(leaves.row0[ids], device=P.device)
    c0 = torch.as_tensor(leaves.col0[ids], device=P.device)
    m = int(leaves.row1[ids[0]] - leaves.row0[ids[0]])
    n = int(leaves.col1[ids[0]] - leaves.col0[ids[0]])
    ri = r0[:, None] + torch.arange(m, device=P.device)[None, :]
    ci = c0[:, None] + torch.arange(n, device=P.device)[None, :]
    return kernel.block(P[ri], P[ci], separated)


def _fill_blocks(P, leaves, ids, kernel, out, off, batch_bytes):
    if not len(ids):
        return
    rows = leaves.row1[ids] - leaves.row0[ids]
    cols = leaves.col1[ids] - leaves.col0[ids]
    groups = {}
    for i, l in enumerate(ids):
        groups.setdefault((int(rows[i]), int(cols[i])), []).append(int(l))
    for (m, n), g in groups.items():
        per = max(1, batch_bytes // (8 * m * n * 2))
        for c0 in range(0, len(g), per):
            chunk = np.array(g[c0: c0 + per])
            A = _blocks(P, leaves, chunk, kernel)            # [B, m, n]
            colmaj = A.transpose(1, 2).reshape(len(chunk), -1)  # column-major per leaf
            o = torch.as_tensor(off[chunk], device=P.device)
            idx = o[:, None] + torch.arange(m * n, device=P.device)[None, :]
            out[idx.reshape(-1)] = colmaj.reshape(-1)


def assemble_complex(points_internal: np.ndarray, leaves: BlockLeaves, kernel: PointKernel, eps: float,
                     device: str | None = None, batch_bytes: int | None = None) -> tuple[Assembled, Assembled]:
    """Complex kernels (config 5): A = Ar + i Ai as two real H-matrices on the same
    tree, so every factor's real and imaginary parts are separate codec streams.

    Dense leaves: Re / Im of the block.  Lowrank leaves: complex SVD A ~= U S V^H
    truncated by the same rank rule; with U = Ur + i Ui, V = Vr + i Vi,
        Re(A) = [Ur Ui] diag(S, S) [Vr Vi]^T,   Im(A) = [Ui -Ur] diag(S, S) [Vr Vi]^T,
    i.e. real APLR leaves of rank 2k whose column precisions follow S (the
    reference is real-only)."""
    dev = torch.device(device or ("cuda" if torch.cuda.is_available() else "cpu"))
    if batch_bytes is None:
        batch_bytes = (4 << 30) if dev.type == "cuda" else (1 << 30)
    P = torch.as_tensor(np.ascontiguousarray(points_internal, dtype=np.float64), device=dev)
    L = len(leaves)
    kind = np.where(leaves.admissible, 1, 0).astype(np.int64)
    rows = (leaves.row1 - leaves.row0).astype(np.int64)
    cols = (leaves.col1 - leaves.col0).astype(np.int64)
    rank = np.zeros(L, np.int64)
    dense_off = np.full(L, -1, np.int64)
    didx = np.nonzero(kind == 0)[0]
    sizes = rows[didx] * cols[didx]
    dense_off[didx] = np.concatenate([[0], np.cumsum(sizes)[:-1]]) if didx.size else []
    dre = torch.empty(int(sizes.sum()), dtype=torch.float64, device=dev)
    dim = torch.empty_like(dre)
    groups = {}
    for l in didx:
        groups.setdefault((int(rows[l]), int(cols[l])), []).append(int(l))
    for (m, n), g in groups.items():
        per = max(1, batch_bytes // (16 * m * n * 2))
        for c0 in range(0, len(g), per):
            chunk = np.array(g[c0: c0 + per])
            A = _blocks(P, leaves, chunk, kernel).transpose(1, 2).reshape(len(chunk), -1)  # column-major
            o = torch.as_tensor(dense_off[chunk], device=dev)
            idx = (o[:, None] + torch.arange(m * n, device=dev)[None, :]).reshape(-1)
            dre[idx] = A.real.reshape(-1)
            dim[idx] = A.imag.reshape(-1)
    lidx = np.nonzero(kind == 1)[0]
    w_off = np.full(L, -1, np.int64)
    x_off = np.full(L, -1, np.int64)
    sig_off = np.full(L, -1, np.int64)
    wr, wi, xl, sl = [], [], [], []
    wo = xo = so = 0
    shapes = {}
    for l in lidx:
        shapes.setdefault((int(rows[l]), int(cols[l])), []).append(int(l))
    for (m, n), ids in shapes.items():
        per = max(1, batch_bytes // (16 * m * n * 3))
        for c0 in range(0, len(ids), per):
            chunk = np.array(ids[c0: c0 + per])
            t1 = time.time()
            A = _blocks(P, leaves, chunk, kernel, separated=True)  # admissible: separated clusters
            _tick("kernel blocks", t1)
            U, S, Vh = _svd_batch(A, eps)
            ks_t = rank_from_singular_values(S, eps)
            keep = torch.arange(S.shape[1], device=S.device)[None, :] < ks_t[:, None]
            keep2 = keep[:, None, :].expand(-1, 2, -1)                # (B, 2, p): [real part, imag part]
            Ut = U.mT                                                  # rows = columns of U
            Wre = torch.stack([Ut.real, Ut.imag], 1)[keep2].reshape(-1)   # [Ur Ui]
            Wim = torch.stack([Ut.imag, -Ut.real], 1)[keep2].reshape(-1)  # [Ui -Ur]
            Xc = torch.stack([Vh.real, -Vh.imag], 1)[keep2].reshape(-1)   # [Vr Vi], V = Vh^H
            Sc = torch.stack([S, S], 1)[keep2].cpu().numpy()
            ks = 2 * ks_t.cpu().numpy().astype(np.int64)
            rank[chunk] = ks
            w_off[chunk] = wo + np.concatenate([[0], np.cumsum(ks * m)[:-1]])
            x_off[chunk] = xo + np.concatenate([[0], np.cumsum(ks * n)[:-1]])
            sig_off[chunk] = so + np.concatenate([[0], np.cumsum(ks)[:-1]])
            wr.append(Wre); wi.append(Wim); xl.append(Xc); sl.append(Sc)
            wo += Wre.numel(); xo += Xc.numel(); so += Sc.size
    z = torch.zeros(0, dtype=torch.float64, device=dev)
    Wr = torch.cat(wr) if wr else z
    Wi = torch.cat(wi) if wi else z
    X = torch.cat(xl) if xl else z
    sigma = np.concatenate(sl) if sl else np.zeros(0)
    n = points_internal.shape[0]
    mk = lambda dense, W: Assembled(n, leaves, kind, rank, dense, dense_off, W, X, w_off, x_off, sigma, sig_off)
    return mk(dre, Wr), mk(dim, Wi)
