"""Test helper: a small compressed H-matrix built and compressed entirely on the
CPU with the checkers (oracle/), in the flat layout shared by the oracle and
the C-ABI (hcmx_hmat_desc).  Test infrastructure only."""
from __future__ import annotations

import os
import sys
from dataclasses import dataclass

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "oracle"))

from oracle import Oracle, RefOracle  # noqa: E402

FIELDS_I64 = ("row0", "row1", "col0", "col1", "kind", "rank", "buf0", "sig0", "count", "poff",
              "plen")


@dataclass
class Flat:
    n_rows: int
    n_cols: int
    row0: np.ndarray
    row1: np.ndarray
    col0: np.ndarray
    col1: np.ndarray
    kind: np.ndarray
    rank: np.ndarray
    buf0: np.ndarray
    sig0: np.ndarray
    sigma: np.ndarray
    scheme: np.ndarray
    e: np.ndarray
    m: np.ndarray
    scale: np.ndarray
    count: np.ndarray
    poff: np.ndarray
    plen: np.ndarray
    blob: np.ndarray
    raw: np.ndarray | None = None

    def arrays(self) -> dict:
        d = {k: getattr(self, k) for k in FIELDS_I64}
        d.update(sigma=self.sigma, scheme=self.scheme, e=self.e, m=self.m, scale=self.scale,
                 blob=self.blob, dims=np.array([self.n_rows, self.n_cols], np.int64))
        return d

    @staticmethod
    def from_npz(z) -> "Flat":
        n_rows, n_cols = (int(v) for v in z["dims"])
        kw = {k: z[k] for k in FIELDS_I64}
        return Flat(n_rows, n_cols, sigma=z["sigma"], scheme=z["scheme"], e=z["e"], m=z["m"],
                    scale=z["scale"], blob=z["blob"], **kw)

    def to_product(self):
        """as paper_2308_10960_b200.hmatrix.FlatHMatrix (for the GPU path)"""
        from paper_2308_10960_b200._lib import DESC_DTYPE
        from paper_2308_10960_b200.hmatrix import FlatHMatrix
        desc = np.zeros(self.count.size, DESC_DTYPE)
        desc["scheme"], desc["exp_bits"], desc["mant_bits"] = self.scheme, self.e, self.m
        sc = self.scheme.astype(np.int64)
        unit = np.array([1, 8, 8, 16, 1, 1, 1])[sc]
        w = 1 + self.e.astype(np.int64) + self.m.astype(np.int64)
        w = w + (unit - w % unit) % unit
        w = np.where(sc >= 4, np.array([0, 0, 0, 0, 64, 32, 16])[sc], w)  # raw FP64 / FP32 / FP16
        desc["bit_width"] = w
        desc["scale"] = self.scale
        return FlatHMatrix(self.n_rows, self.n_cols, self.row0, self.row1, self.col0, self.col1,
                           self.kind, self.rank, self.buf0, self.sig0, self.sigma, desc, self.count,
                           self.poff, self.plen, np.ascontiguousarray(self.blob, np.uint8))

    def dense(self, oracle=None) -> np.ndarray:
        """materialised matrix (hmatrix.hpp:131 to_dense) from the decoded leaves"""
        o = oracle or Oracle()
        from oracle import Buf
        M = np.zeros((self.n_rows, self.n_cols))
        for l in range(self.row0.size):
            r0, r1, c0, c1 = self.row0[l], self.row1[l], self.col0[l], self.col1[l]
            buf = lambda b: Buf(int(self.scheme[b]), int(self.e[b]), int(self.m[b]),
                                float(self.scale[b]), int(self.count[b]),
                                self.blob[self.poff[b]: self.poff[b] + self.plen[b]].tobytes())
            if self.kind[l] == 0:
                M[r0:r1, c0:c1] = o.decompress(buf(self.buf0[l])).reshape(c1 - c0, r1 - r0).T
            else:
                k = int(self.rank[l])
                W = np.stack([o.decompress(buf(self.buf0[l] + i)) for i in range(k)], 1) if k else np.zeros((r1 - r0, 0))
                X = np.stack([o.decompress(buf(self.buf0[l] + k + i)) for i in range(k)], 1) if k else np.zeros((c1 - c0, 0))
                s = self.sigma[self.sig0[l]: self.sig0[l] + k]
                M[r0:r1, c0:c1] = (W * s) @ X.T
        return M


def build_small_flat(n=1024, eps=1e-6, scheme=0, use_ref=False, geometry="fibonacci",
                     kernel="laplace", seed=1, leaf=64, eta=2.0, mode="aplr", dense_too=True,
                     return_assembled=False):
    """points -> trees -> FP64 assembly (torch CPU) -> CPU codec -> Flat, x.
    mode (StorageMode kind, hmatrix.hpp:32-40): 'aplr' (default), 'codec'
    (CodecDense + CodecLowrank of U = W diag(sigma), V = X), 'mp' (FP64 dense +
    MP-D-S-H column groups), 'fp64' (uncompressed)"""
    from paper_2308_10960_b200 import assemble, problems, tree
    o = RefOracle() if use_ref else Oracle()
    pts = problems.make_points(geometry, n, seed)
    ct = tree.build_cluster_tree(pts, leaf)
    lv = tree.build_block_tree(ct, ct, eta)
    A = assemble.assemble(pts[ct.i2e], lv, problems.make_kernel(kernel), eps, device="cpu")
    if mode != "aplr":
        flat = _build_mode_flat(o, A, lv, n, eps, scheme, mode, dense_too)
        x = np.random.default_rng(seed + 100).uniform(-1.0, 1.0, n)
        return (flat, x, A) if return_assembled else (flat, x)
    dense = A.dense.numpy()
    W, X = A.W.numpy(), A.X.numpy()
    L = len(lv)
    rows = (lv.row1 - lv.row0).astype(np.int64)
    cols = (lv.col1 - lv.col0).astype(np.int64)
    bufs, buf0 = [], np.zeros(L, np.int64)
    for l in range(L):
        buf0[l] = len(bufs)
        if A.kind[l] == 0:
            v = dense[A.dense_off[l]: A.dense_off[l] + rows[l] * cols[l]]
            bufs.append(o.compress(v, eps, scheme))
        else:
            k = int(A.rank[l])
            if k == 0:
                continue
            Wl = W[A.w_off[l]: A.w_off[l] + rows[l] * k].reshape(k, rows[l]).T
            Xl = X[A.x_off[l]: A.x_off[l] + cols[l] * k].reshape(k, cols[l]).T
            s = A.sigma[A.sig_off[l]: A.sig_off[l] + k]
            bufs.extend(o.aplr_compress(Wl, Xl, s, eps, scheme))
    poff, off, parts = [], 0, []
    for b in bufs:
        poff.append(off)
        pad = (-len(b.payload)) % 16
        parts.append(np.frombuffer(b.payload + b"\0" * pad, np.uint8))
        off += len(b.payload) + pad
    sig0 = A.sig_off.copy()
    sig0[sig0 < 0] = 0
    flat = Flat(n, n, lv.row0.astype(np.int64), lv.row1.astype(np.int64), lv.col0.astype(np.int64),
                lv.col1.astype(np.int64), A.kind.astype(np.int64), A.rank.astype(np.int64), buf0,
                sig0, A.sigma.astype(np.float64), np.array([b.scheme for b in bufs], np.uint8),
                np.array([b.e for b in bufs], np.uint8), np.array([b.m for b in bufs], np.uint8),
                np.array([b.scale for b in bufs]), np.array([b.count for b in bufs], np.int64),
                np.array(poff, np.int64), np.array([len(b.payload) for b in bufs], np.int64),
                np.concatenate(parts) if parts else np.zeros(16, np.uint8))
    x = np.random.default_rng(seed + 100).uniform(-1.0, 1.0, n)
    return (flat, x, A) if return_assembled else (flat, x)


def _raw_buf(o, v, fmt):
    from oracle import Buf
    return Buf(fmt, 0, 0, 1.0, int(np.asarray(v).size), o.pack_raw(v, fmt))


def _build_mode_flat(o, A, lv, n, eps, scheme, mode, dense_too):
    """CPU construction of the other StorageModes with the checkers' codec and
    the restated PackedSlice / mp_partition (oracle/hcmx_oracle.c)"""
    dense = A.dense.numpy()
    W, X = A.W.numpy(), A.X.numpy()
    L = len(lv)
    rows = (lv.row1 - lv.row0).astype(np.int64)
    cols = (lv.col1 - lv.col0).astype(np.int64)
    kind = A.kind.astype(np.int64).copy()
    rank = A.rank.astype(np.int64).copy()
    bufs, buf0 = [], np.zeros(L, np.int64)
    for l in range(L):
        buf0[l] = len(bufs)
        if A.kind[l] == 0:
            v = dense[A.dense_off[l]: A.dense_off[l] + rows[l] * cols[l]]
            if mode == "codec" and dense_too:
                bufs.append(o.compress(v, eps, scheme))
            else:
                bufs.append(_raw_buf(o, v, 4))
            continue
        k = int(A.rank[l])
        if mode in ("codec", "fp64"):
            kind[l] = 2
        if k == 0:
            continue
        Wl = W[A.w_off[l]: A.w_off[l] + rows[l] * k]            # column-major rows x k
        Xl = X[A.x_off[l]: A.x_off[l] + cols[l] * k]
        s = A.sigma[A.sig_off[l]: A.sig_off[l] + k]
        if mode in ("codec", "fp64"):
            U = (Wl.reshape(k, rows[l]) * s[:, None]).reshape(-1)  # W diag(sigma), one product each
            if mode == "codec":
                bufs += [o.compress(U, eps, scheme), o.compress(Xl, eps, scheme)]
            else:
                bufs += [_raw_buf(o, U, 4), _raw_buf(o, Xl, 4)]
        else:  # mp
            r = o.mp_partition(s, eps * s[0])
            assert r.sum() == k
            fmt = np.repeat([4, 5, 6], r)
            for i in range(k):
                bufs.append(_raw_buf(o, Wl[i * rows[l]:(i + 1) * rows[l]], int(fmt[i])))
            for i in range(k):
                bufs.append(_raw_buf(o, Xl[i * cols[l]:(i + 1) * cols[l]], int(fmt[i])))
    poff, off, parts = [], 0, []
    for b in bufs:
        poff.append(off)
        pad = (-len(b.payload)) % 16
        parts.append(np.frombuffer(b.payload + b"\0" * pad, np.uint8))
        off += len(b.payload) + pad
    sig0 = A.sig_off.copy()
    sig0[sig0 < 0] = 0
    return Flat(n, n, lv.row0.astype(np.int64), lv.row1.astype(np.int64), lv.col0.astype(np.int64),
                lv.col1.astype(np.int64), kind, rank, buf0, sig0, A.sigma.astype(np.float64),
                np.array([b.scheme for b in bufs], np.uint8), np.array([b.e for b in bufs], np.uint8),
                np.array([b.m for b in bufs], np.uint8), np.array([b.scale for b in bufs]),
                np.array([b.count for b in bufs], np.int64), np.array(poff, np.int64),
                np.array([len(b.payload) for b in bufs], np.int64),
                np.concatenate(parts) if parts else np.zeros(16, np.uint8))


def flat_from_leaves(n_rows, n_cols, leaves, eps=1e-6, scheme=0, seed=7, use_ref=False):
    """A synthetic flat H-matrix from explicit leaves (no geometry): each entry
    (kind, r0, r1, c0, c1, k) is a dense block (kind 0, entries sign 10^U[-3,0])
    or an APLR leaf W diag(sigma) X^T of rank k (kind 1: orthonormal W, X from a
    seeded QR, sigma = 10^-linspace(0, 7, k)), compressed by the checkers'
    codec.  Lets a test hit leaf shapes the sphere problems never produce
    (very wide lowrank leaves, odd / ragged chunk counts)."""
    o = RefOracle() if use_ref else Oracle()
    rng = np.random.default_rng(seed)
    L = len(leaves)
    row0, row1, col0, col1, kind, rank, buf0, sig0 = (np.zeros(L, np.int64) for _ in range(8))
    sigmas, bufs = [], []
    nsig = 0
    for l, (kd, r0, r1, c0, c1, k) in enumerate(leaves):
        row0[l], row1[l], col0[l], col1[l], kind[l] = r0, r1, c0, c1, kd
        buf0[l] = len(bufs)
        rows, cols = r1 - r0, c1 - c0
        if kd == 0:
            v = np.sign(rng.standard_normal(rows * cols)) * 10 ** rng.uniform(-3, 0, rows * cols)
            bufs.append(o.compress(v, eps, scheme))
            continue
        rank[l] = k
        sig0[l] = nsig
        W = np.linalg.qr(rng.standard_normal((rows, k)))[0]
        X = np.linalg.qr(rng.standard_normal((cols, k)))[0]
        s = 10.0 ** -np.linspace(0, 7, k)
        sigmas.append(s)
        nsig += k
        bufs.extend(o.aplr_compress(np.asfortranarray(W), np.asfortranarray(X), s, eps, scheme))
    poff, off, parts = [], 0, []
    for b in bufs:
        poff.append(off)
        pad = (-len(b.payload)) % 16
        parts.append(np.frombuffer(b.payload + b"\0" * pad, np.uint8))
        off += len(b.payload) + pad
    return Flat(n_rows, n_cols, row0, row1, col0, col1, kind, rank, buf0, sig0,
                np.concatenate(sigmas) if sigmas else np.zeros(1),
                np.array([b.scheme for b in bufs], np.uint8), np.array([b.e for b in bufs], np.uint8),
                np.array([b.m for b in bufs], np.uint8), np.array([b.scale for b in bufs]),
                np.array([b.count for b in bufs], np.int64), np.array(poff, np.int64),
                np.array([len(b.payload) for b in bufs], np.int64), np.concatenate(parts))
