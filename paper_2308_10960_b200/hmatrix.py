"""hcmx H-matrix on the B200: compress_in_place, the device-resident compressed
H-matrix and matvec (hmatrix.hpp:93-153).

The reference declares these functions but ships no hmatrix.cpp, so the
contract comes from hmatrix.hpp and SPEC.md:
  * compress_in_place(M, eps, mode, dense_too): lowrank leaves -> APLR
    (per-column codec, mixedprec.cpp:155-187), dense leaves -> codec::compress
    when dense_too; returns a MemoryReport
  * matvec(alpha, M, x, beta, y, transpose=False): y := alpha M x + beta y in the
    internal (cluster-permuted) index space; alpha == 0 leaves M untouched;
    dimension mismatch -> ValueError (std::invalid_argument)

The flattened form (FlatHMatrix) is the exchange format with the C-ABI
(hcmx_hmat_desc) and with the CPU oracle: leaves in for_each_leaf preorder,
one codec buffer per dense leaf (column-major scan, hmatrix.hpp:42-44), 2k
buffers per APLR leaf (W columns, then X columns).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from ._lib import DESC_DTYPE, check, lib, ptr, u64p
from .assemble import Assembled, assemble, assemble_complex
from .codec import Scheme, compress_batch
from .problems import config as problem_config, make_kernel, make_points
from .tree import build_block_tree, build_cluster_tree

__all__ = ["FlatHMatrix", "MemoryReport", "compress_in_place", "HMatrix", "matvec", "build_config",
           "StorageMode"]


@dataclass
class StorageMode:
    """hmatrix.hpp:32-40 (the GPU matvec covers kind 'aplr' + dense codec)"""
    kind: str = "aplr"
    scheme: Scheme = Scheme.afl

    @staticmethod
    def parse(name: str) -> "StorageMode":
        name = name.lower()
        if name.endswith("-aplr"):
            return StorageMode("aplr", Scheme[name[:-5]])
        if name in ("afl", "aflp", "bfl", "dfl"):
            return StorageMode("codec", Scheme[name])
        if name in ("fp64", "mp"):
            return StorageMode(name, Scheme.afl)
        if name.startswith("mp-") or name == "mp-d-s-h":
            return StorageMode("mp", Scheme.afl)
        raise ValueError(f"unknown storage mode {name}")

    def name(self) -> str:
        if self.kind == "aplr":
            return f"{self.scheme.name}-aplr"
        return self.scheme.name if self.kind == "codec" else self.kind


@dataclass
class MemoryReport:
    """hmatrix.hpp:96-113"""
    dense_raw: int = 0
    dense_compressed: int = 0
    lowrank_raw: int = 0
    lowrank_compressed: int = 0
    overhead: int = 0
    uncompressed_equivalent: int = 0

    def payload_total(self) -> int:
        return self.dense_raw + self.dense_compressed + self.lowrank_raw + self.lowrank_compressed

    def total(self) -> int:
        return self.payload_total() + self.overhead

    def rate(self) -> float:
        t = self.payload_total()
        return 0.0 if t == 0 else self.uncompressed_equivalent / t


@dataclass
class FlatHMatrix:
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
    desc: np.ndarray          # DESC_DTYPE per buffer
    count: np.ndarray         # int64
    poff: np.ndarray          # int64 byte offsets into blob
    plen: np.ndarray          # int64 payload bytes
    blob: object              # np.uint8 (host) or torch.uint8 (cuda)
    raw: np.ndarray | None = None
    meta: dict = field(default_factory=dict)

    # oracle-facing views
    @property
    def scheme(self):
        return self.desc["scheme"]

    @property
    def e(self):
        return self.desc["exp_bits"]

    @property
    def m(self):
        return self.desc["mant_bits"]

    @property
    def scale(self):
        return self.desc["scale"]

    @property
    def nleaves(self):
        return self.row0.size

    def host(self) -> "FlatHMatrix":
        if isinstance(self.blob, torch.Tensor):
            return FlatHMatrix(**{**self.__dict__, "blob": self.blob.cpu().numpy()})
        return self

    def compressed_bytes(self) -> int:
        """sum of CompressedBuffer::byte_size (20 + payload) + 8 k sigma per APLR leaf"""
        return int((self.plen + 20).sum() + 8 * self.rank[self.kind == 1].sum())

    def memory_footprint(self) -> MemoryReport:
        """hmatrix.hpp:124 memory_footprint for the compressed payload kinds"""
        r = MemoryReport()
        rows, cols = self.row1 - self.row0, self.col1 - self.col0
        for l in range(self.nleaves):
            if self.kind[l] == 0:
                r.dense_compressed += 20 + int(self.plen[self.buf0[l]])
                r.uncompressed_equivalent += 8 * int(rows[l] * cols[l])
            else:
                k = int(self.rank[l])
                b = int(self.buf0[l])
                r.lowrank_compressed += 8 + 8 * k + int((self.plen[b: b + 2 * k] + 20).sum())
                r.uncompressed_equivalent += 8 * int((rows[l] + cols[l]) * k)
        r.overhead = 16 * self.nleaves
        return r


RAW_F64, RAW_F32, RAW_F16 = 4, 5, 6   # hcmx_scheme raw storage (include/hcmx_gpu.h)
_RAW_BYTES = {RAW_F64: 8, RAW_F32: 4, RAW_F16: 2}
MP_ROUNDOFFS = (1.1e-16, 6.0e-8, 4.9e-4)   # mixedprec.hpp:23 (MP-D-S-H)


def _raw_desc(n: int, fmt: int) -> np.ndarray:
    d = np.zeros(n, dtype=DESC_DTYPE)
    d["scheme"] = fmt
    d["bit_width"] = 8 * _RAW_BYTES[fmt]
    d["scale"] = 1.0
    return d


def _pack_raw(v: torch.Tensor, fmt: int) -> torch.Tensor:
    """PackedSlice::pack (mixedprec.cpp:16-41) on the device: FP64 words as is,
    FP32 = (float)v, FP16 = float_to_half((float)v) (half.hpp:75: two rounding
    steps, both round-to-nearest-even; torch's float -> half is the IEEE one)"""
    v = v.to(torch.float64).contiguous()
    if fmt == RAW_F64:
        return v.view(torch.uint8)
    if fmt == RAW_F32:
        return v.to(torch.float32).contiguous().view(torch.uint8)
    return v.to(torch.float32).to(torch.float16).contiguous().view(torch.uint8)


def mp_partition(sigma: np.ndarray, delta: float) -> np.ndarray:
    """mixedprec.cpp:66-82: per column, the cheapest of FP64 / FP32 / FP16 whose
    unit roundoff keeps sigma_j * rho <= delta; columns with sigma_j <= delta are
    truncated (-1)."""
    g = np.zeros(sigma.size, np.int64)
    g[sigma * MP_ROUNDOFFS[1] <= delta] = 1
    g[sigma * MP_ROUNDOFFS[2] <= delta] = 2
    g[sigma <= delta] = -1
    return g


def compress_in_place(A: Assembled, eps: float, mode: StorageMode | str = "afl-aplr",
                      dense_too: bool = True, threads: int = 1) -> FlatHMatrix:
    """hmatrix.hpp:115-119 on the device, for every StorageMode kind
    (hmatrix.hpp:32-40):
      aplr  dense -> codec::compress (iff dense_too, else FP64); lowrank -> APLR
            (hcmx_gpu_aplr_compress: per-column precision from sigma)
      codec dense as above; lowrank U = W diag(sigma), V = X each compressed as
            one buffer (CodecLowrank, hmatrix.hpp:46-49)
      mp    dense FP64 (MP never compresses dense); lowrank W Sigma X^H with the
            columns in FP64 / FP32 / FP16 groups (mp_compress, mixedprec.cpp:94-120)
      fp64  uncompressed: dense FP64, lowrank U, V in FP64 (LowrankBlock)
    Returns the flattened H-matrix (payload blob resident on the GPU)."""
    if isinstance(mode, str):
        mode = StorageMode.parse(mode)
    _lib.ensure_device()
    scheme = int(mode.scheme)
    lv = A.leaves
    L = len(lv)
    rows = (lv.row1 - lv.row0).astype(np.int64)
    cols = (lv.col1 - lv.col0).astype(np.int64)
    didx = np.nonzero(A.kind == 0)[0]
    lidx = np.nonzero(A.kind == 1)[0]
    kind = A.kind.astype(np.int64).copy()
    rank = A.rank.astype(np.int64).copy()
    sigma = np.ascontiguousarray(A.sigma, np.float64)
    sig0 = A.sig_off.copy()
    sig0[sig0 < 0] = 0

    uniform = mode.kind in ("codec", "fp64")  # lowrank leaves as U, V (kind 2)
    if uniform:
        kind[lidx] = 2
    nbuf_leaf = np.where(kind == 0, 1, np.where(kind == 2, np.where(rank > 0, 2, 0), 2 * rank))
    buf0 = np.concatenate([[0], np.cumsum(nbuf_leaf)[:-1]]).astype(np.int64)
    nb = int(nbuf_leaf.sum())
    desc = np.zeros(nb, dtype=DESC_DTYPE)
    count = np.zeros(nb, np.int64)
    poff = np.zeros(nb, np.int64)
    parts, total = [], 0

    def add(payload: torch.Tensor, nbytes: int) -> int:
        nonlocal total
        at = total
        pad = (-nbytes) % 16
        parts.append(payload[:nbytes])
        if pad:
            parts.append(torch.zeros(pad, dtype=torch.uint8, device="cuda"))
        total += nbytes + pad
        return at

    # dense leaves
    dn = rows[didx] * cols[didx]
    if didx.size:
        if mode.kind in ("aplr", "codec") and dense_too:
            bb = compress_batch(A.dense, dn.astype(np.uint64), eps, scheme,
                                voff=A.dense_off[didx].astype(np.uint64))
            at = add(bb.payload, bb.total)
            b = buf0[didx]
            desc[b] = bb.desc
            count[b] = dn
            poff[b] = bb.poff.astype(np.int64) + at
        else:  # FP64 (StorageMode fp64 / mp, or dense_too = false)
            dev = A.dense.to("cuda")
            off = A.dense_off[didx]
            idx = torch.as_tensor(np.concatenate([np.arange(o, o + c) for o, c in zip(off, dn)])
                                  if didx.size else np.zeros(0, np.int64)).cuda()
            raw = _pack_raw(dev.index_select(0, idx), RAW_F64)
            at = add(raw, raw.numel())
            b = buf0[didx]
            desc[b] = _raw_desc(didx.size, RAW_F64)
            count[b] = dn
            poff[b] = at + 8 * np.concatenate([[0], np.cumsum(dn)[:-1]])

    kk = rank[lidx]
    if lidx.size and kk.sum() > 0:
        W = A.W.to("cuda")
        X = A.X.to("cuda")
        if mode.kind == "aplr":
            lr_boff = np.concatenate([[0], np.cumsum(2 * kk)[:-1]]).astype(np.uint64)
            nlb = int(2 * kk.sum())
            cap = int(8 * (A.W.numel() + A.X.numel()) + 16 * nlb + 16)
            lr_payload = torch.empty(cap, dtype=torch.uint8, device="cuda")
            lr_desc = np.zeros(nlb, dtype=DESC_DTYPE)
            lr_poff = np.zeros(nlb, dtype=np.uint64)
            tot = C.c_uint64()
            rr = rows[lidx].astype(np.uint64); cc = cols[lidx].astype(np.uint64)
            wo = A.w_off[lidx].astype(np.uint64); xo = A.x_off[lidx].astype(np.uint64)
            so = A.sig_off[lidx].astype(np.uint64)
            check(lib().hcmx_gpu_aplr_compress(lidx.size, u64p(rr), u64p(cc), u64p(kk.astype(np.uint64)),
                                               ptr(W), u64p(wo), ptr(X), u64p(xo), ptr(sigma), u64p(so),
                                               u64p(lr_boff), float(eps), scheme, ptr(lr_payload), cap,
                                               ptr(lr_desc), u64p(lr_poff), C.byref(tot),
                                               torch.cuda.current_stream().cuda_stream), "aplr_compress")
            at = add(lr_payload, tot.value)
            j = 0
            for l in lidx:
                k = int(rank[l])
                sl = slice(int(buf0[l]), int(buf0[l]) + 2 * k)
                desc[sl] = lr_desc[j: j + 2 * k]
                count[sl] = [rows[l]] * k + [cols[l]] * k
                poff[sl] = lr_poff[j: j + 2 * k].astype(np.int64) + at
                j += 2 * k
        elif uniform:
            # U = W diag(sigma) (one FP64 product per element), V = X; one buffer each
            sig_t = torch.as_tensor(sigma).cuda()
            us, ucount = [], []
            for l in lidx:
                k = int(rank[l])
                if k == 0:
                    continue
                r, c = int(rows[l]), int(cols[l])
                Wl = W[A.w_off[l]: A.w_off[l] + r * k].view(k, r)
                s = sig_t[A.sig_off[l]: A.sig_off[l] + k]
                us.append((Wl * s[:, None]).reshape(-1))
                us.append(X[A.x_off[l]: A.x_off[l] + c * k])
                ucount += [r * k, c * k]
            vals = torch.cat(us) if us else torch.zeros(0, dtype=torch.float64, device="cuda")
            ucount = np.array(ucount, np.int64)
            bidx = np.concatenate([[int(buf0[l]), int(buf0[l]) + 1] for l in lidx if rank[l] > 0])
            if mode.kind == "codec":
                bb = compress_batch(vals, ucount.astype(np.uint64), eps, scheme)
                at = add(bb.payload, bb.total)
                desc[bidx] = bb.desc
                poff[bidx] = bb.poff.astype(np.int64) + at
            else:
                raw = _pack_raw(vals, RAW_F64)
                at = add(raw, raw.numel())
                desc[bidx] = _raw_desc(bidx.size, RAW_F64)
                poff[bidx] = at + 8 * np.concatenate([[0], np.cumsum(ucount)[:-1]])
            count[bidx] = ucount
            sigma = np.ones(max(1, sigma.size))  # unused by U V^T leaves
        else:  # mp: per-column raw formats by the D-S-H partition
            cols_fmt, ws, xs_, wcnt, xcnt, keep_rank = [], [], [], [], [], rank.copy()
            for l in lidx:
                k = int(rank[l])
                if k == 0:
                    continue
                sl = sigma[A.sig_off[l]: A.sig_off[l] + k]
                g = mp_partition(sl, eps * sl[0])
                assert (g >= 0).all() and (np.diff(g) >= 0).all(), "sigma must be decreasing above delta"
                cols_fmt.append(RAW_F64 + g)
            fmts = np.concatenate(cols_fmt) if cols_fmt else np.zeros(0, np.int64)
            # buffers in leaf order: W columns then X columns of each leaf
            wbytes, chunks = [], []
            j = 0
            bi, bcount, bfmt = [], [], []
            for l in lidx:
                k = int(rank[l])
                if k == 0:
                    continue
                r, c = int(rows[l]), int(cols[l])
                Wl = W[A.w_off[l]: A.w_off[l] + r * k]
                Xl = X[A.x_off[l]: A.x_off[l] + c * k]
                for i in range(k):
                    f = int(fmts[j + i])
                    chunks.append((_pack_raw(Wl[i * r:(i + 1) * r], f), r, f, int(buf0[l]) + i))
                for i in range(k):
                    f = int(fmts[j + i])
                    chunks.append((_pack_raw(Xl[i * c:(i + 1) * c], f), c, f, int(buf0[l]) + k + i))
                j += k
            for pl, n, f, b in chunks:
                at = add(pl, pl.numel())
                desc[b] = _raw_desc(1, f)[0]
                count[b] = n
                poff[b] = at
    blob = torch.cat(parts) if parts else torch.zeros(16, dtype=torch.uint8, device="cuda")
    plen = (count * desc["bit_width"].astype(np.int64) + 7) // 8
    return FlatHMatrix(A.n, A.n, lv.row0.astype(np.int64), lv.row1.astype(np.int64),
                       lv.col0.astype(np.int64), lv.col1.astype(np.int64), kind, rank, buf0, sig0,
                       np.ascontiguousarray(sigma), desc, count, poff, plen, blob,
                       meta={"eps": eps, "mode": mode.name(), "dense_too": dense_too})


def build_config(cfg, scheme="afl", device=None, n=None, seed=1, eps=None) -> tuple[FlatHMatrix, dict]:
    """setup for a BASELINE config (or a dict): points -> cluster/block tree ->
    FP64 assembly -> compress_in_place on the GPU"""
    c = problem_config(cfg) if not isinstance(cfg, dict) else dict(cfg)
    if n is not None:
        c["n"] = n
    if eps is not None:
        c["eps"] = eps
    pts = make_points(c["geometry"], c["n"], seed)
    ct = build_cluster_tree(pts, c["leaf"])
    leaves = build_block_tree(ct, ct, c["eta"])
    A = assemble(pts[ct.i2e], leaves, make_kernel(c["kernel"]), c["eps"], device=device)
    flat = compress_in_place(A, c["eps"], f"{Scheme[scheme].name if isinstance(scheme, str) else Scheme(scheme).name}-aplr")
    info = dict(c, leaves=len(leaves), dense_leaves=int((A.kind == 0).sum()),
                lowrank_leaves=int((A.kind == 1).sum()), mean_rank=float(A.rank[A.kind == 1].mean())
                if (A.kind == 1).any() else 0.0, max_rank=int(A.rank.max()) if len(A.rank) else 0,
                depth=ct.depth())
    return flat, info


def flat_desc(flat: FlatHMatrix, row_range=None, with_transpose=False, nrhs_block=0):
    """hcmx_hmat_desc over the arrays of a flattened H-matrix (+ the objects the
    pointers refer to, to be kept alive while the descriptor is used)"""
    keep = {}
    a = lambda x, t: keep.setdefault(id(x), np.ascontiguousarray(x, dtype=t))
    i64 = lambda x: a(x, np.int64).ctypes.data_as(C.POINTER(C.c_int64))
    sigma = np.ascontiguousarray(flat.sigma if flat.sigma.size else np.zeros(1), dtype=np.float64)
    desc = np.ascontiguousarray(flat.desc)
    blob = flat.blob
    on_dev = isinstance(blob, torch.Tensor) and blob.is_cuda
    if isinstance(blob, torch.Tensor) and not on_dev:
        blob = blob.numpy()
    d = _lib.hcmx_hmat_desc()
    d.n_rows, d.n_cols, d.nleaves = int(flat.n_rows), int(flat.n_cols), flat.nleaves
    d.nbuffers, d.nsigma = desc.size, flat.sigma.size
    d.blob_bytes = blob.numel() if isinstance(blob, torch.Tensor) else blob.size
    for name in ("row0", "row1", "col0", "col1", "kind", "rank", "buf0", "sig0"):
        setattr(d, name, i64(getattr(flat, name)))
    d.sigma = sigma.ctypes.data_as(C.POINTER(C.c_double))
    d.desc = desc.ctypes.data_as(C.POINTER(_lib.hcmx_descriptor))
    d.count, d.poff, d.plen = i64(flat.count), i64(flat.poff), i64(flat.plen)
    d.blob = ptr(blob)
    d.blob_on_device = int(on_dev)
    d.row_begin, d.row_end = (0, 0) if row_range is None else row_range
    d.with_transpose = int(with_transpose)
    d.nrhs_block = int(nrhs_block)  # 4: matmat decodes once for 4 right-hand sides
    return d, (keep, sigma, desc, blob)


class HMatrix:
    """Device-resident compressed H-matrix (handle over hcmx_gpu_hmat_*)."""

    def __init__(self, flat: FlatHMatrix, row_range: tuple[int, int] | None = None,
                 with_transpose: bool = False, nrhs_block: int = 0):
        _lib.ensure_device()
        self.n_rows, self.n_cols = int(flat.n_rows), int(flat.n_cols)
        self.row_range = row_range or (0, self.n_rows)
        d, self._keep = flat_desc(flat, row_range, with_transpose, nrhs_block)
        h = C.c_void_p()
        check(lib().hcmx_gpu_hmat_create(C.byref(d), C.byref(h)), "hmat_create")
        self._h = h
        self._keep = None

    def close(self):
        if getattr(self, "_h", None):
            check(lib().hcmx_gpu_hmat_destroy(self._h), "hmat_destroy")
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def memory(self) -> _lib.hcmx_memory_report:
        r = _lib.hcmx_memory_report()
        check(lib().hcmx_gpu_hmat_memory(self._h, C.byref(r)), "hmat_memory")
        return r

    def matvec_device(self, alpha: float, x: torch.Tensor, beta: float, y: torch.Tensor,
                      stream=None) -> torch.Tensor:
        """device pointers, asynchronous on `stream` (default: torch's current)"""
        if x.dtype != torch.float64 or y.dtype != torch.float64 or not (x.is_cuda and y.is_cuda):
            raise ValueError("matvec: x and y must be cuda float64 tensors")
        if x.numel() != self.n_cols or y.numel() != self.n_rows:
            raise ValueError("matvec: dimension mismatch")
        s = stream if stream is not None else torch.cuda.current_stream().cuda_stream
        check(lib().hcmx_gpu_hmat_matvec_device(self._h, float(alpha), ptr(x), float(beta), ptr(y), s),
              "matvec")
        return y

    def matmat4_device(self, alpha: float, X4: torch.Tensor, beta: float, Y4: torch.Tensor):
        """Y4 := alpha M X4 + beta Y4 with X4 (n_cols, 4), Y4 (n_rows, 4) row-major
        cuda float64 tensors, every field decoded once for the 4 columns (handle
        built with nrhs_block=4), on the current stream"""
        if X4.shape != (self.n_cols, 4) or Y4.shape != (self.n_rows, 4) or not (X4.is_contiguous() and
                                                                             Y4.is_contiguous()):
            raise ValueError("matmat4: contiguous (n, 4) float64 tensors required")
        check(lib().hcmx_gpu_hmat_matmat4_device(self._h, float(alpha), ptr(X4), float(beta), ptr(Y4),
                                                 torch.cuda.current_stream().cuda_stream), "matmat4")
        return Y4

    def matvec(self, alpha: float, x, beta: float, y, transpose: bool = False):
        """hmatrix.hpp:126-128 with host vectors (copies in/out inside); transpose:
        y := alpha M^T x + beta y (handle built with with_transpose=True)"""
        if isinstance(x, torch.Tensor) and x.is_cuda and not transpose:
            return self.matvec_device(alpha, x, beta, y)
        xa = np.ascontiguousarray(x, dtype=np.float64)
        nx, ny = (self.n_rows, self.n_cols) if transpose else (self.n_cols, self.n_rows)
        if xa.size != nx or np.asarray(y).size != ny:
            raise ValueError("matvec: dimension mismatch")
        if not (isinstance(y, np.ndarray) and y.dtype == np.float64 and y.flags.c_contiguous):
            raise ValueError("matvec: y must be a contiguous float64 array")
        check(lib().hcmx_gpu_hmat_matvec(self._h, float(alpha), ptr(xa), float(beta), ptr(y),
                                         int(bool(transpose))), "matvec")
        return y

    def matmat(self, alpha: float, X, beta: float, Y, transpose: bool = False):
        """Y := alpha op(M) X + beta Y for the columns of X (host, float64; C5's
        multi-RHS products)"""
        X = np.asfortranarray(X, dtype=np.float64)
        nx, ny = (self.n_rows, self.n_cols) if transpose else (self.n_cols, self.n_rows)
        if X.ndim != 2 or X.shape[0] != nx or Y.shape != (ny, X.shape[1]):
            raise ValueError("matmat: dimension mismatch")
        if not (isinstance(Y, np.ndarray) and Y.dtype == np.float64 and Y.flags.f_contiguous):
            raise ValueError("matmat: Y must be a Fortran-ordered float64 array")
        check(lib().hcmx_gpu_hmat_matmat(self._h, float(alpha), ptr(X), nx, X.shape[1], float(beta), ptr(Y), ny,
                                         int(bool(transpose))), "matmat")
        return Y

    def launches(self) -> int:
        return lib().hcmx_gpu_hmat_last_launches(self._h)

    def timing(self, enable: int):
        a, b, n = C.c_double(), C.c_double(), C.c_uint64()
        check(lib().hcmx_gpu_hmat_timing(self._h, int(enable), C.byref(a), C.byref(b), C.byref(n)),
              "timing")
        return a.value, b.value, n.value

    def export_buffer(self, b: int, nbytes: int) -> bytes:
        out = np.zeros(max(nbytes, 1), np.uint8)
        n = C.c_uint64()
        check(lib().hcmx_gpu_hmat_export_buffer(self._h, b, ptr(out), out.size, C.byref(n)), "export")
        return out[: n.value].tobytes()


def matvec(alpha: float, M: HMatrix, x, beta: float, y, transpose: bool = False):
    """hmatrix.hpp:126-128: y := alpha * op(M) * x + beta * y"""
    return M.matvec(alpha, x, beta, y, transpose)


def build_config_complex(cfg, scheme="afl", device=None, n=None, seed=1, eps=None):
    """setup for config 5 (complex kernel): the real and imaginary H-matrices
    (assemble_complex), each compressed on the GPU with APLR leaves"""
    c = problem_config(cfg) if not isinstance(cfg, dict) else dict(cfg)
    if n is not None:
        c["n"] = n
    if eps is not None:
        c["eps"] = eps
    pts = make_points(c["geometry"], c["n"], seed)
    ct = build_cluster_tree(pts, c["leaf"])
    leaves = build_block_tree(ct, ct, c["eta"])
    Ar, Ai = assemble_complex(pts[ct.i2e], leaves, make_kernel(c["kernel"]), c["eps"], device=device)
    mode = f"{Scheme[scheme].name if isinstance(scheme, str) else Scheme(scheme).name}-aplr"
    fr = compress_in_place(Ar, c["eps"], mode)
    fi = compress_in_place(Ai, c["eps"], mode)
    info = dict(c, leaves=len(leaves), dense_leaves=int((Ar.kind == 0).sum()),
                lowrank_leaves=int((Ar.kind == 1).sum()))
    return fr, fi, info


class ComplexHMatrix:
    """A = Ar + i Ai (config 5): two device-resident real H-matrices on one tree
    whose factors hold the real and imaginary parts as separate codec streams.
    Y = A X for complex X (n x r): [Ar; Ai] applied to [Re X, Im X] (one fused
    product per real column), combined as Re Y = Ar Re X - Ai Im X,
    Im Y = Ar Im X + Ai Re X."""

    def __init__(self, fr: FlatHMatrix, fi: FlatHMatrix, nrhs_block: int = 4):
        self.re, self.im = HMatrix(fr, nrhs_block=nrhs_block), HMatrix(fi, nrhs_block=nrhs_block)
        self.n_rows, self.n_cols = self.re.n_rows, self.re.n_cols

    def close(self):
        self.re.close()
        self.im.close()

    def matmat(self, alpha: complex, X, beta: complex, Y):
        """Y := alpha A X + beta Y (host complex128, X: n x r or n)"""
        X = np.asarray(X, dtype=np.complex128)
        Y = np.asarray(Y)
        vec = X.ndim == 1
        X2 = X[:, None] if vec else X
        if X2.shape[0] != self.n_cols or Y.shape != ((self.n_rows,) if vec else (self.n_rows, X2.shape[1])):
            raise ValueError("matmat: dimension mismatch")
        r = X2.shape[1]
        XX = np.asfortranarray(np.concatenate([X2.real, X2.imag], axis=1))   # [Re X, Im X]
        Pr = np.zeros((self.n_rows, 2 * r), order="F")
        Pi = np.zeros((self.n_rows, 2 * r), order="F")
        self.re.matmat(1.0, XX, 0.0, Pr)
        self.im.matmat(1.0, XX, 0.0, Pi)
        AX = (Pr[:, :r] - Pi[:, r:]) + 1j * (Pr[:, r:] + Pi[:, :r])
        out = alpha * AX + (beta * (Y[:, None] if vec else Y) if beta != 0 else 0.0)
        out = out[:, 0] if vec else out
        Y[...] = out
        return Y

    def matvec(self, alpha: complex, x, beta: complex, y):
        return self.matmat(alpha, x, beta, y)
