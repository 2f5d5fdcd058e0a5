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
    # complex matrices (config 5, complex_flat): per leaf, 1 for the imaginary part
    # of a dense block; None for real matrices
    imag: np.ndarray | None = None

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
MP_ROUNDOFFS = (1.1e-16, 6.0e-8, 4.9e-4)   # mixedprec.hpp:23 (MP-D-S-H)


def mp_partition(sigma: np.ndarray, delta: float) -> np.ndarray:
    """mixedprec.cpp:66-82: per column, the cheapest of FP64 / FP32 / FP16 whose
    unit roundoff keeps sigma_j * rho <= delta; columns with sigma_j <= delta are
    truncated (-1)."""
    g = np.zeros(sigma.size, np.int64)
    g[sigma * MP_ROUNDOFFS[1] <= delta] = 1
    g[sigma * MP_ROUNDOFFS[2] <= delta] = 2
    g[sigma <= delta] = -1
    return g


_STORE = {"aplr": 0, "codec": 1, "mp": 2, "fp64": 3}   # enum hcmx_storage (include/hcmx_gpu.h)


def compress_in_place(A: Assembled, eps: float, mode: StorageMode | str = "afl-aplr",
                      dense_too: bool = True, threads: int = 1) -> FlatHMatrix:
    """hmatrix.hpp:115-119 on the device through hcmx_gpu_compress_in_place, for
    every StorageMode kind (hmatrix.hpp:32-40):
      aplr  dense -> codec::compress (iff dense_too, else FP64); lowrank -> APLR
            (per-column precision from sigma, mixedprec.cpp:155-187)
      codec dense as above; lowrank U = W diag(sigma), V = X each compressed as
            one buffer (CodecLowrank, hmatrix.hpp:46-49)
      mp    dense FP64 (MP never compresses dense); lowrank W Sigma X^H with the
            columns in FP64 / FP32 / FP16 groups (mp_compress, mixedprec.cpp:94-120)
      fp64  uncompressed: dense FP64, lowrank U, V in FP64 (LowrankBlock)
    Returns the flattened H-matrix (payload blob resident on the GPU); the
    MemoryReport of the reference is FlatHMatrix.memory_footprint()."""
    if isinstance(mode, str):
        mode = StorageMode.parse(mode)
    _lib.ensure_device()
    lv = A.leaves
    L = len(lv)
    keep = []
    i64 = lambda x: keep.append(np.ascontiguousarray(x, dtype=np.int64)) or keep[-1].ctypes.data_as(C.POINTER(C.c_int64))
    dense = A.dense.to("cuda").contiguous()
    W = A.W.to("cuda").contiguous()
    X = A.X.to("cuda").contiguous()
    sigma = np.ascontiguousarray(A.sigma if A.sigma.size else np.zeros(1), np.float64)
    a = _lib.hcmx_assembled()
    a.n_rows = a.n_cols = int(A.n)
    a.nleaves = L
    a.row0, a.row1, a.col0, a.col1 = i64(lv.row0), i64(lv.row1), i64(lv.col0), i64(lv.col1)
    a.kind, a.rank = i64(A.kind), i64(A.rank)
    a.d_dense, a.dense_off = ptr(dense), i64(np.maximum(A.dense_off, 0))
    a.d_W, a.d_X = ptr(W), ptr(X)
    a.w_off, a.x_off = i64(np.maximum(A.w_off, 0)), i64(np.maximum(A.x_off, 0))
    a.sigma = sigma.ctypes.data_as(C.POINTER(C.c_double))
    a.sig_off = i64(np.maximum(A.sig_off, 0))
    h = C.c_void_p()
    rep = _lib.hcmx_memory_report()
    # the library allocates with cudaMalloc: hand torch's cached (free) blocks back first
    torch.cuda.synchronize()
    torch.cuda.empty_cache()
    check(lib().hcmx_gpu_compress_in_place(C.byref(a), float(eps), _STORE[mode.kind], int(mode.scheme),
                                           int(bool(dense_too)), C.byref(h), C.byref(rep),
                                           torch.cuda.current_stream().cuda_stream), "compress_in_place")
    try:
        d = _lib.hcmx_hmat_desc()
        check(lib().hcmx_gpu_flat_desc(h, C.byref(d)), "flat_desc")
        nl, nb, ns = int(d.nleaves), int(d.nbuffers), int(d.nsigma)
        arr = lambda p_, n: np.ctypeslib.as_array(p_, shape=(n,)).copy() if n else np.zeros(0, np.int64)
        desc = np.frombuffer(C.string_at(C.cast(d.desc, C.c_void_p), 16 * nb), dtype=DESC_DTYPE).copy()
        blob = torch.empty(max(int(d.blob_bytes), 16), dtype=torch.uint8, device="cuda")
        check(lib().hcmx_gpu_flat_copy_blob(h, ptr(blob), torch.cuda.current_stream().cuda_stream), "flat_copy_blob")
        flat = FlatHMatrix(int(d.n_rows), int(d.n_cols), arr(d.row0, nl), arr(d.row1, nl), arr(d.col0, nl),
                           arr(d.col1, nl), arr(d.kind, nl), arr(d.rank, nl), arr(d.buf0, nl), arr(d.sig0, nl),
                           np.ctypeslib.as_array(d.sigma, shape=(ns,)).copy(), desc, arr(d.count, nb),
                           arr(d.poff, nb), arr(d.plen, nb), blob,
                           meta={"eps": eps, "mode": mode.name(), "dense_too": dense_too})
    finally:
        check(lib().hcmx_gpu_flat_destroy(h), "flat_destroy")
    return flat


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
    imag = None
    if flat.imag is not None:  # a complex matrix: [Ur Ui] / [Vr Vi] lowrank leaves, Re / Im dense leaves
        imag = np.ascontiguousarray(flat.imag, dtype=np.uint8)
        d.complex_pairs = 1
        d.dense_imag = imag.ctypes.data_as(C.POINTER(C.c_uint8))
    return d, (keep, sigma, desc, blob, imag)


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
        self.nrhs_block = int(lib().hcmx_gpu_hmat_nrhs_block(h))

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

    def matmat_block_device(self, alpha: float, X: torch.Tensor, beta: float, Y: torch.Tensor):
        """Y := alpha M X + beta Y with X (n_cols, B), Y (n_rows, B) row-major cuda
        float64, B = nrhs_block (4 or 8): every field decoded once for the B columns"""
        B = self.nrhs_block
        if not B or X.shape != (self.n_cols, B) or Y.shape != (self.n_rows, B) or not (X.is_contiguous() and
                                                                                     Y.is_contiguous()):
            raise ValueError("matmat_block: contiguous (n, nrhs_block) float64 tensors required")
        check(lib().hcmx_gpu_hmat_matmat_block_device(self._h, float(alpha), ptr(X), float(beta), ptr(Y),
                                                      torch.cuda.current_stream().cuda_stream), "matmat_block")
        return Y

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


def complex_flat(fr: FlatHMatrix, fi: FlatHMatrix) -> FlatHMatrix:
    """One complex H-matrix from the real / imaginary pair of assemble_complex:
    every lowrank leaf of fr already holds A's truncated SVD as W = [Ur Ui], X =
    [Vr Vi], sigma = [S S] (fi's lowrank leaves, [Ui -Ur], are the same streams up
    to signs and are dropped); dense leaves are fr's (Re) plus fi's (Im, flagged
    in `imag`).  Each real / imaginary stream is stored -- and decoded -- once."""
    if fr.n_rows != fi.n_rows or fr.nleaves != fi.nleaves or not np.array_equal(fr.kind, fi.kind):
        raise ValueError("complex_flat: the real and imaginary parts must share one block tree")
    dl = np.nonzero(fi.kind == 0)[0]
    fb = fi.buf0[dl]
    nb = fr.desc.size
    br, bi = fr.blob, fi.blob
    if isinstance(br, torch.Tensor) != isinstance(bi, torch.Tensor):
        raise ValueError("complex_flat: both blobs on the device or both on the host")
    base = (int(br.numel() if isinstance(br, torch.Tensor) else br.size) + 15) // 16 * 16
    if isinstance(br, torch.Tensor):
        pad = torch.zeros(base - br.numel(), dtype=torch.uint8, device=br.device)
        blob = torch.cat([br, pad, bi])
    else:
        blob = np.concatenate([br, np.zeros(base - br.size, np.uint8), bi])
    cat = lambda a, b: np.concatenate([np.asarray(a), np.asarray(b)])
    z = np.zeros(dl.size, np.int64)
    return FlatHMatrix(fr.n_rows, fr.n_cols, cat(fr.row0, fi.row0[dl]), cat(fr.row1, fi.row1[dl]),
                       cat(fr.col0, fi.col0[dl]), cat(fr.col1, fi.col1[dl]), cat(fr.kind, z), cat(fr.rank, z),
                       cat(fr.buf0, nb + np.arange(dl.size, dtype=np.int64)), cat(fr.sig0, z), fr.sigma,
                       np.concatenate([fr.desc, fi.desc[fb]]), cat(fr.count, fi.count[fb]),
                       cat(fr.poff, fi.poff[fb] + base), cat(fr.plen, fi.plen[fb]), blob,
                       meta=dict(fr.meta, complex=True),
                       imag=np.concatenate([np.zeros(fr.nleaves, np.uint8), np.ones(dl.size, np.uint8)]))


class ComplexHMatrix:
    """A = Ar + i Ai (config 5) as ONE device-resident complex arena (complex_flat:
    hcmx_hmat_desc::complex_pairs): each real / imaginary factor or block stream
    is decoded once per product and feeds the real and the imaginary output.
    Products take nrhs_block / 2 complex columns at a time through the block
    kernels ([Re x1, Im x1, Re x2, ...] in, [Re y1, Im y1, ...] out); the
    complex combination of the X^T x halves runs on the device between the
    phases (k_ccombine), so Y = A X needs no host arithmetic."""

    def __init__(self, fr: FlatHMatrix, fi: FlatHMatrix | None = None, nrhs_block: int = 4):
        cf = fr if fi is None else complex_flat(fr, fi)
        if cf.imag is None:
            raise ValueError("ComplexHMatrix: a complex flat (complex_flat) or the real / imaginary pair")
        self.h = HMatrix(cf, nrhs_block=nrhs_block)
        self.pairs = nrhs_block // 2  # complex columns per device product
        self.n_rows, self.n_cols = self.h.n_rows, self.h.n_cols

    def close(self):
        self.h.close()

    def memory(self):
        return self.h.memory()

    def matmat_device(self, X: torch.Tensor, Y: torch.Tensor | None = None, alpha: complex = 1.0,
                      beta: complex = 0.0) -> torch.Tensor:
        """Y := alpha A X + beta Y for complex128 cuda X (n x r), nrhs_block / 2
        columns per device product"""
        if X.dtype != torch.complex128 or not X.is_cuda or X.ndim != 2 or X.shape[0] != self.n_cols:
            raise ValueError("matmat_device: complex128 cuda X (n_cols x r) required")
        r, n = X.shape[1], self.n_rows
        if Y is None:
            Y = torch.zeros(n, r, dtype=torch.complex128, device="cuda")
        elif Y.dtype != torch.complex128 or Y.shape != (n, r):
            raise ValueError("matmat_device: Y must be complex128 n_rows x r")
        q, B = self.pairs, 2 * self.pairs
        XB = torch.zeros(self.n_cols, B, dtype=torch.float64, device="cuda")
        YB = torch.empty(n, B, dtype=torch.float64, device="cuda")
        for j in range(0, r, q):
            m = min(q, r - j)
            if m < q:
                XB.zero_()
            XB[:, 0: 2 * m].copy_(torch.view_as_real(X[:, j: j + m]).reshape(self.n_cols, 2 * m))
            self.h.matmat_block_device(1.0, XB, 0.0, YB)
            AX = torch.view_as_complex(YB.view(n, q, 2))[:, :m]
            if beta == 0:
                Y[:, j: j + m] = alpha * AX if alpha != 1 else AX
            else:
                Y[:, j: j + m] = alpha * AX + beta * Y[:, j: j + m]
        return Y

    def matmat(self, alpha: complex, X, beta: complex, Y):
        """Y := alpha A X + beta Y (host complex128, X: n x r or n)"""
        X = np.asarray(X, dtype=np.complex128)
        vec = X.ndim == 1
        X2 = X[:, None] if vec else X
        if X2.shape[0] != self.n_cols or Y.shape != ((self.n_rows,) if vec else (self.n_rows, X2.shape[1])):
            raise ValueError("matmat: dimension mismatch")
        Yd = torch.as_tensor(np.ascontiguousarray(Y).reshape(self.n_rows, -1)).cuda()
        out = self.matmat_device(torch.as_tensor(np.ascontiguousarray(X2)).cuda(), Yd, alpha, beta).cpu().numpy()
        Y[...] = out[:, 0] if vec else out
        return Y

    def matvec(self, alpha: complex, x, beta: complex, y):
        return self.matmat(alpha, x, beta, y)
