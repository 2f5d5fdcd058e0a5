"""TEST INFRASTRUCTURE ONLY -- ctypes front end of the two CPU checkers.

* ``Oracle``    -> oracle/liboracle.so, our plain-C restatement (hcmx_oracle.c)
* ``RefOracle`` -> oracle/_ref/libhcmx_ref.so, the unmodified reference codec
                   (/root/reference/proj/src/codec.cpp) + restated APLR/matvec glue

Only tests/, ``__graft_entry__.smoke()`` and bench.py's CPU legs may import
this module.  The product package never does.  Both classes expose the same
methods so tests can run one against the other.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
OK, INVALID_ARGUMENT, CORRUPT_BUFFER = 0, 1, 2
SCHEMES = {"afl": 0, "aflp": 1, "bfl": 2, "dfl": 3}


class CorruptBufferError(RuntimeError):
    """mirror of hcmx::corrupt_buffer_error (common.hpp:17-19)"""


def _check(st: int, what: str) -> None:
    if st == OK:
        return
    if st == INVALID_ARGUMENT:
        raise ValueError(f"{what}: invalid argument")
    if st == CORRUPT_BUFFER:
        raise CorruptBufferError(f"{what}: corrupt buffer")
    raise RuntimeError(f"{what}: status {st}")


@dataclass
class Buf:
    """mirror of codec::CompressedBuffer (codec.hpp:58-65)"""
    scheme: int
    e: int
    m: int
    scale: float
    count: int
    payload: bytes

    def bit_width(self) -> int:
        unit = {0: 1, 1: 8, 2: 8, 3: 16}[self.scheme]
        w = 1 + self.e + self.m
        return w + (unit - w % unit) % unit


def _p(a, t):
    return a.ctypes.data_as(C.POINTER(t))


_d, _i64, _u8, _i32, _u64 = C.c_double, C.c_int64, C.c_uint8, C.c_int, C.c_uint64
_pd, _pi64, _pu8, _pi32 = C.POINTER(_d), C.POINTER(_i64), C.POINTER(_u8), C.POINTER(_i32)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


class _Base:
    prefix = ""
    libpath = ""

    def __init__(self, path: str | None = None):
        self.lib = C.CDLL(path or self.libpath)
        self._bind()

    def _fn(self, name, res, *args):
        f = getattr(self.lib, self.prefix + name)
        f.restype = res
        f.argtypes = list(args)
        return f

    def _bind(self):
        self._mt = self._fn("mt64_raw", None, _u64, _i64, C.POINTER(_u64))
        self._analyze = self._fn("analyze", None, _pd, _i64, _pd, _pd, _pi32)
        self._mbits = self._fn("mantissa_bits_for", _i32, _d, _pi32)
        self._ebits = self._fn("exponent_bits_for", _i32, _pd, _i64)
        self._ebits_st = self._fn("exponent_bits_for_stats", _i32, _d, _d, _i32)
        self._bw = self._fn("bit_width", _i32, _i32, _i32, _i32)
        self._csize = self._fn("compressed_size", _i64, _i64, _i32, _i32, _i32)

    # --- scalar layout --------------------------------------------------
    def mt64_raw(self, seed: int, n: int) -> np.ndarray:
        out = np.empty(n, dtype=np.uint64)
        self._mt(seed, n, _p(out, _u64))
        return out

    def analyze(self, v):
        v = _f64(v)
        mn, mx, az = _d(), _d(), _i32()
        self._analyze(_p(v, _d), v.size, C.byref(mn), C.byref(mx), C.byref(az))
        return mn.value, mx.value, bool(az.value)

    def mantissa_bits_for(self, eps: float) -> int:
        out = _i32()
        _check(self._mbits(eps, C.byref(out)), "mantissa_bits_for")
        return out.value

    def exponent_bits_for(self, v) -> int:
        v = _f64(v)
        return self._ebits(_p(v, _d), v.size)

    def exponent_bits_for_stats(self, mn, mx, az) -> int:
        return self._ebits_st(mn, mx, int(az))

    def bit_width(self, scheme, e, m) -> int:
        return self._bw(scheme, e, m)

    def compressed_size(self, count, scheme, e, m) -> int:
        return self._csize(count, scheme, e, m)


class Oracle(_Base):
    """our C restatement (oracle/hcmx_oracle.c)"""
    prefix = "orc_"
    libpath = os.path.join(HERE, "liboracle.so")

    def _bind(self):
        super()._bind()
        self._mkd = self._fn("make_descriptor", _i32, _i32, _d, _i32, _pi32, _pi32)
        self._cb = self._fn("compress_block", _i32, _pd, _i64, _i32, _i32, _i32, _d, _pu8)
        self._c = self._fn("compress", _i32, _pd, _i64, _d, _i32, _pi32, _pi32, _pd, _pu8)
        self._dc = self._fn("decompress", _i32, _i32, _i32, _i32, _d, _i64, _pu8, _i64, _pd)
        self._aplr = self._fn("aplr_compress", _i32, _pd, _i64, _pd, _i64, _i64, _pd, _d, _i32,
                              _pi32, _pi32, _pd, _pi64, _pu8)
        self._mv = self._fn("hmat_matvec_flat", _i32, _i64, _i64, _i64, *([_pi64] * 8), _pd,
                            _pu8, _pu8, _pu8, _pd, _pi64, _pi64, _pi64, _pu8, _pd, _d, _pd, _d,
                            _pd, _i32)
        self._mvt = self._fn("hmat_matvec_t_flat", _i32, _i64, _i64, _i64, *([_pi64] * 8), _pd,
                             _pu8, _pu8, _pu8, _pd, _pi64, _pi64, _pi64, _pu8, _pd, _d, _pd, _d,
                             _pd, _i32, _i32)
        self._cbat = self._fn("compress_batch", _i32, _pd, _pi64, _pi64, _i64, _d, _i32, _pi32,
                              _pi32, _pd, _pi64, _pu8, _i32)
        self._dbat = self._fn("decompress_batch", _i32, _pu8, _pi64, _pi64, _pi64, _i64, _i32,
                              _pi32, _pi32, _pd, _pd, _i32)
        self._lus = self._fn("log_uniform_signed", None, _u64, _i64, _d, _d, _pd)
        self._c2 = self._fn("config2_values", None, _u64, _i64, _pd)
        self._f2h = self._fn("float_to_half", C.c_uint16, C.c_float)
        self._h2f = self._fn("half_to_float", C.c_float, C.c_uint16)
        self._praw = self._fn("pack_raw", None, _pd, _i64, _i32, _pu8)
        self._mpp = self._fn("mp_partition", None, _pd, _i64, _d, _pi64)

    def float_to_half(self, f: float) -> int:
        """half.hpp:14-45"""
        return int(self._f2h(f))

    def half_to_float(self, h: int) -> float:
        """half.hpp:47-72"""
        return float(self._h2f(h))

    def pack_raw(self, v, fmt: int) -> bytes:
        """PackedSlice::pack (mixedprec.cpp:16-41); fmt 4 fp64, 5 fp32, 6 fp16"""
        v = np.ascontiguousarray(v, np.float64)
        out = np.zeros(v.size * {4: 8, 5: 4, 6: 2}[fmt] + 1, np.uint8)
        self._praw(_p(v, _d), v.size, fmt, _p(out, _u8))
        return out[:-1].tobytes()

    def mp_partition(self, sigma, delta: float):
        """mixedprec.cpp:66-82: ranks of the FP64 / FP32 / FP16 groups"""
        sigma = np.ascontiguousarray(sigma, np.float64)
        out = np.zeros(3, np.int64)
        self._mpp(_p(sigma, _d), sigma.size, float(delta), _p(out, _i64))
        return out

    def log_uniform_signed(self, seed, n, lo, hi):
        out = np.empty(n)
        self._lus(seed, n, lo, hi, _p(out, _d))
        return out

    def config2_values(self, seed, n):
        out = np.empty(n)
        self._c2(seed, n, _p(out, _d))
        return out

    def make_descriptor(self, scheme, eps, exp_bits):
        e, m = _i32(), _i32()
        _check(self._mkd(scheme, eps, exp_bits, C.byref(e), C.byref(m)), "make_descriptor")
        return e.value, m.value

    def payload_bytes(self, count, scheme, e, m):
        return (count * self.bit_width(scheme, e, m) + 7) // 8

    def compress_block(self, v, scheme, e, m, scale) -> bytes:
        v = _f64(v)
        out = np.zeros(self.payload_bytes(v.size, scheme, e, m) + 8, dtype=np.uint8)
        _check(self._cb(_p(v, _d), v.size, scheme, e, m, scale, _p(out, _u8)), "compress_block")
        return out[: self.payload_bytes(v.size, scheme, e, m)].tobytes()

    def compress(self, v, eps, scheme) -> Buf:
        v = _f64(v)
        out = np.zeros(8 * v.size + 16, dtype=np.uint8)
        e, m, sc = _i32(), _i32(), _d()
        _check(self._c(_p(v, _d), v.size, eps, scheme, C.byref(e), C.byref(m), C.byref(sc),
                       _p(out, _u8)), "compress")
        n = self.payload_bytes(v.size, scheme, e.value, m.value)
        return Buf(scheme, e.value, m.value, sc.value, v.size, out[:n].tobytes())

    def decompress(self, b: Buf) -> np.ndarray:
        out = np.empty(b.count)
        p = np.frombuffer(b.payload, dtype=np.uint8).copy() if b.payload else np.zeros(1, np.uint8)
        _check(self._dc(b.scheme, b.e, b.m, b.scale, b.count, _p(p, _u8), len(b.payload),
                        _p(out, _d)), "decompress")
        return out

    def aplr_compress(self, W, X, sigma, eps, scheme):
        return _aplr(self._aplr, W, X, sigma, eps, scheme)

    def hmat_matvec(self, h, alpha, x, beta, y, threads=1, transpose=False):
        """hmatrix.hpp:126-128 (transpose: y := alpha M^T x + beta y)"""
        if transpose:
            return _matvec(self._mvt, h, alpha, x, beta, y, threads, transpose=True)
        return _matvec(self._mv, h, alpha, x, beta, y, threads)

    def compress_batch(self, values, counts, eps, scheme, threads=1):
        values = _f64(values)
        counts = np.ascontiguousarray(counts, dtype=np.int64)
        nb = counts.size
        voff = np.zeros(nb, np.int64)
        voff[1:] = np.cumsum(counts)[:-1]
        poff = voff * 8
        blob = np.zeros(int(counts.sum()) * 8 + 16, np.uint8)
        e = np.zeros(nb, np.int32); m = np.zeros(nb, np.int32); sc = np.zeros(nb)
        _check(self._cbat(_p(values, _d), _p(voff, _i64), _p(counts, _i64), nb, eps, scheme,
                          _p(e, _i32), _p(m, _i32), _p(sc, _d), _p(poff, _i64), _p(blob, _u8),
                          threads), "compress_batch")
        return e, m, sc, poff, blob

    def decompress_batch(self, blob, poff, counts, scheme, e, m, sc, threads=1):
        counts = np.ascontiguousarray(counts, dtype=np.int64)
        nb = counts.size
        voff = np.zeros(nb, np.int64)
        voff[1:] = np.cumsum(counts)[:-1]
        out = np.empty(int(counts.sum()))
        _check(self._dbat(_p(blob, _u8), _p(poff, _i64), _p(counts, _i64), _p(voff, _i64), nb,
                          scheme, _p(e, _i32), _p(m, _i32), _p(sc, _d), _p(out, _d), threads),
               "decompress_batch")
        return out


class RefOracle(_Base):
    """the reference codec itself (oracle/_ref/libhcmx_ref.so)"""
    prefix = "ref_"
    libpath = os.path.join(HERE, "_ref", "libhcmx_ref.so")

    @staticmethod
    def available(path: str | None = None) -> bool:
        return os.path.exists(path or RefOracle.libpath)

    def float_to_half(self, f: float) -> int:
        return int(self._f2h(f))

    def half_to_float(self, h: int) -> float:
        return float(self._h2f(h))

    def _bind(self):
        super()._bind()
        self._f2h = self._fn("float_to_half", C.c_uint16, C.c_float)
        self._h2f = self._fn("half_to_float", C.c_float, C.c_uint16)
        self._mkd = self._fn("make_descriptor", _i32, _i32, _d, _d, _i32, _pi32, _pi32)
        self._mkds = self._fn("make_descriptor_stats", _i32, _i32, _d, _d, _d, _i32, _pi32,
                              _pi32, _pd)
        self._cb = self._fn("compress_block", _i32, _pd, _i64, _i32, _i32, _i32, _d, _pu8, _i64,
                            _pi64)
        self._c = self._fn("compress", _i32, _pd, _i64, _d, _i32, _pi32, _pi32, _pd, _pu8, _i64,
                           _pi64)
        self._dc = self._fn("decompress", _i32, _i32, _i32, _i32, _d, _i64, _pu8, _i64, _pd)
        self._ser = self._fn("serialize", _i64, _i32, _i32, _i32, _d, _i64, _pu8, _i64, _pu8)
        self._des = self._fn("deserialize", _i32, _pu8, _i64, _pi64, _pi32, _pi32, _pi32, _pd,
                             _pi64, _pi64, _pi64)
        self._aplr = self._fn("aplr_compress", _i32, _pd, _i64, _pd, _i64, _i64, _pd, _d, _i32,
                              _pi32, _pi32, _pd, _pi64, _pu8)
        self._mv = self._fn("hmat_matvec_flat", _i32, _i64, _i64, _i64, *([_pi64] * 8), _pd,
                            _pu8, _pu8, _pu8, _pd, _pi64, _pi64, _pi64, _pu8, _pd, _d, _pd, _d,
                            _pd, _i32)
        self._cbat = self._fn("compress_batch", _i32, _pd, _pi64, _pi64, _i64, _d, _i32, _pi32,
                              _pi32, _pd, _pi64, _pu8, _pi64, _i32)
        self._dbat = self._fn("decompress_batch", _i32, _pu8, _pi64, _pi64, _pi64, _pi64, _i64,
                              _i32, _pi32, _pi32, _pd, _pd, _i32)

    def make_descriptor(self, scheme, eps, exp_bits, scale=1.0):
        e, m = _i32(), _i32()
        _check(self._mkd(scheme, eps, scale, exp_bits, C.byref(e), C.byref(m)), "make_descriptor")
        return e.value, m.value

    def make_descriptor_stats(self, scheme, eps, mn, mx, az):
        e, m, sc = _i32(), _i32(), _d()
        _check(self._mkds(scheme, eps, mn, mx, int(az), C.byref(e), C.byref(m), C.byref(sc)),
               "make_descriptor")
        return e.value, m.value, sc.value

    def compress_block(self, v, scheme, e, m, scale) -> bytes:
        v = _f64(v)
        out = np.zeros(8 * v.size + 16, dtype=np.uint8)
        ln = _i64()
        _check(self._cb(_p(v, _d), v.size, scheme, e, m, scale, _p(out, _u8), out.size,
                        C.byref(ln)), "compress_block")
        return out[: ln.value].tobytes()

    def compress(self, v, eps, scheme) -> Buf:
        v = _f64(v)
        out = np.zeros(8 * v.size + 16, dtype=np.uint8)
        e, m, sc, ln = _i32(), _i32(), _d(), _i64()
        _check(self._c(_p(v, _d), v.size, eps, scheme, C.byref(e), C.byref(m), C.byref(sc),
                       _p(out, _u8), out.size, C.byref(ln)), "compress")
        return Buf(scheme, e.value, m.value, sc.value, v.size, out[: ln.value].tobytes())

    def decompress(self, b: Buf) -> np.ndarray:
        out = np.empty(b.count)
        p = np.frombuffer(b.payload, dtype=np.uint8).copy() if b.payload else np.zeros(1, np.uint8)
        _check(self._dc(b.scheme, b.e, b.m, b.scale, b.count, _p(p, _u8), len(b.payload),
                        _p(out, _d)), "decompress")
        return out

    def serialize(self, b: Buf) -> bytes:
        p = np.frombuffer(b.payload, dtype=np.uint8).copy() if b.payload else np.zeros(1, np.uint8)
        out = np.zeros(20 + len(b.payload), np.uint8)
        n = self._ser(b.scheme, b.e, b.m, b.scale, b.count, _p(p, _u8), len(b.payload),
                      _p(out, _u8))
        return out[:n].tobytes()

    def deserialize(self, data: bytes, offset: int = 0):
        d = np.frombuffer(data, dtype=np.uint8).copy() if data else np.zeros(1, np.uint8)
        off = _i64(offset)
        s, e, m, sc, cnt, at, ln = _i32(), _i32(), _i32(), _d(), _i64(), _i64(), _i64()
        _check(self._des(_p(d, _u8), len(data), C.byref(off), C.byref(s), C.byref(e), C.byref(m),
                         C.byref(sc), C.byref(cnt), C.byref(at), C.byref(ln)), "deserialize")
        b = Buf(s.value, e.value, m.value, sc.value, cnt.value,
                bytes(data[at.value: at.value + ln.value]))
        return b, off.value

    def aplr_compress(self, W, X, sigma, eps, scheme):
        return _aplr(self._aplr, W, X, sigma, eps, scheme)

    def hmat_matvec(self, h, alpha, x, beta, y, threads=1):
        return _matvec(self._mv, h, alpha, x, beta, y, threads)

    def compress_batch(self, values, counts, eps, scheme, threads=1):
        values = _f64(values)
        counts = np.ascontiguousarray(counts, dtype=np.int64)
        nb = counts.size
        voff = np.zeros(nb, np.int64)
        voff[1:] = np.cumsum(counts)[:-1]
        poff = voff * 8
        blob = np.zeros(int(counts.sum()) * 8 + 16, np.uint8)
        plen = np.zeros(nb, np.int64)
        e = np.zeros(nb, np.int32); m = np.zeros(nb, np.int32); sc = np.zeros(nb)
        _check(self._cbat(_p(values, _d), _p(voff, _i64), _p(counts, _i64), nb, eps, scheme,
                          _p(e, _i32), _p(m, _i32), _p(sc, _d), _p(poff, _i64), _p(blob, _u8),
                          _p(plen, _i64), threads), "compress_batch")
        return e, m, sc, poff, blob, plen

    def decompress_batch(self, blob, poff, plen, counts, scheme, e, m, sc, threads=1):
        counts = np.ascontiguousarray(counts, dtype=np.int64)
        nb = counts.size
        voff = np.zeros(nb, np.int64)
        voff[1:] = np.cumsum(counts)[:-1]
        out = np.empty(int(counts.sum()))
        _check(self._dbat(_p(blob, _u8), _p(poff, _i64), _p(plen, _i64), _p(counts, _i64),
                          _p(voff, _i64), nb, scheme, _p(e, _i32), _p(m, _i32), _p(sc, _d),
                          _p(out, _d), threads), "decompress_batch")
        return out


def _aplr(fn, W, X, sigma, eps, scheme):
    W = np.asfortranarray(W, dtype=np.float64)
    X = np.asfortranarray(X, dtype=np.float64)
    sigma = _f64(sigma)
    rows, k = W.shape
    cols = X.shape[0]
    nb = 2 * k
    e = np.zeros(max(nb, 1), np.int32); m = np.zeros(max(nb, 1), np.int32)
    sc = np.zeros(max(nb, 1)); offs = np.zeros(nb + 1, np.int64)
    blob = np.zeros(8 * (rows + cols) * max(k, 1) + 16, np.uint8)
    Wf = W.ravel(order="F").copy()
    Xf = X.ravel(order="F").copy()
    _check(fn(_p(Wf, _d), rows, _p(Xf, _d), cols, k, _p(sigma, _d) if sigma.size else None, eps,
              scheme, _p(e, _i32), _p(m, _i32), _p(sc, _d), _p(offs, _i64), _p(blob, _u8)),
           "aplr_compress")
    bufs = []
    for b in range(nb):
        cnt = rows if b < k else cols
        bufs.append(Buf(scheme, int(e[b]), int(m[b]), float(sc[b]), cnt,
                        blob[offs[b]: offs[b + 1]].tobytes()))
    return bufs


def _matvec(fn, h, alpha, x, beta, y, threads, transpose=None):
    """h: any object with the flat H-matrix arrays (see hcmx_oracle.c)"""
    x = _f64(x)
    y = np.array(y, dtype=np.float64, copy=True)
    a = lambda name, t: np.ascontiguousarray(getattr(h, name), dtype=t)
    arrs = {k: a(k, np.int64) for k in ("row0", "row1", "col0", "col1", "kind", "rank", "buf0",
                                        "sig0", "count", "poff", "plen")}
    u8 = {k: a(k, np.uint8) for k in ("scheme", "e", "m")}
    sigma = a("sigma", np.float64)
    scale = a("scale", np.float64)
    blob = a("blob", np.uint8)
    raw = a("raw", np.float64) if getattr(h, "raw", None) is not None else np.zeros(1)
    if sigma.size == 0:
        sigma = np.zeros(1)
    if blob.size == 0:
        blob = np.zeros(1, np.uint8)
    _check(fn(h.n_rows, h.n_cols, arrs["row0"].size,
              *[_p(arrs[k], _i64) for k in ("row0", "row1", "col0", "col1", "kind", "rank",
                                           "buf0", "sig0")],
              _p(sigma, _d), _p(u8["scheme"], _u8), _p(u8["e"], _u8), _p(u8["m"], _u8),
              _p(scale, _d), _p(arrs["count"], _i64), _p(arrs["poff"], _i64),
              _p(arrs["plen"], _i64), _p(blob, _u8), _p(raw, _d), alpha, _p(x, _d), beta,
              _p(y, _d), threads, *([] if transpose is None else [int(transpose)])), "hmat_matvec")
    return y
