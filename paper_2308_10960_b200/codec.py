"""hcmx::codec on the B200 -- same names, argument meaning and errors as
/root/reference/proj/include/hcmx/codec.hpp:74-110, computed by the sm_100a
kernels behind include/hcmx_gpu.h.

Errors: std::invalid_argument -> ValueError, hcmx::corrupt_buffer_error ->
CorruptBufferError.  Single-buffer calls take and return host data (the
reference-facing form); the batched calls keep everything resident in HBM.
"""
from __future__ import annotations

import ctypes as C
import enum
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from ._lib import DESC_DTYPE, STATS_DTYPE, CorruptBufferError, check, lib, ptr, u64p

__all__ = ["Scheme", "FormatDescriptor", "CompressedBuffer", "BlockStats", "analyze",
           "mantissa_bits_for", "exponent_bits_for", "make_descriptor", "compress",
           "compress_block", "decompress", "decompress_into", "compressed_size", "header_bytes",
           "serialize", "deserialize", "scheme_name", "compress_batch", "decompress_batch",
           "CorruptBufferError", "BatchBuffers"]

header_bytes = 20  # codec.hpp:105-107


class Scheme(enum.IntEnum):
    """codec.hpp:22"""
    afl = 0
    aflp = 1
    bfl = 2
    dfl = 3


def scheme_name(s) -> str:
    return Scheme(s).name


@dataclass
class FormatDescriptor:
    """codec.hpp:35-56"""
    scheme: Scheme = Scheme.afl
    exp_bits: int = 2
    mant_bits: int = 2
    scale: float = 1.0

    @staticmethod
    def alignment_unit(s) -> int:
        return {0: 1, 1: 8, 2: 8, 3: 16}[int(s)]

    def bit_width(self) -> int:
        unit = self.alignment_unit(self.scheme)
        w = 1 + self.exp_bits + self.mant_bits
        return w + (unit - w % unit) % unit

    def _c(self) -> _lib.hcmx_descriptor:
        return _lib.hcmx_descriptor(int(self.scheme), self.exp_bits, self.mant_bits,
                                    self.bit_width(), 0, self.scale)

    @staticmethod
    def _from_c(d) -> "FormatDescriptor":
        return FormatDescriptor(Scheme(d.scheme), d.exp_bits, d.mant_bits, d.scale)


@dataclass
class CompressedBuffer:
    """codec.hpp:58-65"""
    descriptor: FormatDescriptor = field(default_factory=FormatDescriptor)
    count: int = 0
    payload: bytes = b""

    def byte_size(self) -> int:
        return header_bytes + len(self.payload)


@dataclass
class BlockStats:
    """codec.hpp:68-72"""
    min_mag: float = 0.0
    max_mag: float = 0.0
    all_zero: bool = True

    def _c(self):
        return _lib.hcmx_stats(self.min_mag, self.max_mag, int(self.all_zero), 0)


def _dev_f64(values) -> torch.Tensor:
    _lib.ensure_device()
    if isinstance(values, torch.Tensor):
        if values.is_cuda and values.dtype == torch.float64 and values.is_contiguous():
            return values.detach()
        return values.detach().to(device="cuda", dtype=torch.float64).contiguous()
    return torch.as_tensor(np.ascontiguousarray(values, dtype=np.float64)).cuda()


def _stream() -> int:
    return torch.cuda.current_stream().cuda_stream


# ------------------------------------------------------------ layout rules --
def mantissa_bits_for(eps: float) -> int:
    """codec.cpp:62-67"""
    out = C.c_uint8()
    check(lib().hcmx_gpu_mantissa_bits_for(float(eps), C.byref(out)), "mantissa_bits_for")
    return out.value


def analyze(values) -> BlockStats:
    """codec.cpp:44-60 (device min/max reduction)"""
    v = _dev_f64(values)
    counts = np.array([v.numel()], dtype=np.uint64)
    voff = torch.zeros(1, dtype=torch.int64, device="cuda")
    st = torch.empty(STATS_DTYPE.itemsize, dtype=torch.uint8, device="cuda")
    check(lib().hcmx_gpu_codec_analyze(ptr(v), ptr(voff), u64p(counts), 1, ptr(st), _stream()),
          "analyze")
    s = np.frombuffer(st.cpu().numpy().tobytes(), dtype=STATS_DTYPE)[0]
    return BlockStats(float(s["min_mag"]), float(s["max_mag"]), bool(s["all_zero"]))


def exponent_bits_for(x) -> int:
    """codec.cpp:69-79 (from values or from BlockStats)"""
    st = x if isinstance(x, BlockStats) else analyze(x)
    out = C.c_uint8()
    cs = st._c()
    check(lib().hcmx_gpu_exponent_bits_for(C.byref(cs), C.byref(out)), "exponent_bits_for")
    return out.value


def make_descriptor(scheme, eps: float, stats_or_scale, exp_bits: int | None = None) -> FormatDescriptor:
    """codec.cpp:81-84 make_descriptor(scheme, eps, stats) and
    codec.cpp:86-101 make_descriptor(scheme, eps, scale, exp_bits)"""
    out = _lib.hcmx_descriptor()
    if isinstance(stats_or_scale, BlockStats):
        cs = stats_or_scale._c()
        check(lib().hcmx_gpu_make_descriptor(int(scheme), float(eps), C.byref(cs), C.byref(out)),
              "make_descriptor")
    else:
        check(lib().hcmx_gpu_make_descriptor_pinned(int(scheme), float(eps), float(stats_or_scale),
                                                     int(exp_bits), C.byref(out)), "make_descriptor")
    return FormatDescriptor._from_c(out)


def compressed_size(count: int, desc: FormatDescriptor) -> int:
    """codec.cpp:179-181"""
    d = desc._c()
    return lib().hcmx_gpu_compressed_size(int(count), C.byref(d))


# ------------------------------------------------------- single buffers ----
def compress(values, eps: float, scheme) -> CompressedBuffer:
    """codec.cpp:142-144 (host in, host out; device kernels in between)"""
    v = np.ascontiguousarray(values, dtype=np.float64).ravel()
    _lib.ensure_device()
    d = _lib.hcmx_descriptor()
    cap = 8 * v.size + 16
    out = np.zeros(cap, dtype=np.uint8)
    n = C.c_uint64()
    check(lib().hcmx_gpu_compress(ptr(v), v.size, float(eps), int(scheme), C.byref(d), ptr(out),
                                  cap, C.byref(n)), "compress")
    return CompressedBuffer(FormatDescriptor._from_c(d), v.size, out[: n.value].tobytes())


def compress_block(values, desc: FormatDescriptor) -> CompressedBuffer:
    """codec.cpp:103-140 with a caller-pinned layout"""
    v = np.ascontiguousarray(values, dtype=np.float64).ravel()
    _lib.ensure_device()
    d = desc._c()
    cap = (v.size * desc.bit_width() + 7) // 8 + 16
    out = np.zeros(cap, dtype=np.uint8)
    n = C.c_uint64()
    check(lib().hcmx_gpu_compress_block(ptr(v), v.size, C.byref(d), ptr(out), cap, C.byref(n)),
          "compress_block")
    return CompressedBuffer(desc, v.size, out[: n.value].tobytes())


def decompress_into(buf: CompressedBuffer, out: np.ndarray) -> None:
    """codec.cpp:146-171"""
    if out.dtype != np.float64 or not out.flags.c_contiguous or out.size < buf.count:
        raise ValueError("decompress_into: out must be a contiguous float64 array of count values")
    _lib.ensure_device()
    d = buf.descriptor._c()
    p = np.frombuffer(buf.payload, dtype=np.uint8) if buf.payload else np.zeros(1, np.uint8)
    check(lib().hcmx_gpu_decompress_into(C.byref(d), buf.count, ptr(p), len(buf.payload), ptr(out)),
          "decompress")


def decompress(buf: CompressedBuffer) -> np.ndarray:
    """codec.cpp:173-177"""
    out = np.empty(buf.count, dtype=np.float64)
    decompress_into(buf, out)
    return out


def serialize(buf: CompressedBuffer) -> bytes:
    """codec.cpp:187-199"""
    d = buf.descriptor._c()
    p = np.frombuffer(buf.payload, dtype=np.uint8) if buf.payload else np.zeros(1, np.uint8)
    out = np.zeros(header_bytes + len(buf.payload), dtype=np.uint8)
    n = lib().hcmx_gpu_serialize(C.byref(d), buf.count, ptr(p), len(buf.payload), ptr(out))
    return out[:n].tobytes()


def deserialize(data: bytes, offset: int = 0):
    """codec.cpp:201-225 -> (CompressedBuffer, new offset)"""
    arr = np.frombuffer(data, dtype=np.uint8) if data else np.zeros(1, np.uint8)
    off = C.c_uint64(offset)
    d = _lib.hcmx_descriptor()
    cnt, at, ln = C.c_uint64(), C.c_uint64(), C.c_uint64()
    check(lib().hcmx_gpu_deserialize(ptr(arr), len(data), C.byref(off), C.byref(d), C.byref(cnt),
                                     C.byref(at), C.byref(ln)), "deserialize")
    return (CompressedBuffer(FormatDescriptor._from_c(d), cnt.value,
                             bytes(data[at.value: at.value + ln.value])), off.value)


# -------------------------------------------------------- batched (HBM) ----
@dataclass
class BatchBuffers:
    """nbuf packed buffers resident in one device arena"""
    desc: np.ndarray          # DESC_DTYPE [nbuf]
    count: np.ndarray         # uint64 [nbuf]
    poff: np.ndarray          # uint64 [nbuf] (16-byte aligned byte offsets)
    payload: torch.Tensor     # uint8 cuda arena
    total: int                # arena bytes used
    _dev: dict = field(default_factory=dict, repr=False)  # cached device copies of the tables

    def dev(self, name: str, host: np.ndarray) -> torch.Tensor:
        t = self._dev.get(name)
        if t is None:
            t = torch.as_tensor(np.ascontiguousarray(host).view(np.uint8)).cuda()
            self._dev[name] = t
        return t

    def __len__(self):
        return self.count.size

    def bit_width(self, b: int) -> int:
        return int(self.desc["bit_width"][b])

    def payload_bytes(self, b: int) -> int:
        return (int(self.count[b]) * self.bit_width(b) + 7) // 8

    def buffer(self, b: int, host_payload: np.ndarray | None = None) -> CompressedBuffer:
        d = self.desc[b]
        fd = FormatDescriptor(Scheme(int(d["scheme"])), int(d["exp_bits"]), int(d["mant_bits"]),
                              float(d["scale"]))
        n = self.payload_bytes(b)
        src = host_payload if host_payload is not None else self.payload.cpu().numpy()
        o = int(self.poff[b])
        return CompressedBuffer(fd, int(self.count[b]), src[o: o + n].tobytes())


def _offsets(counts: np.ndarray) -> np.ndarray:
    voff = np.zeros(counts.size, dtype=np.uint64)
    if counts.size > 1:
        voff[1:] = np.cumsum(counts[:-1], dtype=np.uint64)
    return voff


def compress_batch(values: torch.Tensor, counts, eps: float, scheme, capacity: int | None = None,
                   voff=None, payload: torch.Tensor | None = None,
                   d_voff: torch.Tensor | None = None) -> BatchBuffers:
    """codec::compress over nbuf independent buffers laid end to end in `values`
    (a cuda float64 tensor): one fused kernel per batch (analyze, layout
    selection on the device with a host re-check next to the exponent-width
    thresholds, pack).  Payload slots are sized for the widest layout the scheme
    allows; each buffer's payload is the first payload_bytes(b) of its slot."""
    values = _dev_f64(values)
    counts = np.ascontiguousarray(counts, dtype=np.uint64)
    nb = counts.size
    if d_voff is None:
        vo = _offsets(counts) if voff is None else np.ascontiguousarray(voff, dtype=np.uint64)
        d_voff = torch.as_tensor(vo.view(np.int64)).cuda()
    if capacity is None:
        capacity = int(8 * counts.sum() + 16 * nb + 16)
    if payload is None:
        payload = torch.empty(capacity, dtype=torch.uint8, device="cuda")
    desc = np.zeros(nb, dtype=DESC_DTYPE)
    poff = np.zeros(nb, dtype=np.uint64)
    total = C.c_uint64()
    check(lib().hcmx_gpu_codec_compress(ptr(values), ptr(d_voff), u64p(counts), nb, float(eps),
                                        int(scheme), ptr(payload), payload.numel(), ptr(desc),
                                        u64p(poff), C.byref(total), _stream()), "compress")
    bb = BatchBuffers(desc, counts, poff, payload, total.value)
    if voff is None:
        bb._dev["voff"] = d_voff.view(torch.uint8) if d_voff.dtype != torch.uint8 else d_voff
    return bb


@dataclass
class DeviceBatch:
    """a compress_device batch: every table on the device, nothing read back"""
    count: np.ndarray         # uint64 [nbuf] (host copy, for the fix-up)
    poff: np.ndarray          # uint64 [nbuf] slot offsets (host copy)
    d_count: torch.Tensor
    d_voff: torch.Tensor
    d_poff: torch.Tensor
    d_desc: torch.Tensor      # uint8 [nbuf * 16] (hcmx_descriptor)
    d_flags: torch.Tensor     # int32 [nbuf]
    payload: torch.Tensor
    eps: float
    scheme: int


def device_batch(values: torch.Tensor, counts, eps: float, scheme, voff=None) -> DeviceBatch:
    """tables for compress_device over `values`: slots sized for the widest layout
    the scheme allows (exp_bits 11), 16-byte aligned"""
    counts = np.ascontiguousarray(counts, dtype=np.uint64)
    nb = counts.size
    widest = make_descriptor(scheme, eps, 1.0, 11).bit_width()
    slot = ((counts * np.uint64(widest) + np.uint64(7)) // np.uint64(8) + np.uint64(15)) // np.uint64(16) * np.uint64(16)
    poff = _offsets(slot)
    vo = _offsets(counts) if voff is None else np.ascontiguousarray(voff, dtype=np.uint64)
    tot = int(slot.sum()) + 16
    dv = lambda a: torch.as_tensor(a.view(np.int64)).cuda()
    return DeviceBatch(counts, poff, dv(counts), dv(vo), dv(poff),
                       torch.zeros(16 * max(nb, 1), dtype=torch.uint8, device="cuda"),
                       torch.zeros(max(nb, 1), dtype=torch.int32, device="cuda"),
                       torch.empty(tot, dtype=torch.uint8, device="cuda"), float(eps), int(scheme))


def compress_device(values: torch.Tensor, db: DeviceBatch) -> DeviceBatch:
    """hcmx_gpu_codec_compress_device: one asynchronous launch, no read-back"""
    values = _dev_f64(values)
    check(lib().hcmx_gpu_codec_compress_device(ptr(values), ptr(db.d_voff), ptr(db.d_count), db.count.size,
                                               int(db.count.max()) if db.count.size else 0, db.eps, db.scheme,
                                               ptr(db.d_poff), ptr(db.payload), ptr(db.d_desc), ptr(db.d_flags),
                                               _stream()), "compress_device")
    return db


def compress_device_finish(values: torch.Tensor, db: DeviceBatch) -> tuple[BatchBuffers, int]:
    """hcmx_gpu_codec_compress_fixup, then the batch as BatchBuffers (host descriptors)"""
    values = _dev_f64(values)
    n = C.c_uint64()
    check(lib().hcmx_gpu_codec_compress_fixup(ptr(values), ptr(db.d_voff), u64p(db.count), db.count.size, db.eps,
                                              db.scheme, u64p(db.poff), ptr(db.payload), ptr(db.d_desc),
                                              ptr(db.d_flags), C.byref(n), _stream()), "compress_fixup")
    desc = db.d_desc.cpu().numpy()[: 16 * db.count.size].view(DESC_DTYPE).copy()
    tot = int(db.poff[-1] + (int(db.count[-1]) * int(desc["bit_width"][-1]) + 7) // 8) if db.count.size else 0
    return BatchBuffers(desc, db.count, db.poff, db.payload, tot), n.value


def decompress_batch(bb: BatchBuffers, out: torch.Tensor | None = None, voff=None) -> torch.Tensor:
    """codec::decompress_into for every buffer of a batch (device -> device)"""
    _lib.ensure_device()
    if out is None:
        out = torch.empty(int(bb.count.sum()), dtype=torch.float64, device="cuda")
    if voff is None:
        d_voff = bb.dev("voff", _offsets(bb.count))
    else:
        d_voff = torch.as_tensor(np.ascontiguousarray(voff, dtype=np.uint64).view(np.int64)).cuda()
    d_poff = bb.dev("poff", bb.poff)
    d_desc = bb.dev("desc", bb.desc)
    check(lib().hcmx_gpu_codec_unpack(ptr(bb.payload), ptr(d_poff), u64p(bb.count), ptr(d_desc),
                                      ptr(d_voff), len(bb), ptr(out), _stream()), "decompress")
    return out


def pack_batch(values: torch.Tensor, counts, desc: np.ndarray, voff=None,
               payload: torch.Tensor | None = None) -> BatchBuffers:
    """codec::compress_block over a batch with caller-pinned layouts"""
    values = _dev_f64(values)
    counts = np.ascontiguousarray(counts, dtype=np.uint64)
    nb = counts.size
    vo = _offsets(counts) if voff is None else np.ascontiguousarray(voff, dtype=np.uint64)
    poff = np.zeros(nb, dtype=np.uint64)
    tot = 0
    for b in range(nb):
        poff[b] = tot
        tot += ((int(counts[b]) * int(desc["bit_width"][b]) + 7) // 8 + 15) // 16 * 16
    if payload is None:
        payload = torch.zeros(max(tot, 16), dtype=torch.uint8, device="cuda")
    d_voff = torch.as_tensor(vo.view(np.int64)).cuda()
    d_poff = torch.as_tensor(poff.view(np.int64)).cuda()
    d_desc = torch.as_tensor(np.ascontiguousarray(desc).view(np.uint8)).cuda()
    check(lib().hcmx_gpu_codec_pack(ptr(values), ptr(d_voff), u64p(counts), ptr(d_desc), ptr(d_poff),
                                    nb, ptr(payload), _stream()), "compress_block")
    return BatchBuffers(np.ascontiguousarray(desc), counts, poff, payload, tot)
