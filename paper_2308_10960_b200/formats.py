"""Wire / on-disk formats around the compressed H-matrix.

- APLRLowrank serialization: mixedprec.cpp:300-342 (u32 rank, u8 scheme, three zero
  bytes, f64 sigma[k], then the W columns and the X columns in the codec wire format of
  codec.cpp:187-225).
- MPLowrank serialization: mixedprec.cpp:254-298 (u32 rank, f64 sigma[k], u32 groups,
  then per group u8 format, u32 group rank, W bytes, X bytes; PackedSlice data is
  column-major).
- H-matrix file: magic "HCMX", u32 version, then the leaves in for_each_leaf
  preorder (clustering.cpp:159-166), each as a record (kind, cluster ranges, storage tag)
  followed by its payload buffers in the codec serialization. The reference declares the
  format but ships no writer (hmatrix.hpp:150-153), so the record layout is this
  package's; `load_hcmx` returns a FlatHMatrix the GPU matvec consumes directly.

Host-side byte handling only; malformed input raises CorruptBufferError, mirroring
hcmx::corrupt_buffer_error.
"""
from __future__ import annotations

import struct

import numpy as np

from ._lib import DESC_DTYPE, CorruptBufferError
from .codec import CompressedBuffer, FormatDescriptor, Scheme, deserialize, serialize

MAGIC = b"HCMX"
VERSION = 1
RAW_F64, RAW_F32, RAW_F16 = 4, 5, 6
_RAW_BYTES = {RAW_F64: 8, RAW_F32: 4, RAW_F16: 2}
MP_FORMAT = {RAW_F64: 0, RAW_F32: 1, RAW_F16: 2}  # mixedprec.hpp:20 MpFormat tags


def _need(data: bytes, off: int, n: int, what: str) -> None:
    if off + n > len(data):
        raise CorruptBufferError(f"deserialize: truncated {what}")


# ------------------------------------------------------------------- APLR --
def serialize_aplr(sigma: np.ndarray, scheme: int, w_cols: list[CompressedBuffer],
                   x_cols: list[CompressedBuffer]) -> bytes:
    """mixedprec.cpp:300-311"""
    k = len(sigma)
    if len(w_cols) != k or len(x_cols) != k:
        raise ValueError("serialize_aplr: one W and one X buffer per rank column")
    out = [struct.pack("<IB3x", k, int(scheme)), np.ascontiguousarray(sigma, "<f8").tobytes()]
    out += [serialize(b) for b in w_cols] + [serialize(b) for b in x_cols]
    return b"".join(out)


def deserialize_aplr(data: bytes, offset: int = 0):
    """mixedprec.cpp:313-342 -> (sigma, scheme, w_cols, x_cols, new offset)"""
    _need(data, offset, 8, "aplr header")
    k, tag = struct.unpack_from("<IB", data, offset)
    if tag > 3:
        raise CorruptBufferError("deserialize: unknown codec scheme tag")
    offset += 8
    _need(data, offset, 8 * k, "aplr sigma")
    sigma = np.frombuffer(data, "<f8", k, offset).copy()
    offset += 8 * k
    cols = []
    for _ in range(2 * k):
        b, offset = deserialize(data, offset)
        cols.append(b)
    return sigma, Scheme(tag), cols[:k], cols[k:], offset


# --------------------------------------------------------------------- MP --
def serialize_mp(sigma: np.ndarray, groups: list[tuple[int, int, bytes, bytes]]) -> bytes:
    """mixedprec.cpp:254-264; groups: (raw format 4/5/6, group rank, W bytes, X bytes)"""
    out = [struct.pack("<I", len(sigma)), np.ascontiguousarray(sigma, "<f8").tobytes(),
           struct.pack("<I", len(groups))]
    for fmt, gk, wb, xb in groups:
        out += [struct.pack("<BI", MP_FORMAT[fmt], gk), wb, xb]
    return b"".join(out)


def deserialize_mp(data: bytes, offset: int, rows: int, cols: int):
    """mixedprec.cpp:266-298 -> (sigma, groups, new offset)"""
    _need(data, offset, 4, "mp rank")
    (k,) = struct.unpack_from("<I", data, offset)
    offset += 4
    _need(data, offset, 8 * k + 4, "mp sigma")
    sigma = np.frombuffer(data, "<f8", k, offset).copy()
    offset += 8 * k
    (ng,) = struct.unpack_from("<I", data, offset)
    offset += 4
    groups = []
    for _ in range(ng):
        _need(data, offset, 5, "mp group header")
        tag, gk = struct.unpack_from("<BI", data, offset)
        if tag > 2:
            raise CorruptBufferError("deserialize: unknown mp format tag")
        offset += 5
        fmt = RAW_F64 + tag
        esz = _RAW_BYTES[fmt]
        wbytes, xbytes = esz * rows * gk, esz * cols * gk
        _need(data, offset, wbytes + xbytes, "mp group data")
        groups.append((fmt, gk, bytes(data[offset: offset + wbytes]),
                       bytes(data[offset + wbytes: offset + wbytes + xbytes])))
        offset += wbytes + xbytes
    return sigma, groups, offset


# ------------------------------------------------------------ HCMX file ----
# per leaf: u8 kind (0 dense, 1 per-column lowrank, 2 U V^T), u8 storage tag (codec
# scheme 0-3, or raw 4-6 / MP), u32 row0, row1, col0, col1; then the payload:
#   dense codec      codec::serialize(buffer)
#   dense raw        FP64 words (rows x cols, column-major)
#   kind 1 codec     serialize_aplr          kind 1 raw  serialize_mp
#   kind 2           u32 rank, then U and V: codec::serialize each, or FP64 words
_REC = struct.Struct("<BBIIII")


def _buf(flat, b: int) -> CompressedBuffer:
    d = flat.desc[b]
    fd = FormatDescriptor(Scheme(int(d["scheme"])) if d["scheme"] <= 3 else Scheme.afl,
                          int(d["exp_bits"]), int(d["mant_bits"]), float(d["scale"]))
    p = flat.blob[int(flat.poff[b]): int(flat.poff[b]) + int(flat.plen[b])]
    return CompressedBuffer(fd, int(flat.count[b]), bytes(p))


def _raw_bytes(flat, b: int) -> bytes:
    return bytes(flat.blob[int(flat.poff[b]): int(flat.poff[b]) + int(flat.plen[b])])


def save_hcmx(flat, path: str) -> None:
    """write a FlatHMatrix (host or device blob) as an HCMX file"""
    flat = flat.host()
    out = [MAGIC, struct.pack("<IQQQ", VERSION, flat.n_rows, flat.n_cols, flat.nleaves)]
    for l in range(flat.nleaves):
        kind, b0, k = int(flat.kind[l]), int(flat.buf0[l]), int(flat.rank[l])
        tag = int(flat.desc[b0]["scheme"]) if (kind == 0 or k > 0) and b0 < flat.desc.size else 0
        out.append(_REC.pack(kind, tag, int(flat.row0[l]), int(flat.row1[l]), int(flat.col0[l]),
                             int(flat.col1[l])))
        if kind == 0:
            out.append(serialize(_buf(flat, b0)) if tag <= 3 else _raw_bytes(flat, b0))
        elif kind == 1:
            sig = flat.sigma[int(flat.sig0[l]): int(flat.sig0[l]) + k]
            fmts = [int(flat.desc[b0 + i]["scheme"]) for i in range(k)]
            if k == 0 or fmts[0] <= 3:
                out.append(serialize_aplr(sig, tag, [_buf(flat, b0 + i) for i in range(k)],
                                          [_buf(flat, b0 + k + i) for i in range(k)]))
            else:  # MP: consecutive columns of one format form a group
                groups, i = [], 0
                while i < k:
                    j = i
                    while j < k and fmts[j] == fmts[i]:
                        j += 1
                    groups.append((fmts[i], j - i, b"".join(_raw_bytes(flat, b0 + q) for q in range(i, j)),
                                   b"".join(_raw_bytes(flat, b0 + k + q) for q in range(i, j))))
                    i = j
                out.append(serialize_mp(sig, groups))
        else:
            out.append(struct.pack("<I", k))
            if k > 0:
                for f in range(2):
                    out.append(serialize(_buf(flat, b0 + f)) if tag <= 3 else _raw_bytes(flat, b0 + f))
    with open(path, "wb") as fh:
        fh.write(b"".join(out))


def load_hcmx(path: str):
    """read an HCMX file into a FlatHMatrix (host blob; HMatrix(flat) uploads it)"""
    from .hmatrix import FlatHMatrix
    data = open(path, "rb").read()
    if data[:4] != MAGIC:
        raise CorruptBufferError("hcmx: bad magic")
    _need(data, 4, 28, "hcmx header")
    ver, n_rows, n_cols, nleaves = struct.unpack_from("<IQQQ", data, 4)
    if ver != VERSION:
        raise CorruptBufferError(f"hcmx: unsupported version {ver}")
    off = 32
    leaf = {k: [] for k in ("row0", "row1", "col0", "col1", "kind", "rank", "buf0", "sig0")}
    sigma, descs, counts, payloads = [], [], [], []

    def add(desc_row, count, payload):
        descs.append(desc_row)
        counts.append(count)
        payloads.append(payload)

    def codec_row(b: CompressedBuffer):
        d = np.zeros(1, DESC_DTYPE)[0]
        fd = b.descriptor
        d["scheme"], d["exp_bits"], d["mant_bits"] = int(fd.scheme), fd.exp_bits, fd.mant_bits
        d["bit_width"], d["scale"] = fd.bit_width(), fd.scale
        return d

    def raw_row(fmt):
        d = np.zeros(1, DESC_DTYPE)[0]
        d["scheme"], d["bit_width"], d["scale"] = fmt, 8 * _RAW_BYTES[fmt], 1.0
        return d

    nsig = 0
    for _ in range(nleaves):
        _need(data, off, _REC.size, "hcmx leaf record")
        kind, tag, r0, r1, c0, c1 = _REC.unpack_from(data, off)
        off += _REC.size
        rows, cols = r1 - r0, c1 - c0
        for k_, v in (("row0", r0), ("row1", r1), ("col0", c0), ("col1", c1), ("kind", kind)):
            leaf[k_].append(v)
        leaf["buf0"].append(len(descs))
        leaf["sig0"].append(nsig)
        if kind == 0:
            leaf["rank"].append(0)
            if tag <= 3:
                b, off = deserialize(data, off)
                add(codec_row(b), b.count, b.payload)
            else:
                n = 8 * rows * cols
                _need(data, off, n, "hcmx dense words")
                add(raw_row(RAW_F64), rows * cols, bytes(data[off: off + n]))
                off += n
        elif kind == 1:
            if tag <= 3:
                sig, _, wc, xc, off = deserialize_aplr(data, off)
                for b in wc + xc:
                    add(codec_row(b), b.count, b.payload)
            else:
                sig, groups, off = deserialize_mp(data, off, rows, cols)
                wcol, xcol = [], []
                for fmt, gk, wb, xb in groups:
                    esz = _RAW_BYTES[fmt]
                    wcol += [(fmt, wb[i * esz * rows:(i + 1) * esz * rows]) for i in range(gk)]
                    xcol += [(fmt, xb[i * esz * cols:(i + 1) * esz * cols]) for i in range(gk)]
                for fmt, p in wcol:
                    add(raw_row(fmt), rows, p)
                for fmt, p in xcol:
                    add(raw_row(fmt), cols, p)
            leaf["rank"].append(sig.size)
            sigma.append(sig)
            nsig += sig.size
        elif kind == 2:
            _need(data, off, 4, "hcmx rank")
            (k,) = struct.unpack_from("<I", data, off)
            off += 4
            leaf["rank"].append(k)
            if k > 0:
                for n in (rows * k, cols * k):
                    if tag <= 3:
                        b, off = deserialize(data, off)
                        add(codec_row(b), b.count, b.payload)
                    else:
                        _need(data, off, 8 * n, "hcmx factor words")
                        add(raw_row(RAW_F64), n, bytes(data[off: off + 8 * n]))
                        off += 8 * n
        else:
            raise CorruptBufferError(f"hcmx: unknown leaf kind {kind}")
    poff, blob, at = [], [], 0
    for p in payloads:
        poff.append(at)
        pad = (-len(p)) % 16
        blob.append(p + b"\0" * pad)
        at += len(p) + pad
    desc = np.array(descs, dtype=DESC_DTYPE) if descs else np.zeros(0, DESC_DTYPE)
    arr = {k: np.array(v, np.int64) for k, v in leaf.items()}
    return FlatHMatrix(n_rows, n_cols, arr["row0"], arr["row1"], arr["col0"], arr["col1"], arr["kind"],
                       arr["rank"], arr["buf0"], arr["sig0"],
                       np.concatenate(sigma) if sigma else np.zeros(0), desc,
                       np.array(counts, np.int64), np.array(poff, np.int64),
                       np.array([len(p) for p in payloads], np.int64),
                       np.frombuffer(b"".join(blob) if blob else b"\0" * 16, np.uint8).copy())
