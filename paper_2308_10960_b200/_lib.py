"""ctypes binding of libhcmx_gpu.so (the C-ABI declared in include/hcmx_gpu.h).

The library is built in-tree by ``paper_2308_10960_b200.build``.  There is no
fallback: if the shared object is missing, importing the product API raises.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIBPATH = os.environ.get("HCMX_GPU_LIB") or os.path.join(HERE, "libhcmx_gpu.so")

HCMX_OK, HCMX_INVALID_ARGUMENT, HCMX_CORRUPT_BUFFER = 0, 1, 2
HCMX_CUDA_ERROR, HCMX_NCCL_ERROR, HCMX_OUT_OF_MEMORY = 3, 4, 5


class CorruptBufferError(RuntimeError):
    """hcmx::corrupt_buffer_error (proj/include/hcmx/common.hpp:17-19)"""


class CudaError(RuntimeError):
    pass


class NcclError(RuntimeError):
    """HCMX_NCCL_ERROR: a failed NCCL call of the multi-GPU exchange"""


class hcmx_descriptor(C.Structure):
    _fields_ = [("scheme", C.c_uint8), ("exp_bits", C.c_uint8), ("mant_bits", C.c_uint8),
                ("bit_width", C.c_uint8), ("reserved", C.c_uint32), ("scale", C.c_double)]


class hcmx_stats(C.Structure):
    _fields_ = [("min_mag", C.c_double), ("max_mag", C.c_double), ("all_zero", C.c_uint32),
                ("non_finite", C.c_uint32)]


_pi64 = C.POINTER(C.c_int64)


class hcmx_hmat_desc(C.Structure):
    _fields_ = [("n_rows", C.c_uint64), ("n_cols", C.c_uint64), ("nleaves", C.c_uint64),
                ("nbuffers", C.c_uint64), ("nsigma", C.c_uint64), ("blob_bytes", C.c_uint64),
                ("row0", _pi64), ("row1", _pi64), ("col0", _pi64), ("col1", _pi64),
                ("kind", _pi64), ("rank", _pi64), ("buf0", _pi64), ("sig0", _pi64),
                ("sigma", C.POINTER(C.c_double)), ("desc", C.POINTER(hcmx_descriptor)),
                ("count", _pi64), ("poff", _pi64), ("plen", _pi64),
                ("blob", C.c_void_p), ("blob_on_device", C.c_int),
                ("row_begin", C.c_uint64), ("row_end", C.c_uint64), ("with_transpose", C.c_int),
                ("nrhs_block", C.c_int), ("complex_pairs", C.c_int), ("dense_imag", C.POINTER(C.c_uint8))]


class hcmx_assembled(C.Structure):
    _fields_ = [("n_rows", C.c_uint64), ("n_cols", C.c_uint64), ("nleaves", C.c_uint64),
                ("row0", _pi64), ("row1", _pi64), ("col0", _pi64), ("col1", _pi64),
                ("kind", _pi64), ("rank", _pi64), ("d_dense", C.c_void_p), ("dense_off", _pi64),
                ("d_W", C.c_void_p), ("d_X", C.c_void_p), ("w_off", _pi64), ("x_off", _pi64),
                ("sigma", C.POINTER(C.c_double)), ("sig_off", _pi64)]


class hcmx_memory_report(C.Structure):
    _fields_ = [(n, C.c_uint64) for n in (
        "dense_raw", "dense_compressed", "lowrank_raw", "lowrank_compressed", "overhead",
        "uncompressed_equivalent", "device_arena_bytes", "device_table_bytes",
        "algorithmic_bytes", "dense_leaves", "lowrank_leaves", "stages_a", "stages_b")]


# numpy twin of hcmx_descriptor (16 bytes) for bulk descriptor arrays
DESC_DTYPE = np.dtype([("scheme", "u1"), ("exp_bits", "u1"), ("mant_bits", "u1"),
                       ("bit_width", "u1"), ("reserved", "<u4"), ("scale", "<f8")])
STATS_DTYPE = np.dtype([("min_mag", "<f8"), ("max_mag", "<f8"), ("all_zero", "<u4"),
                        ("non_finite", "<u4")])
assert DESC_DTYPE.itemsize == C.sizeof(hcmx_descriptor) == 16
assert STATS_DTYPE.itemsize == C.sizeof(hcmx_stats) == 24

_u64, _d, _i, _vp = C.c_uint64, C.c_double, C.c_int, C.c_void_p
_pu64 = C.POINTER(C.c_uint64)
_pdesc = C.POINTER(hcmx_descriptor)

# name -> (restype, argtypes); every function declared in include/hcmx_gpu.h
PROTOTYPES = {
    "hcmx_gpu_init": (_i, [_i]),
    "hcmx_gpu_last_error": (C.c_char_p, []),
    "hcmx_gpu_version": (_i, []),
    "hcmx_gpu_mantissa_bits_for": (_i, [_d, C.POINTER(C.c_uint8)]),
    "hcmx_gpu_exponent_bits_for": (_i, [C.POINTER(hcmx_stats), C.POINTER(C.c_uint8)]),
    "hcmx_gpu_make_descriptor": (_i, [_i, _d, C.POINTER(hcmx_stats), _pdesc]),
    "hcmx_gpu_make_descriptor_pinned": (_i, [_i, _d, _d, C.c_uint8, _pdesc]),
    "hcmx_gpu_bit_width": (C.c_uint, [_pdesc]),
    "hcmx_gpu_compressed_size": (_u64, [_u64, _pdesc]),
    "hcmx_gpu_payload_bytes": (_u64, [_u64, _pdesc]),
    "hcmx_gpu_codec_analyze": (_i, [_vp, _vp, _pu64, _u64, _vp, _vp]),
    "hcmx_gpu_codec_pack": (_i, [_vp, _vp, _pu64, _vp, _vp, _u64, _vp, _vp]),
    "hcmx_gpu_codec_unpack": (_i, [_vp, _vp, _pu64, _vp, _vp, _u64, _vp, _vp]),
    "hcmx_gpu_codec_compress": (_i, [_vp, _vp, _pu64, _u64, _d, _i, _vp, _u64, _vp, _pu64,
                                     _pu64, _vp]),
    "hcmx_gpu_codec_compress_device": (_i, [_vp, _vp, _vp, _u64, _u64, _d, _i, _vp, _vp, _vp, _vp, _vp]),
    "hcmx_gpu_codec_compress_fixup": (_i, [_vp, _vp, _pu64, _u64, _d, _i, _pu64, _vp, _vp, _vp, _pu64, _vp]),
    "hcmx_gpu_codec_timing": (_i, [_i, C.POINTER(_d), _pu64, C.POINTER(_d), _pu64]),
    "hcmx_gpu_compress": (_i, [_vp, _u64, _d, _i, _pdesc, _vp, _u64, _pu64]),
    "hcmx_gpu_compress_block": (_i, [_vp, _u64, _pdesc, _vp, _u64, _pu64]),
    "hcmx_gpu_decompress_into": (_i, [_pdesc, _u64, _vp, _u64, _vp]),
    "hcmx_gpu_serialize": (_u64, [_pdesc, _u64, _vp, _u64, _vp]),
    "hcmx_gpu_deserialize": (_i, [_vp, _u64, _pu64, _pdesc, _pu64, _pu64, _pu64]),
    "hcmx_gpu_aplr_compress": (_i, [_u64, _pu64, _pu64, _pu64, _vp, _pu64, _vp, _pu64, _vp,
                                    _pu64, _pu64, _d, _i, _vp, _u64, _vp, _pu64, _pu64, _vp]),
    "hcmx_gpu_hmat_create": (_i, [C.POINTER(hcmx_hmat_desc), C.POINTER(_vp)]),
    "hcmx_gpu_hmat_destroy": (_i, [_vp]),
    "hcmx_gpu_hmat_memory": (_i, [_vp, C.POINTER(hcmx_memory_report)]),
    "hcmx_gpu_hmat_matvec": (_i, [_vp, _d, _vp, _d, _vp, _i]),
    "hcmx_gpu_hmat_matmat": (_i, [_vp, _d, _vp, _u64, _u64, _d, _vp, _u64, _i]),
    "hcmx_gpu_hmat_matvec_device": (_i, [_vp, _d, _vp, _d, _vp, _vp]),
    "hcmx_gpu_hmat_matmat4_device": (_i, [_vp, _d, _vp, _d, _vp, _vp]),
    "hcmx_gpu_hmat_matmat_block_device": (_i, [_vp, _d, _vp, _d, _vp, _vp]),
    "hcmx_gpu_hmat_nrhs_block": (_i, [_vp]),
    "hcmx_gpu_hmat_transposed": (_i, [_vp, C.POINTER(_vp)]),
    "hcmx_gpu_hmat_export_buffer": (_i, [_vp, _u64, _vp, _u64, _pu64]),
    "hcmx_gpu_hmat_last_launches": (_i, [_vp]),
    "hcmx_gpu_hmat_timing": (_i, [_vp, _i, C.POINTER(_d), C.POINTER(_d), _pu64]),
    "hcmx_gpu_compress_in_place": (_i, [C.POINTER(hcmx_assembled), _d, _i, _i, _i, C.POINTER(_vp),
                                        C.POINTER(hcmx_memory_report), _vp]),
    "hcmx_gpu_flat_desc": (_i, [_vp, C.POINTER(hcmx_hmat_desc)]),
    "hcmx_gpu_flat_destroy": (_i, [_vp]),
    "hcmx_gpu_flat_copy_blob": (_i, [_vp, _vp, _vp]),
    "hcmx_gpu_partition_rows": (_i, [C.POINTER(hcmx_hmat_desc), _i, _pu64]),
    "hcmx_gpu_nccl_unique_id": (_i, [_vp]),
    "hcmx_gpu_nccl_comm_init": (_i, [_i, _vp, _i, C.POINTER(_vp)]),
    "hcmx_gpu_nccl_comm_destroy": (_i, [_vp]),
    "hcmx_gpu_hmat_create_partitioned": (_i, [C.POINTER(hcmx_hmat_desc), _vp, C.POINTER(_vp)]),
    "hcmx_gpu_hmat_dist_destroy": (_i, [_vp]),
    "hcmx_gpu_hmat_dist_rows": (_i, [_vp, _pu64, _pu64, C.POINTER(_i), C.POINTER(_i)]),
    "hcmx_gpu_hmat_dist_cuts": (_i, [_vp, _pu64]),
    "hcmx_gpu_hmat_dist_local": (_i, [_vp, C.POINTER(_vp)]),
    "hcmx_gpu_hmat_dist_matvec_device": (_i, [_vp, _d, _vp, _d, _vp, _vp]),
    "hcmx_gpu_hmat_dist_matvec": (_i, [_vp, _d, _vp, _d, _vp]),
}

_lib = None


def lib() -> C.CDLL:
    """Load libhcmx_gpu.so; raise if it was not built (no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIBPATH):
            raise ImportError(f"{LIBPATH} missing: run `python -m paper_2308_10960_b200.build` "
                              "(there is no CPU fallback)")
        L = C.CDLL(LIBPATH)
        for name, (res, args) in PROTOTYPES.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def check(status: int, what: str = "hcmx_gpu") -> None:
    if status == HCMX_OK:
        return
    msg = lib().hcmx_gpu_last_error().decode(errors="replace")
    if status == HCMX_INVALID_ARGUMENT:
        raise ValueError(f"{what}: {msg}")
    if status == HCMX_CORRUPT_BUFFER:
        raise CorruptBufferError(f"{what}: {msg}")
    if status == HCMX_OUT_OF_MEMORY:
        raise MemoryError(f"{what}: {msg}")
    if status == HCMX_NCCL_ERROR:
        raise NcclError(f"{what}: {msg}")
    raise CudaError(f"{what}: {msg} (status {status})")


def ptr(a) -> int:
    """device or host address of a torch tensor / numpy array (None -> 0)"""
    if a is None:
        return 0
    if isinstance(a, np.ndarray):
        return a.ctypes.data
    return a.data_ptr()


def u64p(a: np.ndarray):
    return a.ctypes.data_as(_pu64)


_initialised = set()


def ensure_device(device: int = 0) -> None:
    if device not in _initialised:
        check(lib().hcmx_gpu_init(device), "hcmx_gpu_init")
        _initialised.add(device)
