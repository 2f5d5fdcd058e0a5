"""Block-row partitioning of the compressed H-matrix over the GPUs of one box
(SURVEY 8e), over the C-ABI (include/hcmx_gpu.h, csrc/dist.cpp).

Every leaf writes rows of one row range; each rank keeps the leaves of its rows
(a lowrank leaf crossing a cut is kept by both ranks, each doing phase A for it
and phase B for its own rows), x is replicated, and after every product the
disjoint y slices are exchanged so each rank holds all of y for the next one.
On GPUs the exchange is one NCCL group of in-place broadcasts inside the
library (hcmx_gpu_hmat_dist_matvec_device); the CPU tests run the same
partition and ownership rule with gloo (DistributedHMatrix).  One process per
GPU, torch.distributed for the rendezvous only.

There is ONE partitioner, hcmx_gpu_partition_rows (C++): the bench, the
partitioned handle and the gloo tests all use it.  The reference has no
parallel code; its hooks are the unused `threads` knobs (hmatrix.hpp:83,119)
and SPEC.md:489 (disjoint leaf blocks, deterministic merge).
"""
from __future__ import annotations

import ctypes as C

import numpy as np
import torch
import torch.distributed as dist

from . import _lib
from ._lib import check, lib


def leaf_bytes(flat) -> np.ndarray:
    """compressed payload bytes per leaf"""
    out = np.zeros(flat.row0.size)
    for l in range(out.size):
        b0 = int(flat.buf0[l])
        if flat.kind[l] == 0:
            out[l] = float(flat.plen[b0])
        else:
            k = int(flat.rank[l])
            nb = 2 * k if flat.kind[l] == 1 else (2 if k else 0)
            out[l] = float(flat.plen[b0: b0 + nb].sum()) + 8 * k
    return out


def _product_flat(flat):
    """the checkers' Flat (tests) -> FlatHMatrix; FlatHMatrix unchanged"""
    return flat if hasattr(flat, "desc") else flat.to_product()


def partition_cuts(flat, world: int) -> np.ndarray:
    """world + 1 row cuts from the library's partitioner (host only)"""
    from .hmatrix import flat_desc
    f = _product_flat(flat)
    d, keep = flat_desc(f)
    cuts = np.zeros(world + 1, np.uint64)
    check(lib().hcmx_gpu_partition_rows(C.byref(d), int(world), _lib.u64p(cuts)), "partition_rows")
    del keep
    return cuts.astype(np.int64)


def partition_rows(flat, world: int) -> list[tuple[int, int]]:
    """contiguous row ranges [(a, b)] per rank (multiples of 64 rows), balanced
    by compressed bytes with duplicated X factors charged to both ranks"""
    c = partition_cuts(flat, world)
    return [(int(a), int(b)) for a, b in zip(c[:-1], c[1:])]


def rank_cost(flat, a: int, b: int) -> float:
    """the partitioner's cost of rows [a, b): phase-B bytes landing there plus the
    phase-A bytes of every lowrank leaf overlapping it (for tests / reports)"""
    f = _product_flat(flat)
    tot = 0.0
    for l in range(f.row0.size):
        r0, r1 = int(f.row0[l]), int(f.row1[l])
        ov = min(r1, b) - max(r0, a)
        if ov <= 0:
            continue
        b0, k = int(f.buf0[l]), int(f.rank[l])
        pl = lambda i: float(f.plen[i]) + 20.0
        if f.kind[l] == 0:
            w, x = pl(b0), 0.0
        elif f.kind[l] == 1:
            w = sum(pl(b0 + i) for i in range(k))
            x = sum(pl(b0 + k + i) + 8.0 for i in range(k))
        else:
            w, x = (pl(b0), pl(b0 + 1)) if k else (0.0, 0.0)
        tot += w * ov / (r1 - r0) + x
    return tot


def nccl_comm(group=None):
    """an NCCL communicator over the ranks of a torch.distributed group (the
    unique id travels through torch.distributed); returns (comm, world, rank)"""
    world, rank = dist.get_world_size(group), dist.get_rank(group)
    uid = (C.c_uint8 * 128)()
    if rank == 0:
        check(lib().hcmx_gpu_nccl_unique_id(uid), "nccl_unique_id")
    obj = [bytes(uid)]
    dist.broadcast_object_list(obj, src=0, group=group)
    C.memmove(uid, obj[0], 128)
    comm = C.c_void_p()
    check(lib().hcmx_gpu_nccl_comm_init(world, uid, rank, C.byref(comm)), "nccl_comm_init")
    return comm, world, rank


class PartitionedHMatrix:
    """This rank's rows of a compressed H-matrix (hcmx_gpu_hmat_create_partitioned):
    matvec_device leaves the whole y on every rank (local product + NCCL
    exchange on the given stream)."""

    def __init__(self, flat, comm=None):
        from .hmatrix import flat_desc
        _lib.ensure_device()
        self.n_rows, self.n_cols = int(flat.n_rows), int(flat.n_cols)
        d, keep = flat_desc(flat)
        h = C.c_void_p()
        check(lib().hcmx_gpu_hmat_create_partitioned(C.byref(d), comm, C.byref(h)), "create_partitioned")
        del keep
        self._h = h
        rb, re_ = C.c_uint64(), C.c_uint64()
        rk, ws = C.c_int(), C.c_int()
        check(lib().hcmx_gpu_hmat_dist_rows(h, C.byref(rb), C.byref(re_), C.byref(rk), C.byref(ws)), "dist_rows")
        self.row_range, self.rank, self.world = (rb.value, re_.value), rk.value, ws.value
        cuts = np.zeros(self.world + 1, np.uint64)
        check(lib().hcmx_gpu_hmat_dist_cuts(h, _lib.u64p(cuts)), "dist_cuts")
        self.cuts = cuts.astype(np.int64)
        loc = C.c_void_p()
        check(lib().hcmx_gpu_hmat_dist_local(h, C.byref(loc)), "dist_local")
        self.local = loc  # the rank-local hcmx_hmat (None for an empty range)

    def matvec_device(self, alpha: float, x: torch.Tensor, beta: float, y: torch.Tensor, stream=None):
        if x.numel() != self.n_cols or y.numel() != self.n_rows:
            raise ValueError("matvec: dimension mismatch")
        s = stream if stream is not None else torch.cuda.current_stream().cuda_stream
        check(lib().hcmx_gpu_hmat_dist_matvec_device(self._h, float(alpha), x.data_ptr(), float(beta),
                                                      y.data_ptr(), s), "dist_matvec")
        return y

    def matvec(self, alpha: float, x, beta: float, y):
        """host vectors (the reference-facing call): x in, the whole y out"""
        xa = np.ascontiguousarray(x, dtype=np.float64)
        if xa.size != self.n_cols or y.size != self.n_rows:
            raise ValueError("matvec: dimension mismatch")
        check(lib().hcmx_gpu_hmat_dist_matvec(self._h, float(alpha), _lib.ptr(xa), float(beta), _lib.ptr(y)),
              "dist_matvec")
        return y

    def timing(self, enable: int):
        a, b, n = C.c_double(), C.c_double(), C.c_uint64()
        if self.local:
            check(lib().hcmx_gpu_hmat_timing(self.local, int(enable), C.byref(a), C.byref(b), C.byref(n)),
                  "timing")
        return a.value, b.value, n.value

    def launches(self) -> int:
        return lib().hcmx_gpu_hmat_last_launches(self.local) if self.local else 0

    def memory(self):
        r = _lib.hcmx_memory_report()
        if self.local:
            check(lib().hcmx_gpu_hmat_memory(self.local, C.byref(r)), "hmat_memory")
        return r

    def close(self):
        if getattr(self, "_h", None):
            check(lib().hcmx_gpu_hmat_dist_destroy(self._h), "dist_destroy")
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class DistributedHMatrix:
    """The same ownership rule and exchange with a caller-supplied local product
    and torch.distributed (gloo in the CPU tests): `local` computes this rank's
    y slice into a full-length vector; the exchange is one all_gather of padded
    slices."""

    def __init__(self, parts, rank, local, device, group=None):
        self.parts, self.rank, self.local = parts, rank, local
        self.group = group
        self.maxlen = max(b - a for a, b in parts)
        world = len(parts)
        self.slab = torch.zeros(self.maxlen, dtype=torch.float64, device=device)
        self.gathered = torch.zeros(self.maxlen * world, dtype=torch.float64, device=device)
        self.idx = torch.cat([torch.arange(a, b, device=device) - a + r * self.maxlen
                              for r, (a, b) in enumerate(parts)])

    def matvec(self, alpha: float, x: torch.Tensor, y: torch.Tensor) -> torch.Tensor:
        a, b = self.parts[self.rank]
        self.local(alpha, x, y)               # writes y[a:b]
        self.slab[: b - a].copy_(y[a:b])
        if len(self.parts) > 1:
            dist.all_gather_into_tensor(self.gathered, self.slab, group=self.group)
            y.copy_(self.gathered[self.idx])   # every rank now holds all of y
        return y
