"""Block-row partitioning of the compressed H-matrix over the GPUs of one box
(SURVEY 8e): every leaf writes rows of exactly one row range; each rank keeps
the leaves of its rows (a lowrank leaf crossing a cut is kept by both ranks,
each doing phase A for it and phase B for its own rows), x is replicated, and
after every product the disjoint y slices are all-gathered (NCCL over NVLink on
GPUs; gloo in the CPU tests).  One process per GPU, torch.distributed plumbing.
"""
from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist


def leaf_bytes(flat) -> np.ndarray:
    """compressed payload bytes per leaf"""
    out = np.zeros(flat.nleaves if hasattr(flat, "nleaves") else flat.row0.size)
    for l in range(out.size):
        b0 = int(flat.buf0[l])
        if flat.kind[l] == 0:
            out[l] = float(flat.plen[b0])
        else:
            k = int(flat.rank[l])
            out[l] = float(flat.plen[b0: b0 + 2 * k].sum()) + 8 * k
    return out


def partition_rows(flat, world: int, align: int = 64) -> list[tuple[int, int]]:
    """contiguous row ranges, cut on multiples of `align` (row-leaf clusters for a
    power-of-two n), balanced by the prefix sum of compressed bytes per row"""
    n = int(flat.n_rows)
    if world <= 1:
        return [(0, n)]
    rows = (flat.row1 - flat.row0).astype(np.float64)
    lb = leaf_bytes(flat)
    dens = np.zeros(n + 1)
    np.add.at(dens, flat.row0, lb / rows)
    np.add.at(dens, flat.row1, -lb / rows)
    pref = np.concatenate([[0.0], np.cumsum(np.cumsum(dens)[:-1])])
    cuts = [0]
    for r in range(1, world):
        c = int(np.searchsorted(pref, pref[-1] * r / world))
        c = int(round(c / align)) * align
        c = min(max(c, cuts[-1] + align), n - (world - r) * align)
        cuts.append(c)
    cuts.append(n)
    return list(zip(cuts[:-1], cuts[1:]))


class DistributedHMatrix:
    """y := alpha A x over P ranks.  `local` computes this rank's y slice into a
    full-length vector (the GPU HMatrix with a row_range, or any callable in
    tests); the exchange is one all_gather_into_tensor of padded slices."""

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
