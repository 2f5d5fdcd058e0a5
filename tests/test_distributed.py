"""Multi-rank block-row path on the CPU: world_size 2 over gloo.  The local
product is the CPU oracle restricted to the rank's leaves (the GPU kernel's
row-range handle is covered by test_hmat_gpu.test_row_partitions_compose);
this checks the partition, the ownership rule and the all-gather exchange."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _restrict_rows(f, a, b):
    """leaves writing rows in [a, b) (a crossing lowrank leaf is kept by both ranks)"""
    from dataclasses import replace
    sel = (f.row0 < b) & (f.row1 > a)
    return replace(f, row0=f.row0[sel], row1=f.row1[sel], col0=f.col0[sel], col1=f.col1[sel],
                   kind=f.kind[sel], rank=f.rank[sel], buf0=f.buf0[sel], sig0=f.sig0[sel])


def _worker(rank, world, port, parts, n, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import sys
    sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "oracle"))
    sys.path.insert(0, os.path.dirname(__file__))
    from cpu_hmatrix import Flat
    from oracle import Oracle
    from paper_2308_10960_b200.distributed import DistributedHMatrix
    z = np.load(os.path.join(os.path.dirname(__file__), "golden", "hmat_golden.npz"))
    f = Flat.from_npz(z)
    a, b = parts[rank]
    mine = _restrict_rows(f, a, b)
    o = Oracle()

    def local(alpha, x, y):
        full = o.hmat_matvec(mine, alpha, x.numpy(), 0.0, np.zeros(n))
        y[a:b] = torch.from_numpy(full[a:b])   # rows outside the slice are not ours

    D = DistributedHMatrix(parts, rank, local, "cpu")
    x = torch.from_numpy(z["x"])
    y = torch.full((n,), float("nan"), dtype=torch.float64)
    D.matvec(1.0, x, y)
    # a second product on the gathered vector (the repeated-product pattern)
    y2 = torch.zeros(n, dtype=torch.float64)
    D.matvec(1.0, y.clone(), y2)
    q.put((rank, y.numpy().copy(), y2.numpy().copy()))
    dist.barrier()
    dist.destroy_process_group()


def test_partition_balances_bytes():
    """the library partitioner (hcmx_gpu_partition_rows, host only): contiguous
    64-row-aligned ranges covering the rows, and its largest per-rank cost is the
    optimum over every 64-aligned choice of cuts (brute force, world 2 and 3)"""
    import itertools
    import sys
    sys.path.insert(0, os.path.dirname(__file__))
    from cpu_hmatrix import Flat
    from paper_2308_10960_b200.distributed import leaf_bytes, partition_rows, rank_cost
    z = np.load(os.path.join(os.path.dirname(__file__), "golden", "hmat_golden.npz"))
    f = Flat.from_npz(z)
    n = f.n_rows
    for world in (1, 2, 3, 4):
        parts = partition_rows(f, world)
        assert len(parts) == world
        assert parts[0][0] == 0 and parts[-1][1] == n
        assert all(p[1] == q[0] for p, q in zip(parts[:-1], parts[1:]))
        assert all(b > a and a % 64 == 0 for a, b in parts)
        got = max(rank_cost(f, a, b) for a, b in parts)
        best = min(max(rank_cost(f, a, b) for a, b in zip((0,) + c, c + (n,)))
                   for c in itertools.combinations(range(64, n, 64), world - 1)) if world <= 3 else got
        assert got <= best * (1 + 1e-9), (world, got, best)
    lb = leaf_bytes(f)
    assert lb.sum() > 0
    # more ranks than 64-row units: trailing ranks get empty ranges
    parts = partition_rows(f, n // 64 + 2)
    assert parts[-1] == (n, n) and sum(b - a for a, b in parts) == n


def test_gloo_world2_block_rows():
    import sys
    sys.path.insert(0, os.path.dirname(__file__))
    from cpu_hmatrix import Flat
    from oracle import Oracle
    z = np.load(os.path.join(os.path.dirname(__file__), "golden", "hmat_golden.npz"))
    f = Flat.from_npz(z)
    n = f.n_rows
    from paper_2308_10960_b200.distributed import partition_rows
    parts = partition_rows(f, 2)   # the bench's partitioner
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, parts, n, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(2)]
    for p in procs:
        p.join(60)
        assert p.exitcode == 0
    o = Oracle()
    ref = o.hmat_matvec(f, 1.0, z["x"], 0.0, np.zeros(n))
    ref2 = o.hmat_matvec(f, 1.0, ref, 0.0, np.zeros(n))
    for rank, y, y2 in res:
        assert np.linalg.norm(y - ref) <= 1e-13 * np.linalg.norm(ref)
        assert np.linalg.norm(y2 - ref2) <= 1e-12 * np.linalg.norm(ref2)
