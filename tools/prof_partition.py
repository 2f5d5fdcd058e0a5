"""Per-rank product time of a block-row partition, emulated on one GPU (profiling
aid): the handle of rank r of N (distributed.partition_rows) timed alone, i.e.
the device time each GPU of an N-GPU run spends per product (without the
all-gather)."""
import os
import pickle
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2308_10960_b200.hmatrix import HMatrix  # noqa: E402
import bench  # noqa: E402

flat = pickle.load(open(sys.argv[1], "rb"))
flat.blob = torch.as_tensor(flat.blob).cuda()
n = flat.n_rows
x = torch.as_tensor(np.random.default_rng(0).uniform(-1, 1, n)).cuda()
y = torch.zeros(n, dtype=torch.float64, device="cuda")
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for N in (1, 2, 4, 8):
    parts = bench.partition_rows(flat, N)
    worst = 0.0
    for r in (0, N - 1):
        H = HMatrix(flat, row_range=None if N == 1 else parts[r])
        for _ in range(3):
            H.matvec_device(1.0, x, 0.0, y)
        e0.record()
        for _ in range(30):
            H.matvec_device(1.0, x, 0.0, y)
        e1.record()
        torch.cuda.synchronize()
        worst = max(worst, e0.elapsed_time(e1) / 30)
        H.timing(1)
        for _ in range(30):
            H.matvec_device(1.0, x, 0.0, y)
        torch.cuda.synchronize()
        ma, mb, calls = H.timing(0)
        print(f"   N={N} rank {r}: phase A {ma / calls:.4f} ms, phase B {mb / calls:.4f} ms (events, no PDL)")
        H.close()
    print(f"N={N}: per-rank product {worst:.4f} ms (max of first/last rank), ideal {0 if N == 1 else 0:.0f}", flush=True)
