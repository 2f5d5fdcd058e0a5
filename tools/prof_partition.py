"""Per-rank product time of a block-row partition, emulated on one GPU (profiling
aid): every rank's handle of an N-way partition (hcmx_gpu_partition_rows, the
partitioner the bench and the partitioned C-ABI use) timed alone -- the device
time each GPU of an N-GPU run spends per product, without the y exchange --
and the efficiency T_1 / (N * max_r T_r).

    python tools/prof_partition.py CONFIG [N ...]        (builds the config)
    python tools/prof_partition.py --cache FILE.pkl [N ...]
"""
import os
import pickle
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2308_10960_b200.distributed import partition_rows  # noqa: E402
from paper_2308_10960_b200.hmatrix import HMatrix, build_config  # noqa: E402


def product_ms(H, x, y, reps=20):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for _ in range(3):
        H.matvec_device(1.0, x, 0.0, y)
    e0.record()
    for _ in range(reps):
        H.matvec_device(1.0, x, 0.0, y)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def main():
    args = sys.argv[1:]
    if args[0] == "--cache":
        flat = pickle.load(open(args[1], "rb"))
        flat.blob = torch.as_tensor(flat.blob).cuda()
        Ns = [int(a) for a in args[2:]] or [1, 2, 4, 8]
    else:
        flat, _ = build_config(args[0])
        Ns = [int(a) for a in args[1:]] or [1, 2, 4, 8]
    n = flat.n_rows
    x = torch.as_tensor(np.random.default_rng(0).uniform(-1, 1, n)).cuda()
    y = torch.zeros(n, dtype=torch.float64, device="cuda")
    t1 = None
    for N in Ns:
        parts = partition_rows(flat, N)
        times = []
        for r, rr in enumerate(parts):
            H = HMatrix(flat, row_range=None if N == 1 else rr)
            times.append(product_ms(H, x, y))
            H.close()
        worst = max(times)
        if N == 1:
            t1 = worst
        eff = t1 / (N * worst) if t1 else float("nan")
        print(f"N={N}: per-rank ms {' '.join(f'{t:.4f}' for t in times)} | max {worst:.4f} ms, "
              f"T1/(N*Tmax) = {eff:.3f}", flush=True)


if __name__ == "__main__":
    main()
