"""One build of a BASELINE config, then (profiling aid): setup stage times, the
phase times of the product, and the per-rank product times of every N-way
block-row partition (hcmx_gpu_partition_rows) emulated on this GPU, with the
efficiency T_1 / (N * max_r T_r).

    HCMX_BUILD_STATS=1 python tools/prof_config.py 4 [N ...]
"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2308_10960_b200.distributed import partition_rows  # noqa: E402
from paper_2308_10960_b200.hmatrix import HMatrix, build_config  # noqa: E402


def timed(H, x, y, reps=20):
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
    cfg = sys.argv[1]
    Ns = [int(a) for a in sys.argv[2:]] or [2, 4, 8]
    t = time.time()
    flat, info = build_config(cfg)
    print(f"build_config {time.time() - t:.1f}s: leaves {info['leaves']}, mean rank {info['mean_rank']:.2f}", flush=True)
    t = time.time()
    H = HMatrix(flat)
    print(f"hmat_create {time.time() - t:.1f}s", flush=True)
    n = flat.n_rows
    x = torch.as_tensor(np.random.default_rng(0).uniform(-1, 1, n)).cuda()
    y = torch.zeros(n, dtype=torch.float64, device="cuda")
    rep = H.memory()
    t1 = timed(H, x, y)
    H.timing(1)
    for _ in range(20):
        H.matvec_device(1.0, x, 0.0, y)
    ma, mb, calls = H.timing(0)
    print(f"N=1: product {t1:.4f} ms -> {rep.algorithmic_bytes / t1 / 1e6:.1f} GB/s; phase A {ma / calls:.4f} ms, "
          f"phase B {mb / calls:.4f} ms (algo {rep.algorithmic_bytes / 1e9:.3f} GB, arena "
          f"{rep.device_arena_bytes / 1e9:.3f} GB, stages A {rep.stages_a} B {rep.stages_b})", flush=True)
    H.close()
    for N in Ns:
        times, detail = [], []
        for rr in partition_rows(flat, N):
            Hr = HMatrix(flat, row_range=rr)
            times.append(timed(Hr, x, y))
            Hr.timing(1)
            for _ in range(10):
                Hr.matvec_device(1.0, x, 0.0, y)
            ma, mb, calls = Hr.timing(0)
            r = Hr.memory()
            detail.append(f"[{rr[0]},{rr[1]}) A {ma / calls:.3f} B {mb / calls:.3f} ms, {r.algorithmic_bytes / 1e9:.2f} GB, "
                          f"stages {r.stages_a}/{r.stages_b}")
            Hr.close()
        for d in detail:
            print("     ", d)
        print(f"N={N}: per-rank ms {' '.join(f'{v:.4f}' for v in times)} | max {max(times):.4f}, "
              f"T1/(N*Tmax) = {t1 / (N * max(times)):.3f}", flush=True)


if __name__ == "__main__":
    main()
