"""Timing of the setup-time building blocks on the GPU box (profiling aid):
batched kernel-block evaluation, batched QR, GEMM, host / device SVD."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2308_10960_b200.assemble import _cpu_svd  # noqa: E402


def t(f, *a, reps=2):
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(reps):
        t0 = time.time()
        r = f(*a)
        torch.cuda.synchronize()
        best = min(best, time.time() - t0)
    return best, r


def main():
    dev = "cuda"
    for (B, m, p) in ((2000, 128, 64), (2000, 128, 128), (320, 1024, 96), (40, 8192, 96)):
        A = torch.randn(B, m, m, dtype=torch.float64, device=dev)
        Om = torch.randn(B, m, p, dtype=torch.float64, device=dev)
        tg, Y = t(torch.bmm, A, Om)
        tq, (Q, R) = t(torch.linalg.qr, Y)
        th, _ = t(torch.geqrf, Y)
        Rs = R[:, :p, :p].contiguous()
        tsc, _ = t(_cpu_svd, Rs, reps=1)
        tsg, _ = t(torch.linalg.svd, Rs, reps=1)
        te, _ = t(torch.linalg.eigh, Rs @ Rs.mT, reps=1)
        print(f"B={B} m={m} p={p}: bmm {tg*1e3:.1f} ms, qr {tq*1e3:.1f} ms, geqrf {th*1e3:.1f} ms, "
              f"cpu_svd(pxp) {tsc*1e3:.1f} ms, gpu svd(pxp) {tsg*1e3:.1f} ms, gpu eigh(pxp) {te*1e3:.1f} ms",
              flush=True)
        del A, Om, Y, Q, R


if __name__ == "__main__":
    main()
