"""Setup building blocks, second probe (profiling aid): host SVD with one BLAS
thread per worker, GPU QR variants for the randomized range finder."""
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


def cholqr3(Y):
    """shifted Cholesky QR, three passes (orthonormal Q for cond(Y) up to ~1/u)"""
    m, p = Y.shape[-2:]
    G = Y.mT @ Y
    nrm = torch.linalg.matrix_norm(Y, ord="fro")
    s = 11 * (m * p + p * (p + 1)) * 2.2e-16 * nrm ** 2
    G = G + s[:, None, None] * torch.eye(p, dtype=Y.dtype, device=Y.device)
    R = torch.linalg.cholesky(G, upper=True)
    Q = torch.linalg.solve_triangular(R, Y, upper=True, left=False)
    for _ in range(2):
        R2 = torch.linalg.cholesky(Q.mT @ Q, upper=True)
        Q = torch.linalg.solve_triangular(R2, Q, upper=True, left=False)
        R = R2 @ R
    return Q, R


def hh(Y):
    a, tau = torch.geqrf(Y)
    return torch.linalg.householder_product(a, tau)


def main():
    dev = "cuda"
    print("cpus", os.cpu_count(), flush=True)
    for (B, m) in ((2000, 64), (2000, 96), (2000, 128)):
        A = torch.randn(B, m, m, dtype=torch.float64)
        ts, _ = t(_cpu_svd, A, reps=1)
        print(f"cpu_svd {B} x {m}x{m}: {ts*1e3:.1f} ms", flush=True)
    for (B, n) in ((20000, 16), (20000, 32), (2000, 48), (2000, 64)):
        A = torch.randn(B, n, n, dtype=torch.float64, device=dev)
        tg, _ = t(lambda M: torch.linalg.svd(M, full_matrices=False), A)
        print(f"gpu svd {B} x {n}x{n}: {tg*1e3:.1f} ms", flush=True)
    for (B, m, p) in ((2000, 128, 32), (2000, 128, 64), (320, 1024, 32), (320, 1024, 96), (40, 8192, 32), (40, 8192, 96)):
        # low-rank-ish test matrices: Y = A Omega with fast decaying spectrum
        U = torch.linalg.qr(torch.randn(B, m, p, dtype=torch.float64, device=dev))[0]
        sv = 10.0 ** (-torch.arange(p, dtype=torch.float64, device=dev) * 16.0 / p)
        Vt = torch.linalg.qr(torch.randn(B, p, p, dtype=torch.float64, device=dev))[0]
        Y = (U * sv) @ Vt
        tq, (Q, _) = t(torch.linalg.qr, Y)
        th, Qh = t(hh, Y)
        tc, (Qc, _) = t(cholqr3, Y)
        err = lambda Q: float((Q.mT @ Q - torch.eye(p, dtype=Q.dtype, device=dev)).abs().max())
        cap = lambda Q: float(((Y - Q @ (Q.mT @ Y)).norm() / Y.norm()))
        print(f"B={B} m={m} p={p}: qr {tq*1e3:.1f} ms (orth {err(Q):.1e} res {cap(Q):.1e}), "
              f"geqrf+orgqr {th*1e3:.1f} ms (orth {err(Qh):.1e}), cholqr3 {tc*1e3:.1f} ms "
              f"(orth {err(Qc):.1e} res {cap(Qc):.1e})", flush=True)


if __name__ == "__main__":
    main()
