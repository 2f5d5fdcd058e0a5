"""BASELINE config 5 at size (profiling aid): Helmholtz exp(i kappa r)/(4 pi r),
kappa = 16, n = 262144 sphere points, eps 1e-6, complex FP64, 16 right-hand
sides through ComplexHMatrix.matmat_device (one complex arena: every real /
imaginary stream decoded once per product of two complex columns, the complex
combination on the device).  Prints setup times, ms per 16-RHS product,
FP64 TFLOP/s against the measured DFMA peak, and the parity of two columns
against the CPU oracle (test infrastructure, not timed).

    python tools/prof_c5.py [n]
"""
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
from paper_2308_10960_b200.hmatrix import ComplexHMatrix, build_config_complex  # noqa: E402


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 262144
    block = int(sys.argv[2]) if len(sys.argv) > 2 else 4  # real slots per device product (4 or 8)
    r = 16
    t = time.time()
    fr, fi, info = build_config_complex("5", n=n)
    setup = time.time() - t
    t = time.time()
    H = ComplexHMatrix(fr, fi, nrhs_block=block)
    create = time.time() - t
    rep = H.memory()
    rng = np.random.default_rng(5)
    X = rng.uniform(-1, 1, (n, r)) + 1j * rng.uniform(-1, 1, (n, r))
    Xd = torch.as_tensor(X).cuda()
    Y = torch.empty(n, r, dtype=torch.complex128, device="cuda")
    for _ in range(2):
        H.matmat_device(Xd, Y)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 5
    e0.record()
    for _ in range(reps):
        H.matmat_device(Xd, Y)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    # FP64 work executed: every stored real entry of the complex arena takes 2
    # flops per real right-hand-side slot, 4 slots per product of two complex
    # columns, r / 2 products
    entries = rep.uncompressed_equivalent / 8
    flops = 2.0 * entries * 4 * (r // 2)
    tf = flops / (ms / 1e3) / 1e12
    pk = os.path.join(ROOT, "profiles", "r1_fp64_peak.json")
    peak = json.load(open(pk)).get("fp64_fma_tflops") if os.path.exists(pk) else None
    # bytes streamed per 16-RHS product: the arena's algorithmic bytes per block product x 2 r / block
    gbytes = rep.algorithmic_bytes * (2 * r // block) / 1e9
    from oracle import Oracle
    o = Oracle()
    frh, fih = fr.host(), fi.host()
    Yh = Y.cpu().numpy()
    errs = []
    for j in (0, r - 1):
        yr = o.hmat_matvec(frh, 1.0, X[:, j].real, 0.0, np.zeros(n), threads=os.cpu_count()) - \
            o.hmat_matvec(fih, 1.0, X[:, j].imag, 0.0, np.zeros(n), threads=os.cpu_count())
        yi = o.hmat_matvec(frh, 1.0, X[:, j].imag, 0.0, np.zeros(n), threads=os.cpu_count()) + \
            o.hmat_matvec(fih, 1.0, X[:, j].real, 0.0, np.zeros(n), threads=os.cpu_count())
        ref = yr + 1j * yi
        errs.append(float(np.linalg.norm(Yh[:, j] - ref) / np.linalg.norm(ref)))
    out = {"config": "5", "n": n, "nrhs": r, "nrhs_block": block, "leaves": info["leaves"], "setup_s": round(setup, 1),
           "create_s": round(create, 1), "compressed_bytes": int(rep.algorithmic_bytes), "arena_bytes": int(rep.device_arena_bytes),
           "ms_per_16rhs_product": round(ms, 3), "fp64_tflops": round(tf, 2), "fp64_peak_tflops": peak,
           "fp64_frac": round(tf / peak, 3) if peak else None, "streamed_gb_per_product": round(gbytes, 2),
           "stream_gbs": round(gbytes / (ms / 1e3), 1), "parity_rel_err": errs}
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
