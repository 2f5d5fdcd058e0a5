"""Profiling driver (not part of the product): build a config, time setup
stages, run the H-matvec, print per-phase device times.  With --cache the
compressed matrix is kept in /tmp between runs of the same gpurun call (so an
ncu pass does not redo the setup)."""
import argparse
import os
import pickle
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2308_10960_b200 import assemble, problems, tree  # noqa: E402
from paper_2308_10960_b200.hmatrix import HMatrix, compress_in_place  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="3")
    ap.add_argument("--n", type=int, default=None)
    ap.add_argument("--scheme", default="afl")
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--cache", default=None)
    ap.add_argument("--rhs4", action="store_true", help="also time the 4-right-hand-side arena")
    ap.add_argument("--yref", default=None, help="compare y with this saved product (saved if missing)")
    a = ap.parse_args()
    c = problems.config(a.config)
    if a.n:
        c["n"] = a.n
    T = {}
    if a.cache and os.path.exists(a.cache):
        t = time.time()
        flat = pickle.load(open(a.cache, "rb"))
        flat.blob = torch.as_tensor(flat.blob).cuda()
        T["load_cache"] = time.time() - t
    else:
        t = time.time()
        pts = problems.make_points(c["geometry"], c["n"], 1)
        ct = tree.build_cluster_tree(pts, c["leaf"])
        lv = tree.build_block_tree(ct, ct, c["eta"])
        T["tree"] = time.time() - t
        t = time.time()
        A = assemble.assemble(pts[ct.i2e], lv, problems.make_kernel(c["kernel"]), c["eps"])
        torch.cuda.synchronize()
        T["assemble"] = time.time() - t
        t = time.time()
        flat = compress_in_place(A, c["eps"], f"{a.scheme}-aplr")
        torch.cuda.synchronize()
        T["compress_in_place"] = time.time() - t
        if a.cache:
            h = flat.host()
            pickle.dump(h, open(a.cache, "wb"))
        del A
    t = time.time()
    H = HMatrix(flat, nrhs_block=4 if a.rhs4 else 0)
    T["hmat_create"] = time.time() - t
    n = flat.n_rows
    x = torch.as_tensor(np.random.default_rng(0).uniform(-1, 1, n)).cuda()
    y = torch.zeros(n, dtype=torch.float64, device="cuda")
    for _ in range(3):
        H.matvec_device(1.0, x, 0.0, y)
    torch.cuda.synchronize()
    H.timing(1)
    for _ in range(a.iters):
        H.matvec_device(1.0, x, 0.0, y)
    ms_a, ms_b, calls = H.timing(0)
    # whole products back to back, no per-phase events (the phases chain by
    # programmatic dependent launch)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(a.iters):
        H.matvec_device(1.0, x, 0.0, y)
    e1.record()
    torch.cuda.synchronize()
    wall = e0.elapsed_time(e1) / a.iters
    r = H.memory()
    chk = ""
    if a.yref:
        yv = y.cpu().numpy()
        if os.path.exists(a.yref):
            y0 = np.load(a.yref)
            chk = f" relerr_vs_ref={np.linalg.norm(yv - y0) / np.linalg.norm(y0):.2e}"
        else:
            np.save(a.yref, yv)
    print({k: round(v, 2) for k, v in T.items()})
    print(f"n={n} arena={r.device_arena_bytes/1e6:.1f}MB algo={r.algorithmic_bytes/1e6:.1f}MB "
          f"stagesA={r.stages_a} stagesB={r.stages_b} phaseA={ms_a/calls:.4f}ms phaseB={ms_b/calls:.4f}ms "
          f"total={(ms_a+ms_b)/calls:.4f}ms -> {r.algorithmic_bytes/((ms_a+ms_b)/calls)/1e6:.1f} GB/s "
          f"wall={wall:.4f}ms -> {r.algorithmic_bytes/wall/1e6:.1f} GB/s" + chk, flush=True)
    if a.rhs4:  # 4 right-hand sides decoded once vs 4 single products
        X4 = torch.as_tensor(np.random.default_rng(1).uniform(-1, 1, (n, 4))).cuda().contiguous()
        Y4 = torch.zeros(n, 4, dtype=torch.float64, device="cuda")
        for _ in range(3):
            H.matmat4_device(1.0, X4, 0.0, Y4)
        e0.record()
        for _ in range(a.iters):
            H.matmat4_device(1.0, X4, 0.0, Y4)
        e1.record()
        torch.cuda.synchronize()
        t4 = e0.elapsed_time(e1) / a.iters
        ref = torch.stack([H.matvec_device(1.0, X4[:, c].contiguous(), 0.0, torch.zeros(n, dtype=torch.float64,
                                                                                      device="cuda")) for c in range(4)], 1)
        err = float((Y4 - ref).norm() / ref.norm())
        print(f"rhs4: {t4:.4f} ms per 4-RHS product vs {4 * wall:.4f} ms for 4 products "
              f"({4 * wall / t4:.2f}x), rel diff {err:.2e}")


if __name__ == "__main__":
    main()

