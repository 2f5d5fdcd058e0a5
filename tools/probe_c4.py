"""Setup probe for a BASELINE config on one GPU: time and memory of every setup
stage (points, trees, FP64 assembly, device compress_in_place, hmat_create),
then a few products.  Profiling aid, not part of the product.

    python tools/probe_c4.py [config] [n]
"""
import os
import resource
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("HCMX_VERBOSE", "1")

from paper_2308_10960_b200 import problems, tree  # noqa: E402
from paper_2308_10960_b200.assemble import assemble  # noqa: E402
from paper_2308_10960_b200.hmatrix import HMatrix, compress_in_place  # noqa: E402


def mem():
    rss = resource.getrusage(resource.RUSAGE_SELF).ru_maxrss / 1e6
    return f"gpu {torch.cuda.memory_allocated() / 1e9:.1f} GB (max {torch.cuda.max_memory_allocated() / 1e9:.1f}), host maxrss {rss:.1f} GB"


def main():
    cfg = sys.argv[1] if len(sys.argv) > 1 else "4"
    c = problems.config(cfg)
    if len(sys.argv) > 2:
        c["n"] = int(sys.argv[2])
    print("nproc", os.cpu_count(), flush=True)
    os.system("free -g; nvidia-smi --query-gpu=name,memory.total --format=csv")
    t = time.time()
    pts = problems.make_points(c["geometry"], c["n"], 1)
    ct = tree.build_cluster_tree(pts, c["leaf"])
    lv = tree.build_block_tree(ct, ct, c["eta"])
    print(f"tree: {time.time() - t:.1f}s leaves {len(lv)} adm {int(lv.admissible.sum())}", flush=True)
    t = time.time()
    A = assemble(pts[ct.i2e], lv, problems.make_kernel(c["kernel"]), c["eps"], device="cuda")
    torch.cuda.synchronize()
    print(f"assemble: {time.time() - t:.1f}s ranks mean {A.rank[A.kind == 1].mean():.2f} max {A.rank.max()} | {mem()}",
          flush=True)
    t = time.time()
    f = compress_in_place(A, c["eps"], "afl-aplr")
    torch.cuda.synchronize()
    print(f"compress_in_place: {time.time() - t:.1f}s blob {f.blob.numel() / 1e9:.2f} GB | {mem()}", flush=True)
    del A
    torch.cuda.empty_cache()
    t = time.time()
    H = HMatrix(f)
    print(f"hmat_create: {time.time() - t:.1f}s | {mem()}", flush=True)
    rep = H.memory()
    print("arena", rep.device_arena_bytes / 1e9, "algo", rep.algorithmic_bytes / 1e9, flush=True)
    x = torch.rand(c["n"], dtype=torch.float64, device="cuda") * 2 - 1
    y = torch.zeros_like(x)
    for _ in range(3):
        H.matvec_device(1.0, x, 0.0, y)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        H.matvec_device(1.0, x, 0.0, y)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 20
    print(f"product {ms:.3f} ms  {rep.algorithmic_bytes / ms / 1e6:.1f} GB/s", flush=True)


if __name__ == "__main__":
    main()
