"""Assembly timing for a BASELINE config on the GPU box (profiling aid)."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("HCMX_VERBOSE", "1")
from paper_2308_10960_b200 import problems, tree  # noqa: E402
from paper_2308_10960_b200.assemble import assemble  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "4"
c = problems.config(cfg)
if len(sys.argv) > 2:
    c["n"] = int(sys.argv[2])
t = time.time()
pts = problems.make_points(c["geometry"], c["n"], 1)
ct = tree.build_cluster_tree(pts, c["leaf"])
lv = tree.build_block_tree(ct, ct, c["eta"])
print(f"tree {time.time() - t:.1f}s", flush=True)
t = time.time()
A = assemble(pts[ct.i2e], lv, problems.make_kernel(c["kernel"]), c["eps"], device="cuda")
torch.cuda.synchronize()
lr = A.kind == 1
print(f"assemble {time.time() - t:.1f}s ranks mean {A.rank[lr].mean():.2f} max {A.rank.max()} sum {A.rank.sum()}",
      flush=True)
