"""One config-2 batch (4096 x 4096 values, AFL eps 1e-6): compress + decompress
a few times; for ncu captures of the codec kernels (not part of the product)."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2308_10960_b200 import codec  # noqa: E402

nb, bs = 4096, 4096
rng = np.random.default_rng(2)
vals = np.sign(rng.standard_normal(nb * bs)) * 10 ** rng.uniform(-6, 0, nb * bs)
d = torch.as_tensor(vals).cuda()
counts = np.full(nb, bs, np.uint64)
dv = torch.as_tensor(np.arange(nb, dtype=np.int64) * bs).cuda()
eps = float(sys.argv[1]) if len(sys.argv) > 1 else 1e-6
bb = codec.compress_batch(d, counts, eps, 0, d_voff=dv)
out = codec.decompress_batch(bb)
torch.cuda.synchronize()
for it in range(3):
    t = time.perf_counter()
    for _ in range(10):
        codec.decompress_batch(bb, out=out)
    torch.cuda.synchronize()
    td = (time.perf_counter() - t) / 10
    t = time.perf_counter()
    for _ in range(10):
        codec.compress_batch(d, counts, eps, 0, payload=bb.payload, d_voff=dv)
    torch.cuda.synchronize()
    tc = (time.perf_counter() - t) / 10
    print(f"per call: decompress {td * 1e6:.1f} us, compress {tc * 1e6:.1f} us")
