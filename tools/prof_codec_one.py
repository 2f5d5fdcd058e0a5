"""One config-2 codec call per kernel for ncu (profiling aid): AFL eps 1e-6,
compress_device then decompress_batch, after one warm-up each."""
import os
import sys

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
bb = codec.compress_batch(d, counts, 1e-6, codec.Scheme.afl, d_voff=dv)
dec = codec.decompress_batch(bb)
db = codec.device_batch(d, counts, 1e-6, codec.Scheme.afl)
for _ in range(2):
    codec.compress_device(d, db)
    codec.decompress_batch(bb, out=dec)
torch.cuda.synchronize()
