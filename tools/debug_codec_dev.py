"""debug aid: compress_device flags / descriptors on exponent-threshold blocks"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2308_10960_b200 import codec  # noqa: E402
from paper_2308_10960_b200._lib import DESC_DTYPE  # noqa: E402

rng = np.random.default_rng(5)
blocks = [np.sign(rng.standard_normal(4096)) * 10 ** rng.uniform(-6, 0, 4096) for _ in range(3)]
for span in (6, 14):
    v = 2.0 ** rng.uniform(0, span, 300)
    v[0], v[1] = 1.0, 2.0 ** span
    blocks.append(v)
blocks.append(np.zeros(100))
counts = np.array([b.size for b in blocks], np.uint64)
vals = torch.as_tensor(np.concatenate(blocks)).cuda()
db = codec.device_batch(vals, counts, 1e-6, 0)
codec.compress_device(vals, db)
torch.cuda.synchronize()
print("flags", db.d_flags.cpu().numpy())
print("desc", db.d_desc.cpu().numpy().view(DESC_DTYPE))
bb = codec.compress_batch(vals, counts, 1e-6, 0)
print("host api desc", bb.desc)
