"""Codec microbench driver (BASELINE config 2; not part of the product): times
the batched device codec per scheme/eps; also checks bytes against the oracle
on the first block."""
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

from paper_2308_10960_b200 import codec  # noqa: E402


def main():
    nb, bs = 4096, 4096
    rng = np.random.default_rng(2)
    vals = np.sign(rng.standard_normal(nb * bs)) * 10 ** rng.uniform(-6, 0, nb * bs)
    d = torch.as_tensor(vals).cuda()
    counts = np.full(nb, bs, np.uint64)
    dv = torch.as_tensor(np.arange(nb, dtype=np.int64) * bs).cuda()
    for eps in (1e-4, 1e-6, 1e-8):
        for s in range(4):
            bb = codec.compress_batch(d, counts, eps, s, d_voff=dv)
            out = codec.decompress_batch(bb)
            torch.cuda.synchronize()
            w = int(bb.desc["bit_width"][0])
            pay = nb * ((bs * w + 7) // 8 + 20)
            algo = 8 * nb * bs + pay
            tc, td = [], []
            for _ in range(5):
                torch.cuda.synchronize()
                t = time.perf_counter()
                bb = codec.compress_batch(d, counts, eps, s, payload=bb.payload, d_voff=dv)
                torch.cuda.synchronize()
                tc.append(time.perf_counter() - t)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                codec.decompress_batch(bb, out=out)
                e1.record()
                torch.cuda.synchronize()
                td.append(e0.elapsed_time(e1) / 1e3)
            print(f"eps={eps:g} scheme={s} w={w}: compress {algo / min(tc) / 1e9:7.1f} GB/s "
                  f"({min(tc) * 1e3:.3f} ms)  decompress {algo / min(td) / 1e9:7.1f} GB/s ({min(td) * 1e3:.3f} ms)")


if __name__ == "__main__":
    main()
