"""Workload statistics of a built config (profiling aid, not part of the product):
leaf-size classes, ranks, widths and the packed bytes each class carries in the
two matvec phases (phase A: X factors of lowrank leaves, phase B: dense leaves
and W factors)."""
import argparse
import collections
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2308_10960_b200.hmatrix import build_config  # noqa: E402
from paper_2308_10960_b200 import problems  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="3")
    ap.add_argument("--n", type=int, default=None)
    a = ap.parse_args()
    flat, _ = build_config(problems.config(a.config), n=a.n)
    flat = flat.host()
    rows = flat.row1 - flat.row0
    cols = flat.col1 - flat.col0
    w = 1 + flat.desc["exp_bits"].astype(int) + flat.desc["mant_bits"].astype(int)
    print(f"n={flat.n_rows} leaves={flat.nleaves} dense={(flat.kind == 0).sum()} lowrank={(flat.kind != 0).sum()}")
    # dense leaves
    d = np.nonzero(flat.kind == 0)[0]
    cls = collections.Counter(zip(rows[d].tolist(), cols[d].tolist()))
    print("dense (rows, cols): count", dict(cls.most_common(8)))
    bd = flat.plen[flat.buf0[d]].sum()
    print(f"dense packed bytes {bd / 1e6:.1f} MB, widths {collections.Counter(w[flat.buf0[d]].tolist()).most_common(6)}")
    # lowrank leaves: buffers buf0 .. buf0 + 2k (W columns then X columns)
    lr = np.nonzero(flat.kind != 0)[0]
    byc = collections.defaultdict(lambda: [0, 0, 0, 0.0, collections.Counter()])
    for i in lr:
        k = int(flat.rank[i])
        b0 = int(flat.buf0[i])
        key = (int(rows[i]), int(cols[i]))
        s = byc[key]
        s[0] += 1
        s[1] += int(flat.plen[b0:b0 + k].sum())        # W (phase B)
        s[2] += int(flat.plen[b0 + k:b0 + 2 * k].sum())  # X (phase A)
        s[3] += k
        s[4].update(w[b0 + k:b0 + 2 * k].tolist())
    print("lowrank (rows, cols): leaves, W MB, X MB, mean k, X widths")
    for key in sorted(byc):
        s = byc[key]
        print(f"  {key}: {s[0]:6d} {s[1] / 1e6:8.1f} {s[2] / 1e6:8.1f} {s[3] / s[0]:6.1f} {s[4].most_common(5)}")
    ks = flat.rank[lr]
    print("rank histogram", np.histogram(ks, bins=[0, 4, 8, 12, 16, 20, 24, 28, 32, 48, 64, 1000]))


if __name__ == "__main__":
    main()
