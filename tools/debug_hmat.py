"""Debug driver (not part of the product): GPU matvec vs oracle on subsets of
leaves (dense only / lowrank only) for a given small problem."""
import os
import sys
from dataclasses import replace

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
sys.path.insert(0, os.path.join(ROOT, "tests"))

from cpu_hmatrix import build_small_flat  # noqa: E402
from oracle import Oracle  # noqa: E402
from paper_2308_10960_b200.hmatrix import HMatrix  # noqa: E402


def sub(f, sel):
    return replace(f, row0=f.row0[sel], row1=f.row1[sel], col0=f.col0[sel], col1=f.col1[sel],
                   kind=f.kind[sel], rank=f.rank[sel], buf0=f.buf0[sel], sig0=f.sig0[sel])


def main():
    o = Oracle()
    for geometry, kernel, n, eps in [("sphere", "laplace", 1100, 1e-4), ("fibonacci", "laplace", 1024, 1e-4)]:
        for scheme in range(4):
            f, x = build_small_flat(n=n, eps=eps, scheme=scheme, geometry=geometry, kernel=kernel)
            for name, sel in [("all", np.ones(f.row0.size, bool)), ("dense", f.kind == 0), ("lowrank", f.kind == 1)]:
                g = sub(f, sel)
                ref = o.hmat_matvec(g, 1.0, x, 0.0, np.zeros(n))
                y = np.zeros(n)
                HMatrix(g.to_product()).matvec(1.0, x, 0.0, y)
                err = np.linalg.norm(y - ref) / np.linalg.norm(ref)
                bad = np.nonzero(np.abs(y - ref) > 1e-10 * np.abs(ref).max())[0]
                print(f"{geometry} n={n} eps={eps} scheme={scheme} {name:8s} rel={err:.2e} bad_rows={bad[:12]} nbad={bad.size}")


if __name__ == "__main__":
    main()
