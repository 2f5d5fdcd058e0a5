"""Parity of the benched workloads and of the leaf shapes only they produce.

* the BASELINE config-3 product exactly as bench.py builds and times it
  (build_config(3) -> HMatrix), single and 4-RHS arenas, vs the CPU oracle;
* synthetic lowrank leaves 1000 ... 16384 columns wide: >= 16 phase-A
  segments per rank column, so k_reduce's warp-per-column branch runs (R = 1
  and the 4-RHS arena), plus odd and ragged chunk counts;
* an HCMX file loaded straight into a device handle;
* SPEC.md:456 compression-rate ordering and SPEC.md:466's compressed vs
  uncompressed product bound.
Tolerance: ||y - y_ref|| / ||y_ref|| <= 1e-12 (BASELINE north_star)."""
import os

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu
TOL = 1e-12


def rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


WIDE_LEAVES = [
    # kind, r0, r1, c0, c1, rank
    (1, 0, 64, 0, 8192, 12),         # 128 chunks -> 16 segments of 8 (warp branch, exactly kRedLong)
    (1, 64, 192, 0, 16384, 9),       # 256 chunks -> 32 segments (both halves of the warp loop)
    (1, 192, 256, 1000, 3112, 7),    # 33 chunks (odd) -> G = 1, 33 segments
    (1, 256, 320, 5000, 6000, 5),    # 15 chunks + 40 ragged rows -> 16 segments
    (1, 320, 448, 64, 640, 11),      # 9 chunks -> G = 1, 9 segments (thread branch)
    (1, 448, 512, 9000, 9512, 6),    # 8 chunks -> one segment, final in phase A
    (0, 512, 576, 128, 192, 0),      # dense
    (0, 576, 640, 16320, 16384, 0),  # dense, last columns
]


@pytest.mark.parametrize("scheme", [0, 2])
def test_wide_lowrank_leaves_reduce_branches(gpu, oracle, scheme):
    from cpu_hmatrix import flat_from_leaves
    from paper_2308_10960_b200.hmatrix import HMatrix
    f = flat_from_leaves(640, 16384, WIDE_LEAVES, eps=1e-8, scheme=scheme)
    H = HMatrix(f.to_product(), nrhs_block=4)
    rng = np.random.default_rng(3)
    x = rng.uniform(-1, 1, 16384)
    y0 = rng.standard_normal(640)
    for alpha, beta in ((1.0, 0.0), (-0.25, 1.5)):
        ref = oracle.hmat_matvec(f, alpha, x, beta, y0, threads=4)
        y = y0.copy()
        H.matvec(alpha, x, beta, y)
        assert rel(y, ref) <= TOL, (alpha, beta)
    X = np.asfortranarray(rng.uniform(-1, 1, (16384, 5)))   # 4-RHS arena (segments of 2 chunks)
    Y = np.zeros((640, 5), order="F")
    H.matmat(1.0, X, 0.0, Y)
    for j in range(5):
        assert rel(Y[:, j], oracle.hmat_matvec(f, 1.0, X[:, j], 0.0, np.zeros(640), threads=4)) <= TOL, j
    H.close()


def test_config3_benched_product(gpu, oracle):
    """the product bench.py times (BASELINE config 3, AFL-APLR, n = 131072), single
    right-hand side and the 4-RHS arena, vs the oracle over the whole matrix"""
    from paper_2308_10960_b200.hmatrix import HMatrix, build_config
    f, info = build_config(3)
    fh = f.host()
    n = f.n_rows
    threads = os.cpu_count() or 4
    rng = np.random.default_rng(0)
    x = rng.uniform(-1, 1, n)
    ref = oracle.hmat_matvec(fh, 1.0, x, 0.0, np.zeros(n), threads=threads)
    H = HMatrix(f)
    y = torch.zeros(n, dtype=torch.float64, device="cuda")
    H.matvec_device(1.0, torch.as_tensor(x).cuda(), 0.0, y)
    assert rel(y.cpu().numpy(), ref) <= TOL
    # widest leaves of the config go through k_reduce's warp branch
    cols = fh.col1 - fh.col0
    assert ((fh.kind == 1) & (cols >= 16 * 64)).any()
    H.close()
    H4 = HMatrix(f, nrhs_block=4)
    X4 = rng.uniform(-1, 1, (n, 4))
    Y4 = torch.zeros(n, 4, dtype=torch.float64, device="cuda")
    H4.matmat4_device(1.0, torch.as_tensor(X4).cuda().contiguous(), 0.0, Y4)
    Y4 = Y4.cpu().numpy()
    for j in range(4):
        assert rel(Y4[:, j], oracle.hmat_matvec(fh, 1.0, X4[:, j], 0.0, np.zeros(n), threads=threads)) <= TOL, j
    H4.close()


@pytest.mark.parametrize("mode,scheme", [("aplr", 0), ("codec", 1), ("mp", 0)])
def test_hcmx_file_into_device_handle(gpu, oracle, tmp_path, mode, scheme):
    """save_hcmx -> load_hcmx -> device arena -> matvec (hmatrix.hpp:150-153)"""
    from cpu_hmatrix import build_small_flat
    from paper_2308_10960_b200.formats import load_hcmx, save_hcmx
    from paper_2308_10960_b200.hmatrix import HMatrix
    f, x = build_small_flat(n=1100, eps=1e-6, scheme=scheme, mode=mode, geometry="sphere")
    path = os.path.join(tmp_path, "m.hcmx")
    save_hcmx(f.to_product(), path)
    H = HMatrix(load_hcmx(path))
    y = np.zeros(1100)
    H.matvec(1.0, x, 0.0, y)
    assert rel(y, oracle.hmat_matvec(f, 1.0, x, 0.0, np.zeros(1100), threads=4)) <= TOL
    H.close()


def test_spec_rate_ordering(gpu):
    """compression rate AFL >= AFLP >= BFL >= DFL >= 1 on the same matrix"""
    from paper_2308_10960_b200 import assemble, problems, tree
    from paper_2308_10960_b200.hmatrix import compress_in_place
    pts = problems.make_points("fibonacci", 4096, 1)
    ct = tree.build_cluster_tree(pts, 64)
    lv = tree.build_block_tree(ct, ct, 2.0)
    A = assemble.assemble(pts[ct.i2e], lv, problems.make_kernel("laplace"), 1e-6, device="cuda")
    rates = [compress_in_place(A, 1e-6, f"{s}-aplr").memory_footprint().rate()
             for s in ("afl", "aflp", "bfl", "dfl")]
    assert rates[0] >= rates[1] >= rates[2] >= rates[3] >= 1.0, rates


@pytest.mark.parametrize("scheme", [0, 1, 2, 3])
def test_spec_compressed_vs_uncompressed_bound(gpu, scheme):
    """||y_c - y|| <= 10 eps ||M||_F ||x||, y from the uncompressed
    (fp64) H-matrix, y_c from the compressed one, both on the device"""
    from cpu_hmatrix import build_small_flat
    from paper_2308_10960_b200.hmatrix import HMatrix
    eps = 1e-6
    fu, x = build_small_flat(n=1024, eps=eps, scheme=scheme, mode="fp64")
    fc, _ = build_small_flat(n=1024, eps=eps, scheme=scheme)
    Hu = HMatrix(fu.to_product())
    M = np.zeros((1024, 1024), order="F")
    Hu.matmat(1.0, np.eye(1024, order="F"), 0.0, M)   # the uncompressed matrix, column by column
    y = np.zeros(1024)
    yc = np.zeros(1024)
    Hu.matvec(1.0, x, 0.0, y)
    HMatrix(fc.to_product()).matvec(1.0, x, 0.0, yc)
    assert rel(y, M @ x) <= 1e-13          # SPEC.md:464 (uncompressed vs dense)
    assert np.linalg.norm(yc - y) <= 10 * eps * np.linalg.norm(M) * np.linalg.norm(x)
