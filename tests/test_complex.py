"""Config 5 (complex Helmholtz kernel, multi-RHS): the real / imaginary split of
assemble_complex reproduces every complex block (CPU), and the device product
of the two compressed real H-matrices matches the CPU oracle applied to the
same compressed matrices (||dY|| / ||Y|| <= 1e-12) and the dense complex kernel
matrix to the compression accuracy."""
import numpy as np
import pytest
import torch

TOL = 1e-12  # BASELINE.json north_star


def _setup(n, device):
    from paper_2308_10960_b200 import assemble, problems, tree
    pts = problems.make_points("fibonacci", n, 1)
    ct = tree.build_cluster_tree(pts, 64)
    lv = tree.build_block_tree(ct, ct, 2.0)
    K = problems.make_kernel("helmholtz")
    Ar, Ai = assemble.assemble_complex(pts[ct.i2e], lv, K, 1e-6, device=device)
    return pts[ct.i2e], lv, K, Ar, Ai


def test_complex_split_reconstructs_blocks():
    P, lv, K, Ar, Ai = _setup(1024, "cpu")
    Pt = torch.as_tensor(P)
    assert (Ar.kind == 1).any() and (Ar.kind == 0).any()
    for l in range(len(lv)):
        r0, r1, c0, c1 = lv.row0[l], lv.row1[l], lv.col0[l], lv.col1[l]
        m, n = r1 - r0, c1 - c0
        B = K.block(Pt[r0:r1], Pt[c0:c1]).numpy()
        if Ar.kind[l] == 0:
            o = Ar.dense_off[l]
            R = Ar.dense[o:o + m * n].numpy().reshape(n, m).T + 1j * Ai.dense[o:o + m * n].numpy().reshape(n, m).T
            assert np.array_equal(R, B)
        else:
            k = int(Ar.rank[l])
            assert k % 2 == 0
            Wr = Ar.W[Ar.w_off[l]:Ar.w_off[l] + m * k].numpy().reshape(k, m).T
            Wi = Ai.W[Ai.w_off[l]:Ai.w_off[l] + m * k].numpy().reshape(k, m).T
            X = Ar.X[Ar.x_off[l]:Ar.x_off[l] + n * k].numpy().reshape(k, n).T
            s = Ar.sigma[Ar.sig_off[l]:Ar.sig_off[l] + k]
            assert np.array_equal(s[: k // 2], s[k // 2:])
            R = (Wr * s) @ X.T + 1j * ((Wi * s) @ X.T)
            assert np.abs(R - B).max() <= 1e-5 * np.abs(B).max(), l


@pytest.mark.gpu
def test_complex_multi_rhs_vs_oracle(gpu, oracle):
    from paper_2308_10960_b200.hmatrix import ComplexHMatrix, compress_in_place
    n, r = 2048, 4
    P, lv, K, Ar, Ai = _setup(n, "cuda")
    fr, fi = compress_in_place(Ar, 1e-6, "afl-aplr"), compress_in_place(Ai, 1e-6, "afl-aplr")
    H = ComplexHMatrix(fr, fi)
    rng = np.random.default_rng(7)
    X = rng.uniform(-1, 1, (n, r)) + 1j * rng.uniform(-1, 1, (n, r))   # config 5 right-hand sides
    Y0 = rng.standard_normal((n, r)) + 1j * rng.standard_normal((n, r))
    alpha, beta = 0.5 - 0.25j, 1.0 + 2.0j
    Y = Y0.copy()
    H.matmat(alpha, X, beta, Y)
    hr, hi = fr.host(), fi.host()
    mv = lambda h, v: oracle.hmat_matvec(h, 1.0, v, 0.0, np.zeros(n), threads=4)
    ref = np.empty_like(Y)
    for j in range(r):
        xr, xi = X[:, j].real.copy(), X[:, j].imag.copy()
        ax = (mv(hr, xr) - mv(hi, xi)) + 1j * (mv(hr, xi) + mv(hi, xr))
        ref[:, j] = alpha * ax + beta * Y0[:, j]
    assert np.linalg.norm(Y - ref) / np.linalg.norm(ref) <= TOL
    # against the dense complex kernel matrix: the compression accuracy
    A = K.block(torch.as_tensor(P), torch.as_tensor(P)).numpy()
    y = np.zeros(n, np.complex128)
    H.matvec(1.0, X[:, 0], 0.0, y)
    assert np.linalg.norm(y - A @ X[:, 0]) / np.linalg.norm(A @ X[:, 0]) <= 1e-4
    H.close()


@pytest.mark.gpu
def test_complex_matmat_device_16_rhs(gpu, oracle):
    """config 5's operation at reduced size: 16 complex right-hand sides through the
    4-RHS arenas with the real / imaginary combination on the device, each column
    equal to the oracle applied to the same compressed real / imaginary matrices"""
    from paper_2308_10960_b200.hmatrix import ComplexHMatrix, build_config_complex
    n = 4096
    fr, fi, info = build_config_complex("5", n=n)
    H = ComplexHMatrix(fr, fi, nrhs_block=8)  # 8 real slots: 4 complex columns per device product
    rng = np.random.default_rng(12)
    X = rng.uniform(-1, 1, (n, 16)) + 1j * rng.uniform(-1, 1, (n, 16))
    Y = H.matmat_device(torch.as_tensor(X).cuda()).cpu().numpy()
    frh, fih = fr.host(), fi.host()
    for j in (0, 7, 15):
        yr = oracle.hmat_matvec(frh, 1.0, X[:, j].real, 0.0, np.zeros(n), threads=4) - \
            oracle.hmat_matvec(fih, 1.0, X[:, j].imag, 0.0, np.zeros(n), threads=4)
        yi = oracle.hmat_matvec(frh, 1.0, X[:, j].imag, 0.0, np.zeros(n), threads=4) + \
            oracle.hmat_matvec(fih, 1.0, X[:, j].real, 0.0, np.zeros(n), threads=4)
        ref = yr + 1j * yi
        assert np.linalg.norm(Y[:, j] - ref) <= TOL * np.linalg.norm(ref), j
    H.close()


@pytest.mark.gpu
def test_complex_arena_decodes_each_stream_once(gpu, oracle):
    """the complex arena holds every real / imaginary stream once (the lowrank
    bytes of one real H-matrix -- the other's [Ui -Ur] factors are the same
    streams -- plus both dense parts), odd column counts and beta != 0 work, and
    the real-vector entry points refuse a complex handle"""
    from paper_2308_10960_b200.hmatrix import ComplexHMatrix, HMatrix, compress_in_place, complex_flat
    n, r = 2048, 3
    P, lv, K, Ar, Ai = _setup(n, "cuda")
    fr, fi = compress_in_place(Ar, 1e-6, "afl-aplr"), compress_in_place(Ai, 1e-6, "afl-aplr")
    H = ComplexHMatrix(complex_flat(fr, fi), nrhs_block=4)  # 2 complex columns per product
    Hr, Hi = HMatrix(fr), HMatrix(fi)
    mc, mr, mi = H.memory(), Hr.memory(), Hi.memory()
    assert mc.lowrank_compressed == mr.lowrank_compressed
    assert mc.dense_compressed == mr.dense_compressed + mi.dense_compressed
    Hr.close()
    Hi.close()
    rng = np.random.default_rng(3)
    X = rng.uniform(-1, 1, (n, r)) + 1j * rng.uniform(-1, 1, (n, r))
    Y0 = rng.standard_normal((n, r)) + 1j * rng.standard_normal((n, r))
    Yd = H.matmat_device(torch.as_tensor(X).cuda(), torch.as_tensor(Y0).cuda(), alpha=2.0 - 1.0j, beta=0.5j)
    hr, hi = fr.host(), fi.host()
    mv = lambda h, v: oracle.hmat_matvec(h, 1.0, v, 0.0, np.zeros(n), threads=4)
    Y = Yd.cpu().numpy()
    for j in range(r):
        xr, xi = X[:, j].real.copy(), X[:, j].imag.copy()
        ref = (2.0 - 1.0j) * ((mv(hr, xr) - mv(hi, xi)) + 1j * (mv(hr, xi) + mv(hi, xr))) + 0.5j * Y0[:, j]
        assert np.linalg.norm(Y[:, j] - ref) <= TOL * np.linalg.norm(ref), j
    with pytest.raises(ValueError):
        H.h.matvec(1.0, np.zeros(n), 0.0, np.zeros(n))
    H.close()


@pytest.mark.gpu
@pytest.mark.parametrize("mode,block", [("aflp-aplr", 4), ("bfl-aplr", 8), ("dfl-aplr", 4)])
def test_complex_arena_schemes(gpu, oracle, mode, block):
    """the complex arena over every codec scheme (BFL / DFL: fixed exponent
    widths, the generic decoder for e = 11) and both block widths, against the
    oracle on the same compressed real / imaginary matrices"""
    from paper_2308_10960_b200.hmatrix import ComplexHMatrix, compress_in_place
    n, r = 2048, 5
    P, lv, K, Ar, Ai = _setup(n, "cuda")
    fr, fi = compress_in_place(Ar, 1e-6, mode), compress_in_place(Ai, 1e-6, mode)
    H = ComplexHMatrix(fr, fi, nrhs_block=block)
    rng = np.random.default_rng(9)
    X = rng.uniform(-1, 1, (n, r)) + 1j * rng.uniform(-1, 1, (n, r))
    Y = H.matmat_device(torch.as_tensor(X).cuda()).cpu().numpy()
    hr, hi = fr.host(), fi.host()
    mv = lambda h, v: oracle.hmat_matvec(h, 1.0, v, 0.0, np.zeros(n), threads=4)
    for j in range(r):
        xr, xi = X[:, j].real.copy(), X[:, j].imag.copy()
        ref = (mv(hr, xr) - mv(hi, xi)) + 1j * (mv(hr, xi) + mv(hi, xr))
        assert np.linalg.norm(Y[:, j] - ref) <= TOL * np.linalg.norm(ref), j
    H.close()
