"""Compressed H-matvec on the GPU vs the CPU oracle / reference glue:
||y - y_ref|| / ||y_ref|| <= 1e-12 (BASELINE north star; FP64 reassociation only),
APLR compression bit-exact, device layout round trip, alpha/beta semantics,
row partitions, determinism."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu
TOL = 1e-12  # written in BASELINE.json north_star


def rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


def test_golden_hmatrix(gpu, hmat_golden):
    """reference-compressed leaves (n=768: ragged 48-row clusters), reference-glue y"""
    from cpu_hmatrix import Flat
    from paper_2308_10960_b200.hmatrix import HMatrix
    f = Flat.from_npz(hmat_golden).to_product()
    H = HMatrix(f)
    x = hmat_golden["x"]
    y = np.zeros(f.n_rows)
    H.matvec(1.0, x, 0.0, y)
    assert rel(y, hmat_golden["y"]) <= TOL
    y2 = hmat_golden["y"].copy()
    H.matvec(-0.5, x, 2.0, y2)
    assert rel(y2, hmat_golden["y2"]) <= TOL
    # every packed buffer survives the re-tiling into the device arena bit for bit
    for b in range(0, f.count.size, 7):
        got = H.export_buffer(b, int(f.plen[b]))
        assert got == f.blob[f.poff[b]: f.poff[b] + f.plen[b]].tobytes(), b


@pytest.mark.parametrize("geometry,kernel,n,eps,scheme", [
    ("fibonacci", "laplace", 2048, 1e-6, 0),
    ("fibonacci", "laplace", 1536, 1e-8, 1),
    ("cube", "matern", 1000, 1e-6, 2),
    ("sphere", "laplace", 1100, 1e-4, 3),
    # low ranks (1-3): phase-A items gather many leaves, so their x slices hit
    # the per-item staging cap
    ("cube", "matern", 4096, 1e-2, 0),
])
def test_oracle_compressed_matrices(gpu, oracle, geometry, kernel, n, eps, scheme):
    from cpu_hmatrix import build_small_flat
    from paper_2308_10960_b200.hmatrix import HMatrix
    f, x = build_small_flat(n=n, eps=eps, scheme=scheme, geometry=geometry, kernel=kernel)
    H = HMatrix(f.to_product())
    y0 = np.random.default_rng(1).standard_normal(n)
    for alpha, beta in ((1.0, 0.0), (0.3, 1.0), (-2.0, -0.5)):
        ref = oracle.hmat_matvec(f, alpha, x, beta, y0, threads=4)
        y = y0.copy()
        H.matvec(alpha, x, beta, y)
        assert rel(y, ref) <= TOL, (alpha, beta)


def test_alpha_zero_leaves_matrix_untouched(gpu, hmat_golden):
    from cpu_hmatrix import Flat
    from paper_2308_10960_b200.hmatrix import HMatrix
    H = HMatrix(Flat.from_npz(hmat_golden).to_product())
    y = np.random.default_rng(2).standard_normal(H.n_rows)
    y0 = y.copy()
    H.matvec(0.0, hmat_golden["x"], 3.0, y)
    assert (y == 3.0 * y0).all()
    assert H.launches() == 1
    with pytest.raises(ValueError):
        H.matvec(1.0, np.zeros(H.n_cols + 1), 0.0, np.zeros(H.n_rows))
    with pytest.raises(ValueError):
        H.matvec(1.0, hmat_golden["x"], 0.0, y, transpose=True)


def test_device_compress_in_place_bit_exact(gpu, oracle):
    """the product setup: FP64 assembly -> GPU compress_in_place; every buffer equals
    the oracle's compress / APLR of the same FP64 inputs, and the matvec matches"""
    from paper_2308_10960_b200 import assemble, problems, tree
    from paper_2308_10960_b200.hmatrix import HMatrix, compress_in_place
    pts = problems.make_points("fibonacci", 2048, 1)
    ct = tree.build_cluster_tree(pts, 64)
    lv = tree.build_block_tree(ct, ct, 2.0)
    A = assemble.assemble(pts[ct.i2e], lv, problems.make_kernel("laplace"), 1e-6, device="cuda")
    f = compress_in_place(A, 1e-6, "afl-aplr")
    fh = f.host()
    dense, W, X = A.dense.cpu().numpy(), A.W.cpu().numpy(), A.X.cpu().numpy()
    rows, cols = lv.row1 - lv.row0, lv.col1 - lv.col0
    for l in range(len(lv)):
        b0 = int(fh.buf0[l])
        if A.kind[l] == 0:
            ob = oracle.compress(dense[A.dense_off[l]: A.dense_off[l] + rows[l] * cols[l]], 1e-6, 0)
            bufs = [ob]
        else:
            k = int(A.rank[l])
            Wl = W[A.w_off[l]: A.w_off[l] + rows[l] * k].reshape(k, rows[l]).T
            Xl = X[A.x_off[l]: A.x_off[l] + cols[l] * k].reshape(k, cols[l]).T
            bufs = oracle.aplr_compress(Wl, Xl, A.sigma[A.sig_off[l]: A.sig_off[l] + k], 1e-6, 0)
        for i, ob in enumerate(bufs):
            b = b0 + i
            assert (fh.e[b], fh.m[b], fh.scale[b]) == (ob.e, ob.m, ob.scale)
            assert fh.blob[fh.poff[b]: fh.poff[b] + fh.plen[b]].tobytes() == ob.payload
    x = np.random.default_rng(0).uniform(-1, 1, 2048)
    ref = oracle.hmat_matvec(fh, 1.0, x, 0.0, np.zeros(2048), threads=4)
    y = np.zeros(2048)
    HMatrix(f).matvec(1.0, x, 0.0, y)
    assert rel(y, ref) <= TOL


def test_row_partitions_compose(gpu, oracle):
    """block-row partitioning (multi-GPU layout) on one device: the disjoint y
    slices of two handles equal the full product"""
    from cpu_hmatrix import build_small_flat
    from paper_2308_10960_b200.hmatrix import HMatrix
    f, x = build_small_flat(n=2048, eps=1e-6, scheme=0)
    ref = oracle.hmat_matvec(f, 1.0, x, 0.0, np.zeros(2048), threads=4)
    fp = f.to_product()
    for cuts in ([0, 1024, 2048], [0, 320, 1344, 2048], [0, 64, 2048]):
        y = np.full(2048, np.nan)
        for a, b in zip(cuts[:-1], cuts[1:]):
            H = HMatrix(fp, row_range=(a, b))
            H.matvec(1.0, x, 0.0, y)
        assert rel(y, ref) <= TOL, cuts


def test_deterministic_and_device_api(gpu, hmat_golden):
    from cpu_hmatrix import Flat
    from paper_2308_10960_b200.hmatrix import HMatrix
    H = HMatrix(Flat.from_npz(hmat_golden).to_product())
    x = torch.as_tensor(hmat_golden["x"]).cuda()
    ys = []
    for _ in range(3):
        y = torch.zeros(H.n_rows, dtype=torch.float64, device="cuda")
        H.matvec_device(1.0, x, 0.0, y)
        ys.append(y.cpu().numpy())
    assert all((ys[0].view(np.uint64) == t.view(np.uint64)).all() for t in ys[1:])
    yh = np.zeros(H.n_rows)
    H.matvec(1.0, hmat_golden["x"], 0.0, yh)
    assert (yh.view(np.uint64) == ys[0].view(np.uint64)).all()
    assert H.launches() in (2, 3)  # phase A, phase B (+ k_combine when row blocks are split)


def test_config1_full_size(gpu, oracle):
    """BASELINE config 1 (n=8192 Laplace sphere, eps 1e-6, AFL-APLR) end to end"""
    from paper_2308_10960_b200.hmatrix import HMatrix, build_config
    f, info = build_config(1)
    fh = f.host()
    assert 1300 <= info["dense_leaves"] <= 1400 and 2600 <= info["lowrank_leaves"] <= 2800
    x = np.random.default_rng(0).uniform(-1, 1, f.n_cols)
    ref = oracle.hmat_matvec(fh, 1.0, x, 0.0, np.zeros(f.n_rows), threads=8)
    H = HMatrix(f)
    y = np.zeros(f.n_rows)
    H.matvec(1.0, x, 0.0, y)
    assert rel(y, ref) <= TOL
    rep = H.memory()
    assert rep.dense_leaves == info["dense_leaves"]
    rate = rep.uncompressed_equivalent / (rep.dense_compressed + rep.lowrank_compressed)
    assert rate > 3.0  # ~29% of FP64 storage


@pytest.mark.parametrize("eps,scheme", [(1e-12, 3), (1e-9, 2), (1e-14, 0)])
def test_wide_fields(gpu, oracle, eps, scheme):
    """w > 32 / e = 11 layouts take the generic 64-bit decoder in both phases"""
    from cpu_hmatrix import build_small_flat
    from paper_2308_10960_b200.hmatrix import HMatrix
    f, x = build_small_flat(n=1024, eps=eps, scheme=scheme)
    assert int(f.e.max()) == 11 or (f.e.astype(int) + f.m.astype(int) + 1).max() > 32
    H = HMatrix(f.to_product())
    y = np.zeros(1024)
    H.matvec(1.0, x, 0.0, y)
    assert rel(y, oracle.hmat_matvec(f, 1.0, x, 0.0, np.zeros(1024), threads=4)) <= TOL


def test_rank_zero_and_zero_blocks(gpu, oracle):
    """lowrank leaves of rank 0 and all-zero dense blocks contribute nothing"""
    from dataclasses import replace
    from cpu_hmatrix import build_small_flat
    from paper_2308_10960_b200.hmatrix import HMatrix
    f, x = build_small_flat(n=768, eps=1e-6, scheme=0)
    lr = np.nonzero((f.kind == 1) & (f.rank > 0))[0]
    rank = f.rank.copy()
    rank[lr[::3]] = 0  # drop every third lowrank leaf (its buffers stay unused)
    f0 = replace(f, rank=rank)
    H = HMatrix(f0.to_product())
    y = np.zeros(768)
    H.matvec(1.0, x, 0.0, y)
    assert rel(y, oracle.hmat_matvec(f0, 1.0, x, 0.0, np.zeros(768), threads=4)) <= TOL


@pytest.mark.parametrize("mode,scheme,dense_too", [
    ("codec", 0, True),    # CodecDense + CodecLowrank (AFL)
    ("codec", 2, False),   # BFL lowrank factors, FP64 dense leaves
    ("mp", 0, True),       # FP64 dense + MP-D-S-H lowrank groups
    ("fp64", 0, True),     # uncompressed
])
def test_storage_modes(gpu, oracle, mode, scheme, dense_too):
    """every StorageMode kind (hmatrix.hpp:32-40) through the fused matvec, and the
    device compress_in_place producing the same buffers as the CPU construction"""
    from cpu_hmatrix import build_small_flat
    from paper_2308_10960_b200.hmatrix import HMatrix, compress_in_place
    eps = 1e-6
    f, x, A = build_small_flat(n=1024, eps=eps, scheme=scheme, mode=mode, dense_too=dense_too,
                               return_assembled=True)
    H = HMatrix(f.to_product())
    y0 = np.random.default_rng(3).standard_normal(1024)
    for alpha, beta in ((1.0, 0.0), (0.7, -1.5)):
        y = y0.copy()
        H.matvec(alpha, x, beta, y)
        assert rel(y, oracle.hmat_matvec(f, alpha, x, beta, y0, threads=4)) <= TOL, (alpha, beta)
    name = {"codec": ["afl", "aflp", "bfl", "dfl"][scheme]}.get(mode, mode)
    g = compress_in_place(A, eps, name, dense_too=dense_too).host()
    assert (g.kind == f.kind).all() and (g.count == f.count).all()
    assert (g.desc["scheme"] == f.scheme).all()
    for b in range(f.count.size):
        assert g.blob[g.poff[b]: g.poff[b] + g.plen[b]].tobytes() == \
            f.blob[f.poff[b]: f.poff[b] + f.plen[b]].tobytes(), b
    y = np.zeros(1024)
    HMatrix(g).matvec(1.0, x, 0.0, y)
    assert rel(y, oracle.hmat_matvec(f, 1.0, x, 0.0, np.zeros(1024), threads=4)) <= TOL


@pytest.mark.parametrize("mode,scheme", [("aplr", 0), ("codec", 1), ("mp", 0), ("aplr", 3)])
def test_transpose(gpu, oracle, mode, scheme):
    """hmatrix.hpp:128 matvec(..., transpose = true) vs the oracle's M^T product;
    ragged clusters (n = 1100) and every leaf kind"""
    from cpu_hmatrix import build_small_flat
    from paper_2308_10960_b200.hmatrix import HMatrix
    n = 1100
    f, x = build_small_flat(n=n, eps=1e-6, scheme=scheme, mode=mode, geometry="sphere")
    H = HMatrix(f.to_product(), with_transpose=True)
    y0 = np.random.default_rng(5).standard_normal(n)
    for alpha, beta in ((1.0, 0.0), (-0.4, 2.0)):
        ref = oracle.hmat_matvec(f, alpha, x, beta, y0, threads=4, transpose=True)
        y = y0.copy()
        H.matvec(alpha, x, beta, y, transpose=True)
        assert rel(y, ref) <= TOL, (alpha, beta)
        y = y0.copy()  # the forward product is unchanged by the extra handle
        H.matvec(alpha, x, beta, y)
        assert rel(y, oracle.hmat_matvec(f, alpha, x, beta, y0, threads=4)) <= TOL
    with pytest.raises(ValueError):
        HMatrix(f.to_product()).matvec(1.0, x, 0.0, np.zeros(n), transpose=True)


def test_matmat_multi_rhs(gpu, oracle):
    """several right-hand sides (forward and transposed) == column-wise oracle products"""
    from cpu_hmatrix import build_small_flat
    from paper_2308_10960_b200.hmatrix import HMatrix
    n = 1024
    f, _ = build_small_flat(n=n, eps=1e-6, scheme=0)
    H = HMatrix(f.to_product(), with_transpose=True)
    rng = np.random.default_rng(6)
    X = np.asfortranarray(rng.uniform(-1, 1, (n, 5)))
    Y0 = np.asfortranarray(rng.standard_normal((n, 5)))
    for tr in (False, True):
        Y = Y0.copy(order="F")
        H.matmat(0.5, X, -1.0, Y, transpose=tr)
        for j in range(5):
            ref = oracle.hmat_matvec(f, 0.5, X[:, j], -1.0, Y0[:, j], threads=4, transpose=tr)
            assert rel(Y[:, j], ref) <= TOL, (tr, j)


@pytest.mark.parametrize("mode,scheme,nrhs,block", [("aplr", 0, 4, 4), ("aplr", 1, 7, 4), ("codec", 2, 5, 4),
                                                   ("mp", 0, 2, 4), ("aplr", 0, 11, 8), ("codec", 3, 8, 8),
                                                   ("mp", 1, 3, 8)])
def test_multi_rhs_decode_once(gpu, oracle, mode, scheme, nrhs, block):
    """matmat through the 4- and 8-right-hand-side arenas (every field decoded
    once per block of columns; a short last block padded): each column equals
    the oracle's product (ragged clusters, every leaf kind, alpha / beta)"""
    from cpu_hmatrix import build_small_flat
    from paper_2308_10960_b200.hmatrix import HMatrix
    n = 1100
    f, _ = build_small_flat(n=n, eps=1e-6, scheme=scheme, mode=mode, geometry="sphere")
    H = HMatrix(f.to_product(), nrhs_block=block)
    assert H.nrhs_block == block
    rng = np.random.default_rng(11)
    X = np.asfortranarray(rng.uniform(-1, 1, (n, nrhs)))
    Y0 = np.asfortranarray(rng.standard_normal((n, nrhs)))
    for alpha, beta in ((1.0, 0.0), (-0.7, 1.5)):
        Y = Y0.copy(order="F")
        H.matmat(alpha, X, beta, Y)
        for j in range(nrhs):
            ref = oracle.hmat_matvec(f, alpha, X[:, j], beta, Y0[:, j], threads=4)
            assert rel(Y[:, j], ref) <= TOL, (alpha, beta, j)
    H.close()


@pytest.mark.parametrize("pieces", ["1", "2", "4"])
def test_split_row_blocks(gpu, oracle, monkeypatch, pieces):
    """phase-B row blocks cut into pieces (few blocks per GPU: one rank of a
    block-row partition) whose partial sums k_combine adds, vs whole blocks:
    the same y as the oracle, alpha / beta, R = 1 and the 4-RHS arena"""
    from cpu_hmatrix import build_small_flat
    from paper_2308_10960_b200.hmatrix import HMatrix
    monkeypatch.setenv("HCMX_MAX_PIECES", pieces)
    n = 2048
    f, x = build_small_flat(n=n, eps=1e-6, scheme=0)
    H = HMatrix(f.to_product(), nrhs_block=4)
    y0 = np.random.default_rng(9).standard_normal(n)
    for alpha, beta in ((1.0, 0.0), (0.5, -1.25)):
        y = y0.copy()
        H.matvec(alpha, x, beta, y)
        assert rel(y, oracle.hmat_matvec(f, alpha, x, beta, y0, threads=4)) <= TOL
    X = np.asfortranarray(np.stack([x, -x, 2 * x], 1))
    Y = np.asfortranarray(np.stack([y0, y0, y0], 1))
    H.matmat(0.5, X, -1.25, Y)
    for j, s in enumerate((1.0, -1.0, 2.0)):
        assert rel(Y[:, j], oracle.hmat_matvec(f, 0.5, s * x, -1.25, y0, threads=4)) <= TOL
    H.close()


def test_partition_writes_into_gather_slab(gpu, oracle):
    """the multi-GPU bench step writes a rank's rows straight into its slab of
    the all-gather buffer (y base pointer placed row_begin rows before it):
    the slab equals the rank's rows of the full product and nothing else moves"""
    from cpu_hmatrix import build_small_flat
    from paper_2308_10960_b200._lib import check, lib
    from paper_2308_10960_b200.hmatrix import HMatrix
    import bench
    n = 2048
    f, x = build_small_flat(n=n, eps=1e-6, scheme=0)
    ref = oracle.hmat_matvec(f, 1.0, x, 0.0, np.zeros(n), threads=4)
    world = 2
    parts = bench.partition_rows(f.to_product(), world)  # the library partitioner
    maxlen = max(b - a for a, b in parts)
    gathered = torch.full((maxlen * world,), 7.0, dtype=torch.float64, device="cuda")
    xd = torch.as_tensor(x).cuda()
    for rank, rr in enumerate(parts):
        H = HMatrix(f.to_product(), row_range=rr)
        base = gathered.data_ptr() + (rank * maxlen - rr[0]) * 8
        check(lib().hcmx_gpu_hmat_matvec_device(H._h, 1.0, xd.data_ptr(), 0.0, base,
                                                torch.cuda.current_stream().cuda_stream), "matvec")
        torch.cuda.synchronize()
        H.close()
    g = gathered.cpu().numpy()
    for rank, (a, b) in enumerate(parts):
        slab = g[rank * maxlen: rank * maxlen + (b - a)]
        assert rel(slab, ref[a:b]) <= TOL
        assert (g[rank * maxlen + (b - a): (rank + 1) * maxlen] == 7.0).all()


def test_host_api_pinned_and_pageable_y(gpu, oracle):
    """hcmx_gpu_hmat_matvec with host pointers: a pinned y is written directly by
    the kernels (mapped host memory), a pageable y through the staging copy;
    both equal the oracle, beta != 0 takes the staged path"""
    from cpu_hmatrix import build_small_flat
    from paper_2308_10960_b200._lib import check, lib
    from paper_2308_10960_b200.hmatrix import HMatrix
    n = 2048
    f, x = build_small_flat(n=n, eps=1e-6, scheme=0)
    H = HMatrix(f.to_product())
    xh = torch.as_tensor(x).pin_memory()
    y0 = np.random.default_rng(4).standard_normal(n)
    for beta in (0.0, 0.5):
        ref = oracle.hmat_matvec(f, 1.0, x, beta, y0, threads=4)
        yp = torch.as_tensor(y0.copy()).pin_memory()
        check(lib().hcmx_gpu_hmat_matvec(H._h, 1.0, xh.data_ptr(), beta, yp.data_ptr(), 0), "matvec")
        assert rel(yp.numpy(), ref) <= TOL, beta
        yn = y0.copy()
        H.matvec(1.0, x, beta, yn)
        assert rel(yn, ref) <= TOL, beta
    H.close()


def test_partitioned_handle_single_rank_nccl(gpu, oracle):
    """hcmx_gpu_hmat_create_partitioned with a one-rank NCCL communicator (the
    multi-GPU C-ABI path on one device: local product + the grouped broadcast
    exchange), device and host-pointer calls, and without a communicator"""
    import ctypes as C
    from cpu_hmatrix import build_small_flat
    from paper_2308_10960_b200._lib import check, lib
    from paper_2308_10960_b200.distributed import PartitionedHMatrix
    n = 2048
    f, x = build_small_flat(n=n, eps=1e-6, scheme=0)
    ref = oracle.hmat_matvec(f, 1.0, x, 0.0, np.zeros(n), threads=4)
    uid = (C.c_uint8 * 128)()
    check(lib().hcmx_gpu_nccl_unique_id(uid), "uid")
    comm = C.c_void_p()
    check(lib().hcmx_gpu_nccl_comm_init(1, uid, 0, C.byref(comm)), "comm")
    for c in (comm, None):
        P = PartitionedHMatrix(f.to_product(), c)
        assert P.world == 1 and P.rank == 0 and P.row_range == (0, n)
        y = torch.zeros(n, dtype=torch.float64, device="cuda")
        P.matvec_device(1.0, torch.as_tensor(x).cuda(), 0.0, y)
        torch.cuda.synchronize()
        assert rel(y.cpu().numpy(), ref) <= TOL
        yh = np.zeros(n)
        P.matvec(1.0, x, 0.0, yh)
        assert rel(yh, ref) <= TOL
        P.close()
    check(lib().hcmx_gpu_nccl_comm_destroy(comm), "comm destroy")


@pytest.mark.parametrize("world", [2, 3, 5])
def test_partition_cuts_compose_on_device(gpu, oracle, world):
    """the ranges hcmx_gpu_partition_rows gives (what each rank's partitioned
    handle builds) compose the full product: every rank's slice is exact"""
    from cpu_hmatrix import build_small_flat
    from paper_2308_10960_b200.distributed import partition_rows
    from paper_2308_10960_b200.hmatrix import HMatrix
    n = 2048
    f, x = build_small_flat(n=n, eps=1e-6, scheme=1, geometry="cube", kernel="matern")
    ref = oracle.hmat_matvec(f, 1.0, x, 0.0, np.zeros(n), threads=4)
    fp = f.to_product()
    y = np.full(n, np.nan)
    for a, b in partition_rows(fp, world):
        H = HMatrix(fp, row_range=(a, b))
        H.matvec(1.0, x, 0.0, y)
        H.close()
    assert rel(y, ref) <= TOL


def test_one_handle_two_streams(gpu, oracle):
    """products on one handle issued alternately on two streams (shared device
    scratch): each waits for the previous one, every y is the oracle's"""
    from cpu_hmatrix import build_small_flat
    from paper_2308_10960_b200.hmatrix import HMatrix
    n = 2048
    f, x = build_small_flat(n=n, eps=1e-6, scheme=0)
    H = HMatrix(f.to_product())
    xs = [torch.as_tensor(x * s).cuda() for s in (1.0, -2.0, 0.5, 3.0)]
    refs = [oracle.hmat_matvec(f, 1.0, x * s, 0.0, np.zeros(n), threads=4) for s in (1.0, -2.0, 0.5, 3.0)]
    streams = [torch.cuda.Stream(), torch.cuda.Stream()]
    ys = [torch.zeros(n, dtype=torch.float64, device="cuda") for _ in xs]
    torch.cuda.synchronize()
    for rep in range(5):
        for i, (xd, yd) in enumerate(zip(xs, ys)):
            st = streams[i % 2]
            H.matvec_device(1.0, xd, 0.0, yd, stream=st.cuda_stream)
    torch.cuda.synchronize()
    for yd, r in zip(ys, refs):
        assert rel(yd.cpu().numpy(), r) <= TOL
    H.close()


@pytest.mark.parametrize("block", [4, 8])
def test_multi_rhs_transposed(gpu, oracle, block):
    """M^T with several right-hand sides through the transposed handle's block
    arena (4 or 8 columns decoded once): each column equals the oracle's
    transposed product"""
    from cpu_hmatrix import build_small_flat
    from paper_2308_10960_b200.hmatrix import HMatrix
    n = 1100
    f, _ = build_small_flat(n=n, eps=1e-6, scheme=0, mode="aplr", geometry="sphere")
    H = HMatrix(f.to_product(), with_transpose=True, nrhs_block=block)
    rng = np.random.default_rng(21)
    X = np.asfortranarray(rng.uniform(-1, 1, (n, block + 1)))
    Y0 = np.asfortranarray(rng.standard_normal((n, block + 1)))
    Y = Y0.copy(order="F")
    H.matmat(0.75, X, -0.5, Y, transpose=True)
    for j in range(block + 1):
        ref = oracle.hmat_matvec(f, 0.75, X[:, j], -0.5, Y0[:, j], threads=4, transpose=True)
        assert rel(Y[:, j], ref) <= TOL, j
    H.close()
