"""Host setup: cluster tree / block tree restating clustering.cpp, and the
synthetic problems (CPU only)."""
import numpy as np
import pytest

from paper_2308_10960_b200 import problems, tree


@pytest.mark.parametrize("geometry,n", [("fibonacci", 8192), ("cube", 3000), ("sphere", 777)])
def test_cluster_tree_partitions(geometry, n):
    pts = problems.make_points(geometry, n, 3)
    ct = tree.build_cluster_tree(pts, 64)
    assert sorted(ct.i2e.tolist()) == list(range(n))
    assert (ct.e2i[ct.i2e] == np.arange(n)).all()
    leaf = ct.is_leaf
    assert (ct.last[leaf] - ct.first[leaf] <= 64).all()
    # children split the parent's range at first + size/2 (clustering.cpp:70)
    for v in np.nonzero(~leaf)[0]:
        c0, c1 = ct.child[v]
        mid = ct.first[v] + (ct.last[v] - ct.first[v]) // 2
        assert (ct.first[c0], ct.last[c0], ct.first[c1], ct.last[c1]) == (ct.first[v], mid, mid, ct.last[v])
        # halves separated along the longest axis
        ax = np.argmax(ct.hi[v] - ct.lo[v])
        p = pts[ct.i2e]
        assert p[ct.first[c0]: ct.last[c0], ax].max() <= p[ct.first[c1]: ct.last[c1], ax].min()


@pytest.mark.parametrize("n", [1024, 1000])
def test_block_tree_tiles_matrix_once(n):
    pts = problems.make_points("fibonacci", n, 1)
    ct = tree.build_cluster_tree(pts, 64)
    lv = tree.build_block_tree(ct, ct, 2.0)
    cover = np.zeros((n, n), np.int32)
    for r0, r1, c0, c1 in zip(lv.row0, lv.row1, lv.col0, lv.col1):
        cover[r0:r1, c0:c1] += 1
    assert (cover == 1).all()
    # admissible leaves satisfy min(diam) <= eta * dist; dense leaves are leaf x leaf
    d = ct.diameter()
    for t, s, a in zip(lv.row, lv.col, lv.admissible):
        gap = np.maximum(0, np.maximum(ct.lo[s] - ct.hi[t], ct.lo[t] - ct.hi[s]))
        dist = np.sqrt((gap ** 2).sum())
        assert a == (min(d[t], d[s]) <= 2.0 * dist)
        if not a:
            assert ct.is_leaf[t] or ct.is_leaf[s]


def test_preorder_rowmajor_children():
    """for_each_leaf preorder (clustering.cpp:159-166): recursion order 2i+j"""
    pts = problems.make_points("fibonacci", 2048, 1)
    ct = tree.build_cluster_tree(pts, 64)
    lv = tree.build_block_tree(ct, ct, 2.0)
    out = []

    def rec(t, s):
        d = ct.diameter()
        gap = np.maximum(0, np.maximum(ct.lo[s] - ct.hi[t], ct.lo[t] - ct.hi[s]))
        adm = min(d[t], d[s]) <= 2.0 * np.sqrt((gap ** 2).sum())
        if adm or ct.is_leaf[t] or ct.is_leaf[s]:
            out.append((t, s))
            return
        for i in range(2):
            for j in range(2):
                rec(ct.child[t, i], ct.child[s, j])
    rec(0, 0)
    assert out == list(zip(lv.row.tolist(), lv.col.tolist()))


def test_config1_structure_matches_survey():
    """config 1 has ~1342 dense 64x64 leaves, ~2700 lowrank, depth 8"""
    c = problems.config(1)
    pts = problems.make_points(c["geometry"], c["n"], 1)
    ct = tree.build_cluster_tree(pts, c["leaf"])
    lv = tree.build_block_tree(ct, ct, c["eta"])
    assert ct.depth() == 8
    nd = int((~lv.admissible).sum())
    assert 1300 <= nd <= 1400 and 2600 <= int(lv.admissible.sum()) <= 2800
    assert ((lv.row1 - lv.row0)[~lv.admissible] == 64).all()


def test_kernels():
    import torch
    a = torch.tensor([[0.0, 0.0, 0.0], [1.0, 0.0, 0.0]], dtype=torch.float64)
    L = problems.Laplace().block(a, a)
    assert L[0, 0] == 0.0 and abs(L[0, 1] - 1 / (4 * np.pi)) < 1e-16
    M = problems.Matern15(0.1, 1.0).block(a, a)
    t = np.sqrt(3.0) / 0.1
    assert M[0, 0] == 1.0 and abs(M[0, 1] - (1 + t) * np.exp(-t)) < 1e-16
    p = problems.fibonacci_sphere(100)
    assert np.allclose(np.linalg.norm(p, axis=1), 1.0)
