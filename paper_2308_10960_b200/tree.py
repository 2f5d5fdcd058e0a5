"""Cluster tree and block tree (host setup; not on the hot path).

Restates /root/reference/proj/src/clustering.cpp in vectorised numpy:
  * cluster tree: split along the longest bounding-box axis into two
    cardinality-balanced halves (mid = first + size/2) until size <= n_min
    (clustering.cpp:51-78); the permutation i2e/e2i is rewritten (105-108)
  * admissibility: min(diam t, diam s) <= eta * dist(t, s) on bounding boxes
    (clustering.cpp:16-30, 115-118)
  * block tree: a node is a leaf when admissible or either cluster is a leaf;
    children in row-major order 2i+j (clustering.cpp:134-146)
  * leaves are returned in for_each_leaf preorder (clustering.cpp:159-166)

The median split uses numpy's introselect instead of std::nth_element, so the
order of indices inside a half can differ from a libstdc++ build; the halves
(and hence the tree) are the same for distinct coordinates.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass
class ClusterTree:
    first: np.ndarray     # int64 [nodes]
    last: np.ndarray
    lo: np.ndarray        # float64 [nodes, 3]
    hi: np.ndarray
    child: np.ndarray     # int64 [nodes, 2], -1 for leaves
    i2e: np.ndarray       # internal -> external
    e2i: np.ndarray
    n_min: int

    @property
    def is_leaf(self):
        return self.child[:, 0] < 0

    def diameter(self):
        return np.sqrt(((self.hi - self.lo) ** 2).sum(axis=1))

    def depth(self) -> int:
        d = np.zeros(self.first.size, dtype=np.int64)
        for v in range(self.first.size):  # parents precede children
            for c in self.child[v]:
                if c >= 0:
                    d[c] = d[v] + 1
        return int(d.max()) + 1

    def leaf_count(self) -> int:
        return int(self.is_leaf.sum())


def build_cluster_tree(points: np.ndarray, n_min: int = 64) -> ClusterTree:
    """clustering.cpp:94-110"""
    if n_min <= 0:
        raise ValueError("build_cluster_tree: n_min must be positive")
    pts = np.ascontiguousarray(points, dtype=np.float64)
    n = pts.shape[0]
    order = np.arange(n, dtype=np.int64)
    first, last, lo, hi, child = [], [], [], [], []
    stack = [(0, n, -1, 0)]
    while stack:
        f, l, parent, slot = stack.pop()
        v = len(first)
        if parent >= 0:
            child[parent][slot] = v
        sub = order[f:l]
        p = pts[sub]
        blo = p.min(axis=0) if l > f else np.full(3, np.inf)
        bhi = p.max(axis=0) if l > f else np.full(3, -np.inf)
        first.append(f); last.append(l); lo.append(blo); hi.append(bhi); child.append([-1, -1])
        if l - f <= n_min:
            continue
        axis = int(np.argmax(bhi - blo))  # first longest axis (strict '>' scan, cpp:63-69)
        mid = f + (l - f) // 2
        part = np.argpartition(p[:, axis], mid - f, kind="introselect")
        order[f:l] = sub[part]
        # children pushed so that child 0 is expanded first (preorder numbering)
        stack.append((mid, l, v, 1))
        stack.append((f, mid, v, 0))
    i2e = order
    e2i = np.empty(n, dtype=np.int64)
    e2i[i2e] = np.arange(n)
    return ClusterTree(np.array(first, np.int64), np.array(last, np.int64), np.array(lo),
                       np.array(hi), np.array(child, np.int64), i2e, e2i, n_min)


@dataclass
class BlockLeaves:
    """leaf blocks of a block tree in for_each_leaf preorder"""
    row: np.ndarray        # cluster ids
    col: np.ndarray
    admissible: np.ndarray
    row0: np.ndarray
    row1: np.ndarray
    col0: np.ndarray
    col1: np.ndarray

    def __len__(self):
        return self.row.size


def _bbox_distance(lo_a, hi_a, lo_b, hi_b):
    gap = np.maximum(0.0, np.maximum(lo_b - hi_a, lo_a - hi_b))
    return np.sqrt((gap ** 2).sum(axis=1))


def build_block_tree(rows: ClusterTree, cols: ClusterTree, eta: float = 2.0) -> BlockLeaves:
    """clustering.cpp:122-157 with standard admissibility (level-synchronous)."""
    dr, dc = rows.diameter(), cols.diameter()
    t = np.array([0], np.int64)
    s = np.array([0], np.int64)
    key = np.array([0], np.int64)
    depth = 0
    out = []
    while t.size:
        adm = np.minimum(dr[t], dc[s]) <= eta * _bbox_distance(rows.lo[t], rows.hi[t], cols.lo[s], cols.hi[s])
        leaf = adm | rows.is_leaf[t] | cols.is_leaf[s]
        out.append((t[leaf], s[leaf], adm[leaf], key[leaf], depth))
        t, s, key = t[~leaf], s[~leaf], key[~leaf]
        if not t.size:
            break
        nt, ns, nk = [], [], []
        for i in range(2):
            for j in range(2):
                nt.append(rows.child[t, i]); ns.append(cols.child[s, j]); nk.append(key * 4 + 2 * i + j)
        # order inside a level is irrelevant: preorder comes from the padded keys
        t, s, key = np.concatenate(nt), np.concatenate(ns), np.concatenate(nk)
        depth += 1
    maxd = max(d for *_, d in out)
    T = np.concatenate([o[0] for o in out]); S = np.concatenate([o[1] for o in out])
    A = np.concatenate([o[2] for o in out])
    K = np.concatenate([o[3] * (4 ** (maxd - o[4])) for o in out])
    perm = np.argsort(K, kind="stable")
    T, S, A = T[perm], S[perm], A[perm]
    return BlockLeaves(T, S, A, rows.first[T], rows.last[T], cols.first[S], cols.last[S])
