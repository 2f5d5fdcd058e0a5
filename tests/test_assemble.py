"""Setup-time truncation (assemble._svd_batch, host / CPU torch here): the
randomized range finder keeps exactly the ranks a full SVD gives under the
reference's rank rule sigma_k > eps * sigma_0 (lowrank.cpp:14-21), with the
same retained singular values, and reconstructs the block to the truncation
accuracy.  (Rank parity with Eigen's BDCSVD itself is unpinnable: Eigen is
not vendored.)"""
import numpy as np
import pytest
import torch


@pytest.mark.parametrize("kernel,m,n,eps", [("matern", 128, 128, 1e-6), ("laplace", 256, 512, 1e-8),
                                            ("matern", 512, 256, 1e-8), ("laplace", 100, 300, 1e-6)])
def test_randomized_truncation_matches_full_svd(kernel, m, n, eps):
    from paper_2308_10960_b200 import problems
    from paper_2308_10960_b200.assemble import _svd_batch, rank_from_singular_values
    rng = np.random.default_rng(m + n)
    a = torch.as_tensor(rng.uniform(0, 1, (6, m, 3)))
    b = torch.as_tensor(rng.uniform(0, 1, (6, n, 3)) + np.array([2.2, 0.3, 0.0]))
    A = problems.make_kernel(kernel).block(a, b)
    U, S, Vh = _svd_batch(A, eps)
    S_full = torch.linalg.svdvals(A)
    k = rank_from_singular_values(S, eps)
    k_full = rank_from_singular_values(S_full, eps)
    assert (k == k_full).all()
    for i in range(A.shape[0]):
        ki = int(k[i])
        assert torch.allclose(S[i, :ki], S_full[i, :ki], rtol=1e-12, atol=1e-14 * float(S_full[i, 0]))
        R = (U[i, :, :ki] * S[i, :ki]) @ Vh[i, :ki]
        assert float((R - A[i]).norm()) <= 2 * eps * float(A[i].norm()) * max(1.0, ki ** 0.5)
        # orthonormal factors (svd_factors' W, X, lowrank.cpp:76-93)
        assert torch.allclose(U[i, :, :ki].mT @ U[i, :, :ki], torch.eye(ki, dtype=A.dtype), atol=1e-12)
        assert torch.allclose(Vh[i, :ki] @ Vh[i, :ki].mT, torch.eye(ki, dtype=A.dtype), atol=1e-12)
