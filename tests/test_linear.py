"""SparseLinear (paper_2507_12205_b200/linear.py): the decode-time torch module over EC-CSR."""

import numpy as np
import pytest


def test_dense_to_csr_matches_nonzeros():
    from paper_2507_12205_b200.linear import dense_to_csr

    w = np.random.default_rng(0).standard_normal((37, 53)).astype(np.float32)
    w[np.abs(w) < 0.8] = 0
    c = dense_to_csr(w)
    dense = np.zeros_like(w)
    for r in range(c.num_rows):
        dense[r, c.col_idx[c.row_ptr[r]:c.row_ptr[r + 1]]] = c.values[c.row_ptr[r]:c.row_ptr[r + 1]]
    assert np.array_equal(dense, w) and c.row_ptr[-1] == np.count_nonzero(w)


@pytest.mark.gpu
def test_sparse_linear_matches_dense():
    import torch

    from paper_2507_12205_b200.linear import SparseLinear

    g = torch.Generator().manual_seed(1)
    w = torch.randn(384, 512, generator=g) / 512 ** 0.5
    w[w.abs() < w.abs().flatten().kthvalue(w.numel() // 2).values] = 0  # 50 % magnitude pruning
    b = torch.randn(384, generator=g)
    lin = SparseLinear.from_dense(w, bias=b)
    x = torch.randn(3, 512, generator=g).half()
    y = lin(x.cuda())
    assert y.shape == (3, 384) and y.dtype == torch.float16
    ref = x.float() @ w.half().float().T + b
    err = (y.float().cpu() - ref).norm() / ref.norm()
    assert err < 1e-3, err
    y1 = lin(x[0].cuda())
    assert y1.shape == (384,)
