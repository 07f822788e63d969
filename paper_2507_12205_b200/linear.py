"""`SparseLinear`: a drop-in `torch.nn.Module` for decode-time linear layers whose weight
is stored as EC-CSR (the paper's end-to-end decode use: a GEMV per
weight matrix per generated token, `PAPER.md:773-780`).

y = W x (+ bias) with W on the GPU in the tiled fp16 layout; x of shape [..., K] (each
leading index is one batch-1 SpMV, in order, on the current stream); y keeps x's dtype
unless `out_dtype` is given. CUDA-graph capturable like `spmv`.
"""

from __future__ import annotations

import numpy as np
import torch

from .device import spmv, to_device
from .encoder import convert_csr
from .generators import CsrMatrix


def dense_to_csr(weight) -> CsrMatrix:
    """CSR of the nonzeros of a dense [M, K] weight (numpy or torch), float32 values."""
    w = weight.detach().float().cpu().numpy() if hasattr(weight, "detach") else np.asarray(weight, np.float32)
    if w.ndim != 2:
        raise ValueError("weight must be 2-D [out_features, in_features]")
    m, k = w.shape
    nz = w != 0
    row_ptr = np.concatenate([[0], np.cumsum(nz.sum(axis=1))]).astype(np.int64)
    cols = np.nonzero(nz)[1].astype(np.int64)
    return CsrMatrix(m, k, row_ptr, cols, w[nz].astype(np.float32))


class SparseLinear(torch.nn.Module):
    def __init__(self, ec, bias=None, out_dtype=None, device=None, ordered: bool = False):
        super().__init__()
        self.in_features = int(ec.num_cols)
        self.out_features = int(ec.num_rows)
        self.ordered = ordered
        self.out_dtype = out_dtype
        self.weight_ec = ec  # host container (the encoding; also unpack-able from the device)
        self.W = to_device(ec, device=device)
        if bias is not None:
            b = torch.as_tensor(bias, dtype=torch.float32)
            if b.shape != (self.out_features,):
                raise ValueError(f"bias must have shape ({self.out_features},)")
            self.register_buffer("bias", b.to(f"cuda:{self.W.device_index}"))
        else:
            self.bias = None

    @classmethod
    def from_dense(cls, weight, bias=None, out_dtype=None, device=None, **encode_kw):
        """Encode the nonzeros of a (pruned) dense weight with the native encoder
        (byte-identical to the reference's convert_csr) and upload."""
        return cls(convert_csr(dense_to_csr(weight), **encode_kw), bias=bias, out_dtype=out_dtype,
                   device=device)

    def extra_repr(self) -> str:
        return (f"in_features={self.in_features}, out_features={self.out_features}, "
                f"bias={self.bias is not None}, sets={len(self.weight_ec.sets)}")

    def forward(self, x):
        if x.shape[-1] != self.in_features:
            raise ValueError(f"last dim of x is {x.shape[-1]}, expected {self.in_features}")
        lead = x.shape[:-1]
        xs = x.reshape(-1, self.in_features).to(self.W.x_dtype)
        y = torch.empty(xs.shape[0], self.out_features, dtype=self.W.y_dtype, device=x.device)
        for i in range(xs.shape[0]):  # batch-1 decode: one SpMV per row
            spmv(self.W, xs[i], y=y[i], ordered=self.ordered)
        if self.bias is not None:
            y += self.bias
        return y.to(self.out_dtype or x.dtype).reshape(*lead, self.out_features)
