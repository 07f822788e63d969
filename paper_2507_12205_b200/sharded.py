"""Row-sharded multi-GPU EC-CSR SpMV.

Output rows are independent, so a weight matrix is split into contiguous row ranges,
one per rank. Blocks of a whole-matrix encoding pair rows from anywhere in M
(`extraction.py:237-241`), so the split happens BEFORE encoding ("shard-first"): each
rank encodes its own row slice (the native encoder is byte-identical to the reference's
`convert_csr`, so every shard encoding is checkable against the reference), runs the
single-GPU kernel on its shard with x replicated, and one all-gather (NCCL over
NVLink / NVSwitch) assembles y on every rank.

Shard boundaries are byte-balanced: they follow the prefix sum of per-row nonzeros (the
EC-CSR byte proxy), so unevenly pruned matrices still give every rank the same bytes.
The all-gather uses a fixed `max_rows` slot per rank (NCCL all-gather needs equal
sizes) plus an offset table to assemble the global y.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .generators import CsrMatrix


def shard_bounds(row_ptr, nranks: int) -> list[int]:
    """Row boundaries [b_0 = 0, ..., b_n = M] with ~equal nonzeros per shard."""
    row_ptr = np.asarray(row_ptr, dtype=np.int64)
    m = len(row_ptr) - 1
    if nranks < 1:
        raise ValueError("nranks must be >= 1")
    total = int(row_ptr[-1])
    bounds = [0]
    for r in range(1, nranks):
        target = total * r / nranks
        # first row whose prefix reaches the target; equal splits when nnz is uniform
        b = int(np.searchsorted(row_ptr, target, side="left"))
        b = min(max(b, bounds[-1]), m)
        bounds.append(b)
    bounds.append(m)
    return bounds


def row_slice(matrix, lo: int, hi: int) -> CsrMatrix:
    a, b = int(matrix.row_ptr[lo]), int(matrix.row_ptr[hi])
    return CsrMatrix(hi - lo, matrix.num_cols, np.asarray(matrix.row_ptr[lo:hi + 1]) - a,
                     np.asarray(matrix.col_idx[a:b]).copy(), np.asarray(matrix.values[a:b]).copy())


@dataclass
class ShardPlan:
    """Where each rank's rows live in the global y."""

    bounds: list  # per matrix: row boundaries
    names: list

    def rows_of(self, rank: int) -> int:
        return sum(b[rank + 1] - b[rank] for b in self.bounds)

    def max_rows(self) -> int:
        n = len(self.bounds[0]) - 1
        return max(self.rows_of(r) for r in range(n))

    def assemble(self, gathered: np.ndarray) -> list:
        """gathered: [nranks, max_rows] (rank r's stacked shard outputs, padded) ->
        the per-matrix global y vectors."""
        n = len(self.bounds[0]) - 1
        outs = [np.empty(b[-1], dtype=gathered.dtype) for b in self.bounds]
        for r in range(n):
            off = 0
            for i, b in enumerate(self.bounds):
                k = b[r + 1] - b[r]
                outs[i][b[r]:b[r + 1]] = gathered[r, off:off + k]
                off += k
        return outs


def plan_shards(matrices, names, nranks: int) -> ShardPlan:
    return ShardPlan([shard_bounds(m.row_ptr, nranks) for m in matrices], list(names))


def assemble_torch(gathered, plan: ShardPlan):
    """Device-side assembly of the gathered [nranks, max_rows] tensor (index gather)."""
    import torch

    idx = []
    n = len(plan.bounds[0]) - 1
    for i, b in enumerate(plan.bounds):
        for r in range(n):
            off = sum(bb[r + 1] - bb[r] for bb in plan.bounds[:i])
            idx.append(np.arange(b[r + 1] - b[r]) + off + r * plan.max_rows())
    index = torch.from_numpy(np.concatenate(idx)).to(gathered.device)
    return gathered.reshape(-1).index_select(0, index)
