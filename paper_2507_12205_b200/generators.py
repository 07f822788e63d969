"""Seeded synthetic weight matrices for the EC-CSR SpMV hot path.

Three generators, all deterministic for a given seed and returning a CSR
triple in the reference's `CsrMatrix` shape (`pkg/src/ecsr/core.py:24-93`:
int64 row_ptr/col_idx, strictly increasing columns per row, f32/f64 values):

* `generate_uniform` -- the reference's own Bernoulli generator, restated
  draw-for-draw (`pkg/src/ecsr/core.py:198-220`) so the GPU box can rebuild the
  reference's test matrices without the reference installed.
* `magnitude_pruned` -- random-init LLM weights N(0, 1/K) pruned per output row
  to the top-k magnitudes (Wanda/SparseGPT-style per-row groups). Not in the
  reference; BASELINE.json `north_star` asks for it.
* `planted_blocks` -- g-row groups (g in {8, 4, 2}) sharing one Bernoulli column
  set, plus an unstructured remainder. Random pruning exposes few multi-row
  blocks, so this exercises the g >= 4 kernels (north_star).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass(eq=False)
class CsrMatrix:
    """Duck-type mirror of `ecsr.core.CsrMatrix` (`pkg/src/ecsr/core.py:24-93`)."""

    num_rows: int
    num_cols: int
    row_ptr: np.ndarray
    col_idx: np.ndarray
    values: np.ndarray

    def __post_init__(self):
        self.row_ptr = np.ascontiguousarray(self.row_ptr, dtype=np.int64)
        self.col_idx = np.ascontiguousarray(self.col_idx, dtype=np.int64)
        self.values = np.ascontiguousarray(self.values)
        if self.values.dtype not in (np.float32, np.float64):
            self.values = self.values.astype(np.float64)
        if self.row_ptr.shape != (self.num_rows + 1,):
            raise ValueError("row_ptr must have num_rows + 1 entries")
        if self.row_ptr[0] != 0 or self.row_ptr[-1] != len(self.col_idx):
            raise ValueError("row_ptr must start at 0 and end at nnz")
        if len(self.col_idx) != len(self.values):
            raise ValueError("col_idx and values must have equal length")

    @property
    def nnz(self) -> int:
        return int(self.row_ptr[-1])

    def astype(self, dtype) -> "CsrMatrix":
        return CsrMatrix(self.num_rows, self.num_cols, self.row_ptr.copy(),
                         self.col_idx.copy(), self.values.astype(dtype))

    def row_slice(self, lo: int, hi: int) -> "CsrMatrix":
        """Rows [lo, hi) as their own matrix (the shard-first split)."""
        a, b = int(self.row_ptr[lo]), int(self.row_ptr[hi])
        return CsrMatrix(hi - lo, self.num_cols, self.row_ptr[lo:hi + 1] - a,
                         self.col_idx[a:b].copy(), self.values[a:b].copy())

    def to_dense(self) -> np.ndarray:
        dense = np.zeros((self.num_rows, self.num_cols), dtype=self.values.dtype)
        rows = np.repeat(np.arange(self.num_rows), np.diff(self.row_ptr))
        dense[rows, self.col_idx] = self.values
        return dense


def generate_uniform(num_rows, num_cols, sparsity, seed, dtype=np.float64) -> CsrMatrix:
    """The matrix of `ecsr.core.generate_uniform` (`pkg/src/ecsr/core.py:198-220`),
    bit for bit: every cell is kept with probability 1 - sparsity by one uniform draw in
    row-major order (one PCG64 stream, `default_rng(seed)`), then the kept cells' values
    are drawn from U(-1, 1) in the same order. Only the order of the draws matters, so
    the cells are drawn here in blocks of whole rows of about 16 M cells."""
    if not 0.0 <= sparsity < 1.0:
        raise ValueError("sparsity must lie in [0, 1)")
    rng = np.random.default_rng(seed)
    keep_below = 1.0 - sparsity
    rows_per_draw = max(1, (1 << 24) // max(num_cols, 1))
    row_ptr = np.zeros(num_rows + 1, dtype=np.int64)
    cols = []
    for r0 in range(0, num_rows, rows_per_draw):
        r1 = min(num_rows, r0 + rows_per_draw)
        kept = rng.random((r1 - r0, num_cols)) < keep_below
        row_ptr[r0 + 1:r1 + 1] = kept.sum(axis=1)
        cols.append(np.flatnonzero(kept) % max(num_cols, 1))
    np.cumsum(row_ptr, out=row_ptr)
    col_idx = np.concatenate(cols).astype(np.int64) if cols else np.empty(0, dtype=np.int64)
    values = rng.uniform(-1.0, 1.0, size=col_idx.size).astype(dtype)
    return CsrMatrix(num_rows, num_cols, row_ptr, col_idx, values)


_ROW_CHUNK_ELEMS = 1 << 24


def magnitude_pruned(num_rows, num_cols, sparsity, seed, dtype=np.float32) -> CsrMatrix:
    """W ~ N(0, 1/K) (f32 draws), keep the top round((1-s)*K) |w| in every row.

    Rows are drawn in fixed chunks of `_ROW_CHUNK_ELEMS // K` rows, so peak memory
    stays small and the matrix depends only on (shape, sparsity, seed).
    """
    if not 0.0 <= sparsity < 1.0:
        raise ValueError("sparsity must lie in [0, 1)")
    keep = num_cols - int(round(sparsity * num_cols))
    rng = np.random.default_rng(seed)
    scale = np.float32(1.0 / np.sqrt(num_cols))
    chunk = max(1, _ROW_CHUNK_ELEMS // max(num_cols, 1))
    col_parts, val_parts = [], []
    for start in range(0, num_rows, chunk):
        stop = min(start + chunk, num_rows)
        w = rng.standard_normal((stop - start, num_cols), dtype=np.float32) * scale
        if keep == num_cols:
            idx = np.broadcast_to(np.arange(num_cols), w.shape)
        elif keep == 0:
            idx = np.empty((stop - start, 0), dtype=np.int64)
        else:
            idx = np.argpartition(-np.abs(w), keep - 1, axis=1)[:, :keep]
            idx = np.sort(idx, axis=1)
        col_parts.append(idx.reshape(-1).astype(np.int64))
        val_parts.append(np.take_along_axis(w, idx, axis=1).reshape(-1))
    col_idx = np.concatenate(col_parts) if col_parts else np.empty(0, dtype=np.int64)
    values = (np.concatenate(val_parts) if val_parts else np.empty(0, np.float32)).astype(dtype)
    row_ptr = np.arange(num_rows + 1, dtype=np.int64) * keep
    return CsrMatrix(num_rows, num_cols, row_ptr, col_idx, values)


def planted_blocks(num_rows, num_cols, sparsity, seed, groups=(8, 4, 2),
                   planted_frac=0.5, dtype=np.float32) -> CsrMatrix:
    """Planted multi-granularity structure plus an unstructured remainder.

    A `planted_frac` share of the rows (chosen by a seeded permutation) is split
    evenly between the group sizes in `groups`; each group of g rows shares one
    Bernoulli(1 - sparsity) column set. Every other row draws its own set.
    Values are N(0, 1/K) in f32.
    """
    if not 0.0 <= sparsity < 1.0:
        raise ValueError("sparsity must lie in [0, 1)")
    rng = np.random.default_rng(seed)
    density = 1.0 - sparsity
    perm = rng.permutation(num_rows)
    n_planted = int(planted_frac * num_rows)
    share = n_planted // max(len(groups), 1)
    group_of = np.full(num_rows, -1, dtype=np.int64)
    pos = 0
    gid = 0
    for g in groups:
        for _ in range(share // g):
            group_of[perm[pos:pos + g]] = gid
            pos += g
            gid += 1
    group_masks = rng.random((gid, num_cols)) < density if gid else None
    scale = np.float32(1.0 / np.sqrt(num_cols))
    cols, counts = [], np.zeros(num_rows, dtype=np.int64)
    for r in range(num_rows):
        if group_of[r] >= 0:
            c = np.flatnonzero(group_masks[group_of[r]])
        else:
            c = np.flatnonzero(rng.random(num_cols) < density)
        cols.append(c)
        counts[r] = c.size
    col_idx = np.concatenate(cols).astype(np.int64) if cols else np.empty(0, np.int64)
    values = (rng.standard_normal(col_idx.size, dtype=np.float32) * scale).astype(dtype)
    row_ptr = np.zeros(num_rows + 1, dtype=np.int64)
    np.cumsum(counts, out=row_ptr[1:])
    return CsrMatrix(num_rows, num_cols, row_ptr, col_idx, values)


def make_matrix(kind: str, num_rows: int, num_cols: int, sparsity: float, seed: int,
                dtype=np.float32) -> CsrMatrix:
    if kind == "uniform":
        return generate_uniform(num_rows, num_cols, sparsity, seed, dtype=dtype)
    if kind == "magnitude":
        return magnitude_pruned(num_rows, num_cols, sparsity, seed, dtype=dtype)
    if kind == "planted":
        return planted_blocks(num_rows, num_cols, sparsity, seed, dtype=dtype)
    raise ValueError(f"unknown generator {kind!r}")
