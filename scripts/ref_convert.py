"""Encode a seeded synthetic matrix with the REFERENCE pipeline (this container only).

    python scripts/ref_convert.py KIND M K SPARSITY SEED OUT.ecsr [--shard I N]

Uses baseline/_ref (the reference package built in place) and
writes `serialize(convert_csr(A, ExtractionConfig()))` with f32 values. These
blobs are the reference side of the native-encoder parity check; they never
travel to the GPU box.
"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "baseline", "_ref", "pkg", "src"))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
from ecsr import core, storage  # noqa: E402
from ecsr.extraction import ExtractionConfig  # noqa: E402

from paper_2507_12205_b200.generators import make_matrix  # noqa: E402
from paper_2507_12205_b200.sharded import row_slice, shard_bounds  # noqa: E402


def main():
    kind, m, k, s, seed, out = sys.argv[1:7]
    a = make_matrix(kind, int(m), int(k), float(s), int(seed), dtype=np.float32)
    if len(sys.argv) > 7 and sys.argv[7] == "--shard":  # row shard I of N (shard-first)
        i, n = int(sys.argv[8]), int(sys.argv[9])
        b = shard_bounds(a.row_ptr, n)
        a = row_slice(a, b[i], b[i + 1])
    ref = core.CsrMatrix(a.num_rows, a.num_cols, a.row_ptr, a.col_idx, a.values)
    t0 = time.perf_counter()
    ec = storage.convert_csr(ref, ExtractionConfig())
    dt = time.perf_counter() - t0
    blob = storage.serialize(ec)
    with open(out + ".tmp", "wb") as fh:
        fh.write(blob)
    os.replace(out + ".tmp", out)
    print(f"{out}: {len(blob)} bytes, convert {dt:.1f}s", flush=True)


if __name__ == "__main__":
    main()
