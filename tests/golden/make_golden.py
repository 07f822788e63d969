"""Generate the golden fixtures from the REFERENCE package (run in the dev container).

    python tests/golden/make_golden.py

Requires the reference built in place at baseline/_ref/pkg; the
outputs are committed so the GPU box (no reference) can check against them.

Per case `<name>.npz` holds:
  blob      serialize(convert_csr(A, cfg)) of the f64 container (reference encoder)
  x         f64 input vector
  y64       reference spmv_ec(ec_f64, x) (compiled backend, executor.py:80-96)
  y32       reference spmv_ec(ec_f32, x_f32)
  y16       reference spmv_ec on fp16-rounded values and x, f32 arithmetic: the
            strict target of the FP16-in / FP32-accumulate GPU kernel
  yoracle   core.spmv_oracle(A, x) in f64 (core.py:223-235)
  report_keys/report_vals  storage_report(ec, value_bits=16).components
plus `manifest.json` with the case parameters and the sha256 of each blob.
"""

from __future__ import annotations

import hashlib
import zlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, os.path.join(ROOT, "baseline", "_ref", "pkg", "src"))
sys.path.insert(0, ROOT)

from ecsr import _kernels, core, executor, storage  # noqa: E402
from ecsr.extraction import ExtractionConfig  # noqa: E402

from paper_2507_12205_b200.generators import make_matrix  # noqa: E402


def corpus_params(i):
    """The reference acceptance corpus mix (pkg/tests/test_acceptance.py:51-67)."""
    rng = np.random.default_rng(1000 + i)
    sparsity = (0.5, 0.7, 0.8, 0.9)[i % 4]
    bits = (8, 4)[i % 2]
    if i % 10 == 9:
        lo, hi, wv = 192, 512, (32, 4)
    elif i % 10 in (7, 8):
        lo, hi, wv = 64, 192, (8, 2)
    else:
        lo, hi = 8, 64
        wv = [(2, 2), (4, 1), (2, 1), (4, 2)][i % 4]
    m = int(rng.integers(lo, hi + 1))
    k = int(rng.integers(lo, hi + 1))
    return m, k, sparsity, bits, wv


def cases():
    out = []
    # KAT: two identical rows over {2,4,5,6} (pkg/tests/test_storage.py:112-132)
    rows, cols = [0] * 4 + [1] * 4, [2, 4, 5, 6] * 2
    out.append(("kat_two_row_block", core.csr_from_coo(2, 7, rows, cols, [1.0] * 8),
                ExtractionConfig(2, 2, 8), {"kind": "kat"}))
    out.append(("kat_identity6", core.csr_from_coo(6, 6, range(6), range(6), [1.0] * 6),
                ExtractionConfig(2, 2, 8), {"kind": "kat"}))
    # explicit stored zero (pkg/tests/test_storage.py:162-166)
    out.append(("kat_explicit_zero", core.csr_from_coo(2, 4, [0, 0, 1], [0, 2, 1], [0.0, 3.0, 4.0]),
                ExtractionConfig(2, 2, 8), {"kind": "kat"}))
    # the reference corpus, every 7th case (W in {2,4,8,32}, v in {1,2,4}, B in {4,8})
    for i in range(0, 200, 7):
        m, k, s, bits, (w, v) = corpus_params(i)
        out.append((f"corpus_{i:03d}", core.generate_uniform(m, k, s, seed=i),
                    ExtractionConfig(w, v, bits), {"kind": "corpus", "index": i}))
    # W = 32 / v = 4 default-config cases for the tiled kernel, all generators
    for kind, m, k, s, seed, bits in (
        ("uniform", 256, 256, 0.5, 11, 8), ("uniform", 200, 300, 0.7, 12, 8),
        ("magnitude", 384, 256, 0.5, 13, 8), ("magnitude", 256, 512, 0.7, 14, 8),
        ("planted", 512, 384, 0.5, 15, 8), ("planted", 256, 256, 0.6, 16, 8),
        ("uniform", 256, 256, 0.5, 17, 4), ("uniform", 160, 256, 0.9, 18, 16),
    ):
        a = make_matrix(kind, m, k, s, seed, dtype=np.float64)
        ref = core.CsrMatrix(a.num_rows, a.num_cols, a.row_ptr, a.col_idx, a.values)
        out.append((f"{kind}_{m}x{k}_s{s}_b{bits}_seed{seed}", ref,
                    ExtractionConfig(32, 4, bits),
                    {"kind": kind, "m": m, "k": k, "s": s, "seed": seed}))
    # edge shapes of SURVEY.md §8(a) a15(6): non-power-of-two warps (lane padding to
    # lanes_p2, _speedups.pyx:91-93, 120-127; W = 3 is pkg/tests/test_storage.py:99),
    # v = 2 at W = 32 (generic kernel), a single lane, B = 16 with v = 1
    for kind, m, k, s, seed, (w, v, bits) in (
        ("uniform", 96, 120, 0.6, 21, (3, 1, 8)), ("planted", 128, 150, 0.5, 22, (3, 2, 8)),
        ("uniform", 80, 200, 0.7, 23, (5, 2, 4)), ("planted", 160, 160, 0.6, 24, (6, 4, 8)),
        ("uniform", 100, 333, 0.8, 25, (7, 1, 16)), ("planted", 256, 256, 0.5, 26, (32, 2, 8)),
        ("magnitude", 192, 300, 0.6, 27, (32, 1, 16)), ("uniform", 48, 64, 0.5, 28, (1, 1, 8)),
        ("planted", 200, 256, 0.6, 29, (12, 3, 8)),
    ):
        a = make_matrix(kind, m, k, s, seed, dtype=np.float64)
        ref = core.CsrMatrix(a.num_rows, a.num_cols, a.row_ptr, a.col_idx, a.values)
        out.append((f"edge_{kind}_{m}x{k}_w{w}v{v}b{bits}_seed{seed}", ref,
                    ExtractionConfig(w, v, bits),
                    {"kind": kind, "m": m, "k": k, "s": s, "seed": seed}))
    return out


def spmv(ec, x):
    return executor.spmv_ec(ec, x, validate=True)


def main():
    """`make_golden.py [NAME_PREFIX ...]`: regenerate only the matching cases (the rest
    of the manifest is kept as is)."""
    _kernels.use_backend("compiled")
    only = sys.argv[1:]
    manifest = []
    if only:
        with open(os.path.join(HERE, "manifest.json")) as fh:
            manifest = [c for c in json.load(fh) if not any(c["name"].startswith(p) for p in only)]
    for name, mat, cfg, meta in cases():
        if only and not any(name.startswith(p) for p in only):
            continue
        ec = storage.convert_csr(mat, cfg, dtype=np.float64)
        blob = storage.serialize(ec)
        x = np.random.default_rng(zlib.crc32(name.encode())).uniform(-1, 1, mat.num_cols)
        ec32 = ec.astype(np.float32)
        x32 = x.astype(np.float32)
        ec16 = ec.astype(np.float16).astype(np.float32)
        x16 = x.astype(np.float16).astype(np.float32)
        rep = storage.storage_report(ec, value_bits=16)
        np.savez_compressed(
            os.path.join(HERE, name + ".npz"),
            blob=np.frombuffer(blob, dtype=np.uint8), x=x, y64=spmv(ec, x), y32=spmv(ec32, x32),
            y16=spmv(ec16, x16), yoracle=core.spmv_oracle(mat, x),
            report_keys=np.array(list(rep.components.keys())),
            report_vals=np.array(list(rep.components.values()), dtype=np.int64),
        )
        manifest.append({"name": name, "warp": cfg.warp_size, "vector": cfg.vector_size,
                         "delta_bits": cfg.delta_bits, "rows": mat.num_rows,
                         "cols": mat.num_cols, "nnz": mat.nnz, "sets": len(ec.sets),
                         "sha256": hashlib.sha256(blob).hexdigest(), **meta})
    with open(os.path.join(HERE, "manifest.json"), "w") as fh:
        json.dump(manifest, fh, indent=1)
    print(f"wrote {len(manifest)} golden cases")


if __name__ == "__main__":
    main()
