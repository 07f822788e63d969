"""Config-scale native encodings are byte-identical to the REFERENCE encoder's.

tests/golden/ref_hashes.json holds sha256(storage.serialize(convert_csr(A))) of the
reference's own pipeline (scripts/ref_hashes.py, baseline/_ref) for the bench layer and
the BASELINE.json config shapes the -m gpu tests run (tests/golden/ref_hashes_cases.py).
Here every matrix is re-encoded by the native encoder and its serialized blob hashed:
equal hashes = the same bytes (SURVEY.md §8(f) #1 gate, at full size). The native
encoder is OpenMP-parallel; matrices above 20 M cells are marked `slow` (the whole set
takes ~6 min on 8 cores) and run with ECSR_RUN_SLOW=1 (log: profiles/round2/).
"""

import hashlib
import json
import os
import sys

import numpy as np
import pytest

from conftest import GOLDEN
from paper_2507_12205_b200 import container as C
from paper_2507_12205_b200.encoder import convert_csr
from paper_2507_12205_b200.generators import make_matrix
from paper_2507_12205_b200.sharded import row_slice, shard_bounds

sys.path.insert(0, GOLDEN)
from ref_hashes_cases import CASES, case_name  # noqa: E402

with open(os.path.join(GOLDEN, "ref_hashes.json")) as fh:
    HASHES = json.load(fh)


def test_every_case_is_pinned():
    missing = [case_name(c) for c in CASES if case_name(c) not in HASHES]
    assert not missing, f"run scripts/ref_hashes.py for {missing}"


def _param(c):
    slow = c[1] * c[2] // (c[5][1] if c[5] else 1) > 20_000_000
    return pytest.param(c, id=case_name(c), marks=[pytest.mark.slow] if slow else [])


@pytest.mark.parametrize("case", [_param(c) for c in CASES if case_name(c) in HASHES])
def test_native_encoding_hash_equals_reference(case):
    kind, m, k, s, seed, shard = case
    a = make_matrix(kind, m, k, s, seed, dtype=np.float32)
    if shard is not None:
        b = shard_bounds(a.row_ptr, shard[1])
        a = row_slice(a, b[shard[0]], b[shard[0] + 1])
    blob = C.serialize(convert_csr(a))
    want = HASHES[case_name(case)]
    assert len(blob) == want["bytes"]
    assert hashlib.sha256(blob).hexdigest() == want["sha256"]
