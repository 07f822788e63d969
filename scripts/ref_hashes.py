"""Pin config-scale native encodings to the REFERENCE encoder (this container only).

    python scripts/ref_hashes.py [--jobs N] [--only NAME ...]

For every matrix in tests/golden/ref_hashes_cases.py (the bench layer and the
BASELINE.json config shapes the GPU tests run), encode the seeded synthetic matrix with
the reference's own `storage.convert_csr(A, ExtractionConfig())` (baseline/_ref, the
reference package built in place; scripts/ref_convert.py) and record
sha256(storage.serialize(ec)) with its size in tests/golden/ref_hashes.json. The blobs
themselves are too large to commit (40-110 MB each); tests/test_ref_hashes.py
re-encodes each matrix natively and compares hashes. Bench matrices whose reference
blob already sits in cache/ (scripts/make_cache.sh) are hashed from there.
"""
import argparse
import concurrent.futures as cf
import hashlib
import json
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))
from ref_hashes_cases import CASES, case_name  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden", "ref_hashes.json")


def sha(path):
    h = hashlib.sha256()
    with open(path, "rb") as fh:
        for chunk in iter(lambda: fh.read(1 << 24), b""):
            h.update(chunk)
    return h.hexdigest(), os.path.getsize(path)


def one(case):
    name = case_name(case)
    kind, m, k, s, seed, shard = case
    cached = os.path.join(ROOT, "cache", f"{kind}_{m}x{k}_s{s}_seed{seed}.ecsr")
    if shard is None and os.path.exists(cached):
        digest, size = sha(cached)
        return name, {"sha256": digest, "bytes": size, "source": "cache (scripts/make_cache.sh)"}
    out = f"/tmp/refhash_{name}.ecsr"
    t0 = time.time()
    cmd = [sys.executable, os.path.join(ROOT, "scripts", "ref_convert.py"), kind, str(m), str(k),
           str(s), str(seed), out]
    if shard is not None:
        cmd += ["--shard", str(shard[0]), str(shard[1])]
    subprocess.run(cmd, check=True, stdout=subprocess.DEVNULL)
    digest, size = sha(out)
    os.remove(out)
    return name, {"sha256": digest, "bytes": size, "reference_convert_s": round(time.time() - t0, 1)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--jobs", type=int, default=os.cpu_count())
    ap.add_argument("--only", nargs="*")
    args = ap.parse_args()
    table = {}
    if os.path.exists(OUT):
        with open(OUT) as fh:
            table = json.load(fh)
    todo = [c for c in CASES if (not args.only or case_name(c) in args.only) and case_name(c) not in table]
    with cf.ThreadPoolExecutor(args.jobs) as ex:
        for name, rec in ex.map(one, todo):
            table[name] = rec
            print(name, rec, flush=True)
            with open(OUT + ".tmp", "w") as fh:
                json.dump(dict(sorted(table.items())), fh, indent=1)
            os.replace(OUT + ".tmp", OUT)


if __name__ == "__main__":
    main()
