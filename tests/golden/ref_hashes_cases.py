"""Matrices whose REFERENCE encodings are pinned by sha256 in ref_hashes.json.

(kind, rows, cols, sparsity, seed, shard) with shard = (index, count) of a byte-balanced
row shard (sharded.shard_bounds) or None. The bench layer (bench.py MATRICES) and the
BASELINE.json config shapes the -m gpu tests run (tests/test_gpu_configs.py).
Hashes are made by scripts/ref_hashes.py with the reference's convert_csr.
"""

BENCH = [
    ("magnitude", 4096, 4096, 0.5, 101, None),
    ("magnitude", 4096, 4096, 0.5, 102, None),
    ("magnitude", 4096, 4096, 0.5, 103, None),
    ("magnitude", 4096, 4096, 0.5, 104, None),
    ("magnitude", 11008, 4096, 0.5, 105, None),
    ("magnitude", 11008, 4096, 0.5, 106, None),
    ("magnitude", 4096, 11008, 0.5, 107, None),
]
CONFIGS = [
    # config 1: single 4096x4096 @50 %
    ("magnitude", 4096, 4096, 0.5, 1, None),
    # config 2: LLaMA-7B q / up / down at 60 and 70 % (50 % is the bench layer)
    ("magnitude", 4096, 4096, 0.6, 201, None),
    ("magnitude", 4096, 4096, 0.7, 202, None),
    ("magnitude", 11008, 4096, 0.6, 203, None),
    ("magnitude", 11008, 4096, 0.7, 204, None),
    ("magnitude", 4096, 11008, 0.6, 205, None),
    ("magnitude", 4096, 11008, 0.7, 206, None),
    # config 3: LLaMA-2-13B planted
    ("planted", 5120, 5120, 0.5, 31, None),
    ("planted", 13824, 5120, 0.6, 32, (3, 8)),
    # config 4: OPT-30B @70 %
    ("magnitude", 7168, 7168, 0.7, 33, None),
    ("magnitude", 7168, 28672, 0.7, 34, (0, 8)),
    # config 5: LLaMA-2-70B, row-sharded
    ("magnitude", 28672, 8192, 0.5, 35, (5, 8)),
    ("magnitude", 8192, 8192, 0.5, 36, None),
]
# the OPT-30B layer bench.py times next to the headline (fc1 / fc2 unsharded take the
# reference hours to encode; their shards above pin the same code path)
OPT30B = [
    ("magnitude", 7168, 7168, 0.7, 401, None),
    ("magnitude", 7168, 7168, 0.7, 402, None),
    ("magnitude", 7168, 7168, 0.7, 403, None),
    ("magnitude", 7168, 7168, 0.7, 404, None),
]
CASES = BENCH + CONFIGS + OPT30B


def case_name(case):
    kind, m, k, s, seed, shard = case
    name = f"{kind}_{m}x{k}_s{s}_seed{seed}"
    if shard is not None:
        name += f"_shard{shard[0]}of{shard[1]}"
    return name
