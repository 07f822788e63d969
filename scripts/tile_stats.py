"""Tiled-layout statistics of each launch of a bench workload at several tile sizes:
stages x stage bytes, tiles, arena bytes and the mean tile fill (arena / (tiles x stage)).
python scripts/tile_stats.py WORKLOAD [tile_kb ...]   (0 = the packer's default)"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2507_12205_b200.device import to_device, vstack  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else bench.HEADLINE
kbs = [int(v) for v in sys.argv[2:]] or [0, 20, 24, 28]
ecs, _ = bench.load_workload(name)
for ln, names in bench.WORKLOADS[name]["launches"]:
    e = vstack([ecs[n] for n in names])
    for kb in kbs:
        W = to_device(e, tile_kb=kb or None)
        b = W.bytes()
        fill = b["device_arena_bytes"] / max(1, b["tiles"] * b["stage_bytes"])
        print(f"{name} {ln:8s} tile {kb:2d}: stages {b['stages']} x {b['stage_bytes']}, tiles {b['tiles']}, "
              f"arena {b['device_arena_bytes'] / 1e6:.1f} MB, fill {fill:.3f}, grid {b['grid']}", flush=True)
        W.free()
