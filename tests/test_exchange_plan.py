"""Host logic of the peer-memory y exchange (paper_2507_12205_b200/exchange.py): every
rank's segments together cover y_full exactly once, each inside the rank's own SpMV
output slot (SURVEY.md §8(e) layout)."""

import numpy as np

from paper_2507_12205_b200.exchange import shard_segments
from paper_2507_12205_b200.generators import make_matrix
from paper_2507_12205_b200.sharded import shard_bounds


def test_segments_tile_y_full_exactly_once():
    world = 3
    launches = [[make_matrix("uniform", m, 64, 0.5, s).row_ptr for m, s in [(40, 1), (33, 2)]],
                [make_matrix("uniform", 57, 64, 0.7, 3).row_ptr]]
    bounds = [[shard_bounds(rp, world) for rp in mats] for mats in launches]
    rows = [sum(b[-1] for b in bl) for bl in bounds]
    y_off = np.concatenate([[0], np.cumsum(rows)[:-1]]).tolist()
    slot = [max(sum(b[r + 1] - b[r] for b in bl) for r in range(world)) for bl in bounds]
    slot_off = np.concatenate([[0], np.cumsum(slot)[:-1]]).tolist()
    cover = np.zeros(sum(rows), int)
    for r in range(world):
        mine = sum(sum(b[r + 1] - b[r] for b in bl) for bl in bounds)
        got = 0
        for so, do, n in shard_segments(bounds, slot_off, y_off, r):
            cover[do:do + n] += 1
            got += n
            # inside this rank's slot of the launch the segment came from
            li = max(i for i, o in enumerate(slot_off) if o <= so)
            assert so + n <= slot_off[li] + slot[li]
        assert got == mine
    assert np.all(cover == 1)
