"""Pins of the oracle's geometry (Morton mapping, periodic halo) against the paper's worked values."""
import json
import os

import numpy as np

from oracle import geometry as G

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_values.json")))


def test_morton_worked_example_p557():
    """morton^-1(abcdef_2) = (cf_2, be_2, ad_2), for every assignment of the six bits."""
    ex = GOLD["morton_example"]
    letters = ex["index_bits_msb_first"]
    for i in range(64):
        bits = {letters[k]: (i >> (5 - k)) & 1 for k in range(6)}
        expect = tuple(int("".join(str(bits[b]) for b in cb), 2) for cb in ex["coordinate_bits_msb_first"])
        assert G.morton_inverse(i) == expect
        assert G.morton(expect) == i


def test_partitions_from_p557_formula():
    """P* = morton^-1(C_P - 1) + (1,1,1) gives power-of-two partitions with prod = C_P, and
    the 16-node partition (4, 2, 2) used for P:911-912's model."""
    for cp in (1, 2, 4, 8, 16, 32, 64):
        P = G.partition(cp)
        assert int(np.prod(P)) == cp
        coords = {G.morton_inverse(k) for k in range(cp)}
        assert len(coords) == cp and all(all(c < p for c, p in zip(cc, P)) for cc in coords)
    assert G.partition(2) == (2, 1, 1)
    assert G.partition(4) == (2, 2, 1)
    assert G.partition(8) == (2, 2, 2)
    assert G.partition(16) == (4, 2, 2)


def test_segment_map_formula_p705():
    """s'_i = ((s_i - r) mod n'_i) + r maps halo indices into the neighbour's domain [r, r + n')."""
    r = 3
    for n in (4, 7, 64):
        for s in range(0, n + 2 * r):
            sp = ((s - r) % n) + r
            assert r <= sp < r + n
    # SPEC worked examples (derived): s = 0 -> 64; s = 67 -> 3 for n' = 64
    assert ((0 - 3) % 64) + 3 == 64 and ((67 - 3) % 64) + 3 == 3


def test_local_subgrid_is_periodic_wrap():
    N = (8, 6, 10)
    g = np.arange(np.prod(N), dtype=np.float64).reshape(N)
    P = (2, 1, 2)
    for cz in range(2):
        for cx in range(2):
            sub = G.local_subgrid_with_halo(g, P, (cz, 0, cx))
            assert sub.shape == (4 + 6, 6 + 6, 5 + 6)
            # interior equals the block
            assert np.array_equal(sub[3:-3, 3:-3, 3:-3], G.local_interior(g, P, (cz, 0, cx)))
            # one halo corner cell, by hand
            z, y, x = (cz * 4 - 3) % 8, (0 - 3) % 6, (cx * 5 - 3) % 10
            assert sub[0, 0, 0] == g[z, y, x]


def test_halo_cell_counts():
    """C_M' - C_N' (Eqs. 2-3) at the survey's sizes, and the largest segment at 256^3 is 12 MiB."""
    assert G.halo_cells((32, 32, 32)) == 22104
    assert G.halo_cells((256, 256, 256)) == 1207512
    assert G.halo_cells((512, 512, 512)) == 4774104
    gold = GOLD["largest_segment_256"]
    assert 3 * 256 * 256 * 8 * 8 == gold["bytes"]
