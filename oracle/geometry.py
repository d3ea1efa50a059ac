"""ORACLE — test infrastructure only: decomposition geometry from the paper, written out plainly.

* Morton (Z-order) mapping, P:557 (§3.3): morton^-1 maps the binary index
  i = abcdef_2 to the coordinate (cf_2, be_2, ad_2): bit 3k + j of i is bit k of
  coordinate j.  The partition is P* = morton^-1(C_P - 1) + (1, 1, 1).
* The halo of a subdomain is the periodic wrap of the global grid
  (s'_i = ((s_i - r) mod n'_i) + r) with P:418 periodic boundaries: every halo
  cell equals the global cell at the wrapped global index.

Axis naming (reading R#16 in DESIGN.md): Morton coordinate 0 maps to the
slowest memory axis z, coordinate 1 to y, coordinate 2 to x.
"""
from __future__ import annotations

import numpy as np

R = 3


def morton_inverse(i: int, d: int = 3) -> tuple:
    """de-interleave the bits of i into d coordinates (bit 3k+j of i -> bit k of coord j)."""
    coord = [0] * d
    k = 0
    while i >> (d * k):
        for j in range(d):
            coord[j] |= ((i >> (d * k + j)) & 1) << k
        k += 1
    return tuple(coord)


def morton(coord) -> int:
    """Inverse of morton_inverse (bit interleave)."""
    d = len(coord)
    i = 0
    for j, c in enumerate(coord):
        k = 0
        while c >> k:
            i |= ((c >> k) & 1) << (d * k + j)
            k += 1
    return i


def partition(n_procs: int) -> tuple:
    """P* = morton^-1(C_P - 1) + (1, 1, 1), in Morton coordinate order."""
    return tuple(c + 1 for c in morton_inverse(n_procs - 1))


def partition_zyx(n_procs: int) -> tuple:
    """Partition as (pz, py, px): Morton coordinate 0 -> z (reading R#16)."""
    return partition(n_procs)


def rank_coord_zyx(rank: int) -> tuple:
    """Subdomain coordinate (cz, cy, cx) of a rank: morton^-1(rank)."""
    return morton_inverse(rank)


def local_subgrid_with_halo(global_interior: np.ndarray, P_zyx, coord_zyx, r: int = R) -> np.ndarray:
    """The halo-inclusive subgrid M' of one subdomain, filled by periodic wrap of the global grid.

    global_interior: (..., Nz, Ny, Nx).  Returns (..., nz'+2r, ny'+2r, nx'+2r).
    """
    shape = global_interior.shape[-3:]
    idx = []
    for ax in range(3):
        n_loc = shape[ax] // P_zyx[ax]
        lo = coord_zyx[ax] * n_loc
        idx.append((np.arange(-r, n_loc + r) + lo) % shape[ax])
    g = np.take(global_interior, idx[0], axis=-3)
    g = np.take(g, idx[1], axis=-2)
    g = np.take(g, idx[2], axis=-1)
    return g


def local_interior(global_interior: np.ndarray, P_zyx, coord_zyx) -> np.ndarray:
    shape = global_interior.shape[-3:]
    sl = []
    for ax in range(3):
        n_loc = shape[ax] // P_zyx[ax]
        sl.append(slice(coord_zyx[ax] * n_loc, (coord_zyx[ax] + 1) * n_loc))
    return global_interior[(Ellipsis, sl[0], sl[1], sl[2])]


def halo_cells(n_loc_zyx, r: int = R) -> int:
    """C_M' - C_N' (Eqs. 2-3)."""
    m = 1
    n = 1
    for v in n_loc_zyx:
        m *= v + 2 * r
        n *= v
    return m - n
