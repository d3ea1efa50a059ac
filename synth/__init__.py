"""Seeded synthetic inputs shared by the oracle side and the CUDA side.

This module holds NONE of the method's arithmetic: only the workload recipe
 — random initial conditions, the parameter set P0,
the grid spacing convention and the time step.

* Initial data: "random values in the range [0, 1]".  Two generators:
  - ``pcg64_state``: numpy PCG64(seed).random((8, nz, ny, nx)) — the parity ICs.
  - ``splitmix_state``: counter-based splitmix64 of (seed, field, global cell
    index) -> 53-bit uniform in [0, 1).  Each rank generates only its own cells,
    and the global field does not depend on the decomposition.
* dt = 1.19209e-7, constant.
* Box 2*pi per axis unless stated (reading R#13); ds = L / n.
* Parameters P0 (reading R#12): the paper gives no values (Table B.2 lists
  symbols only).
"""
from __future__ import annotations

import math

import numpy as np

SEED = 210301597
DT = 1.19209e-7
NF = 8
FIELDS = ("lnrho", "ux", "uy", "uz", "ss", "ax", "ay", "az")

# Parameter set "P0" (reading R#12): non-unity values so that placement bugs show.
P0 = dict(nu=5e-3, zeta=1e-3, eta=5e-3, mu0=1.4, cs0=1.0, cp=1.5, gamma=5.0 / 3.0,
          K=1e-3, H=1e-3, C=5e-4, lnrho0=0.2, lnT0=0.0)
PARAM_ORDER = ("nu", "zeta", "eta", "mu0", "cs0", "cp", "gamma", "K", "H", "C", "lnrho0", "lnT0")


def spacing(n_xyz, box_xyz=None):
    """ds per axis (x, y, z) for a periodic box (default 2*pi per axis)."""
    if box_xyz is None:
        box_xyz = (2 * math.pi,) * 3
    return tuple(b / n for b, n in zip(box_xyz, n_xyz))


def pcg64_state(n_zyx, seed: int = SEED, dtype=np.float64) -> np.ndarray:
    """Parity ICs: Generator(PCG64(seed)).random((8, nz, ny, nx)), field order FIELDS."""
    g = np.random.Generator(np.random.PCG64(seed))
    return g.random((NF,) + tuple(n_zyx)).astype(dtype)


_M64 = np.uint64(0xFFFFFFFFFFFFFFFF)


def _splitmix64(x: np.ndarray) -> np.ndarray:
    with np.errstate(over="ignore"):
        z = x + np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return z ^ (z >> np.uint64(31))


def splitmix_state(global_zyx, lo_zyx, n_zyx, seed: int = SEED, dtype=np.float64, fields=None) -> np.ndarray:
    """Counter-based ICs for the block [lo, lo+n) of a global grid: value(field q, global linear
    index g) = (splitmix64(seed ^ (q * C_N + g)) >> 11) * 2^-53.  Decomposition independent.
    fields: the field indices to generate (default all 8), in that order."""
    Nz, Ny, Nx = global_zyx
    cn = np.uint64(Nz * Ny * Nx)
    z = np.arange(lo_zyx[0], lo_zyx[0] + n_zyx[0], dtype=np.uint64)[:, None, None]
    y = np.arange(lo_zyx[1], lo_zyx[1] + n_zyx[1], dtype=np.uint64)[None, :, None]
    x = np.arange(lo_zyx[2], lo_zyx[2] + n_zyx[2], dtype=np.uint64)[None, None, :]
    gidx = (z * np.uint64(Ny) + y) * np.uint64(Nx) + x
    fields = tuple(range(NF)) if fields is None else tuple(fields)
    out = np.empty((len(fields),) + tuple(n_zyx), dtype=dtype)
    with np.errstate(over="ignore"):
        for i, q in enumerate(fields):
            for z0 in range(0, int(n_zyx[0]), 64):  # z slabs bound the temporaries
                h = _splitmix64(np.uint64(seed) ^ (np.uint64(q) * cn + gidx[z0:z0 + 64]))
                out[i, z0:z0 + 64] = ((h >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)).astype(dtype)
    return out
