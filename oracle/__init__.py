"""ORACLE — test infrastructure only.

A plain CPU implementation of what the B200 hot path computes (arXiv
2103.01597: one RK3 substep of compressible MHD on a periodic grid, plus the
radius-3 halo exchange over a Morton-ordered decomposition).  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py`` (its ``cpu_baseline`` leg and
``--impl reference``) may import this package.  It shares no code with
``paper_2103_01597_b200`` and never imports it.

* ``mhd_oracle.c`` — derivatives, RHS (App. B, Eqs. B.1-B.4), RK3,
  periodic fill.  Built twice: ``liboracle.so`` (double) and
  ``liboracle_ld.so`` (long double, to bound the oracle's own rounding).
* ``geometry.py`` — Morton mapping and the halo as a periodic wrap of
  the global grid, in plain Python/numpy.

Parity status of each function is listed in DESIGN.md ("Oracle pins").
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass, astuple

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "mhd_oracle.c")
LIB = {"d": os.path.join(HERE, "liboracle.so"), "ld": os.path.join(HERE, "liboracle_ld.so")}
R = 3
NF = 8
FIELDS = ("lnrho", "ux", "uy", "uz", "ss", "ax", "ay", "az")


def build(force: bool = False) -> None:
    """Compile the oracle with gcc (-O2, no fast-math, no FMA contraction)."""
    for kind, out in LIB.items():
        if not force and os.path.exists(out) and os.path.getmtime(out) >= os.path.getmtime(SRC):
            continue
        cmd = ["gcc", "-O2", "-std=c99", "-fPIC", "-shared", "-ffp-contract=off", "-fopenmp",
               "-o", out, SRC, "-lm"]
        if kind == "ld":
            cmd.insert(1, "-DORACLE_LONG_DOUBLE")
        subprocess.check_call(cmd)


class Params(ctypes.Structure):
    _fields_ = [(n, ctypes.c_double) for n in
                ("nu", "zeta", "eta", "mu0", "cs0", "cp", "gamma", "K", "H", "C", "lnrho0", "lnT0")]


_libs: dict = {}


def _lib(kind: str = "d"):
    if kind not in _libs:
        build()
        lib = ctypes.CDLL(LIB[kind])
        lib.oracle_real_bytes.restype = ctypes.c_int
        lib.oracle_grid_cells.restype = ctypes.c_size_t
        lib.oracle_integrate.restype = ctypes.c_int
        lib.oracle_integrate_w2.restype = ctypes.c_int
        lib.oracle_rhs_of_state.restype = ctypes.c_int
        _libs[kind] = lib
    return _libs[kind]


def _dtype(kind: str):
    return np.float64 if kind == "d" else np.longdouble


def _ptr(a: np.ndarray):
    assert a.flags.c_contiguous
    return a.ctypes.data_as(ctypes.c_void_p)


def _ptrs(arrs):
    return (ctypes.c_void_p * len(arrs))(*[a.ctypes.data for a in arrs])


def _ds(ds):
    return (ctypes.c_double * 3)(*[float(v) for v in ds])


def _params(p) -> Params:
    if isinstance(p, Params):
        return p
    if isinstance(p, dict):
        return Params(**{k: float(v) for k, v in p.items()})
    return Params(*[float(v) for v in p])


def set_threads(n: int) -> None:
    """OpenMP thread count for oracle_rhs (the only parallel loop; per-cell results do not depend on it)."""
    for kind in LIB:
        _lib(kind).oracle_set_threads(int(n))


def get_threads() -> int:
    return int(_lib("d").oracle_get_threads())


# --- grid helpers ------------------------------------------------------------------------------
def with_halo(interior: np.ndarray, r: int = R) -> np.ndarray:
    """Embed an interior (nz, ny, nx) array into a zero (nz+2r, ny+2r, nx+2r) grid."""
    nz, ny, nx = interior.shape
    g = np.zeros((nz + 2 * r, ny + 2 * r, nx + 2 * r), dtype=interior.dtype)
    g[r:r + nz, r:r + ny, r:r + nx] = interior
    return g


def periodic_fill(grid: np.ndarray, kind: str = "d", r: int = R) -> np.ndarray:
    """P:705 halo map on one halo-inclusive field of halo width r (in place, returned)."""
    g = np.ascontiguousarray(grid, dtype=_dtype(kind))
    nz, ny, nx = (s - 2 * r for s in g.shape)
    _lib(kind).oracle_periodic_fill(_ptr(g), nx, ny, nz, r)
    return g


def apply_op(grid: np.ndarray, ds, op: str, a1: int, a2: int = 0, kind: str = "d", r: int = R) -> np.ndarray:
    """Order-2r central-difference operator on a halo-filled field at every interior cell.

    op: 'd1' (first derivative along axis a1), 'd2' (second along a1), 'dx' (cross a1, a2).
    Axes: 0 = x (fastest), 1 = y, 2 = z.
    """
    g = np.ascontiguousarray(grid, dtype=_dtype(kind))
    nz, ny, nx = (s - 2 * r for s in g.shape)
    out = np.empty((nz, ny, nx), dtype=_dtype(kind))
    code = {"d1": 1, "d2": 2, "dx": 3}[op]
    _lib(kind).oracle_apply_op(_ptr(g), nx, ny, nz, r, _ds(ds), code, a1, a2, _ptr(out))
    return out


def rhs(state: np.ndarray, ds, params, kind: str = "d", r: int = R) -> np.ndarray:
    """RHS (B.1-B.4) of an interior state of shape (8, nz, ny, nx), periodic, order 2r."""
    st = [np.ascontiguousarray(state[q], dtype=_dtype(kind)) for q in range(NF)]
    nz, ny, nx = st[0].shape
    out = [np.empty((nz, ny, nx), dtype=_dtype(kind)) for _ in range(NF)]
    p = _params(params)
    rc = _lib(kind).oracle_rhs_of_state(_ptrs(st), nx, ny, nz, r, _ds(ds), ctypes.byref(p), _ptrs(out))
    if rc != 0:
        raise MemoryError("oracle_rhs_of_state")
    return np.stack(out)


def integrate(state: np.ndarray, ds, params, dt: float, nsteps: int, substeps: int | None = None,
              kind: str = "d", return_rhs: bool = False, r: int = R, form: str = "w"):
    """Run nsteps RK3 steps (or exactly `substeps` substeps) from an interior state (8, nz, ny, nx).

    form "w": the explicit 2N register (the definition, R#3); "w2": the algebraically
    identical two-state form of reading R#4 (only to attribute rounding differences).
    Returns the new state (and the RHS of the last substep if return_rhs).
    """
    st = [np.array(state[q], dtype=_dtype(kind), order="C", copy=True) for q in range(NF)]
    nz, ny, nx = st[0].shape
    rh = [np.empty((nz, ny, nx), dtype=_dtype(kind)) for _ in range(NF)]
    p = _params(params)
    fn = _lib(kind).oracle_integrate if form == "w" else _lib(kind).oracle_integrate_w2
    rc = fn(_ptrs(st), nx, ny, nz, r, _ds(ds), ctypes.byref(p), ctypes.c_double(dt),
                                     int(nsteps), -1 if substeps is None else int(substeps), _ptrs(rh))
    if rc != 0:
        raise MemoryError("oracle_integrate")
    out = np.stack(st)
    return (out, np.stack(rh)) if return_rhs else out


def rk3_linear(y0: np.ndarray, lam: float, dt: float, nsteps: int, kind: str = "d") -> np.ndarray:
    y = np.array(y0, dtype=_dtype(kind), order="C", copy=True)
    _lib(kind).oracle_rk3_linear(_ptr(y), ctypes.c_size_t(y.size), ctypes.c_double(lam),
                                 ctypes.c_double(dt), int(nsteps))
    return y
