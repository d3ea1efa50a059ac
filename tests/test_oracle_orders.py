"""Pins of the oracle at every stencil order the paper's solver supports: 2nd, 4th, 6th, 8th
(P:829-830), i.e. radius r = 1..4 (k = 2r).  Same kinds of pins as test_oracle_pins.py:
FFT symbols, polynomial exactness (and its failure one degree up), convergence order 2r,
periodic fill, the Eq. 14 footprint (18 r + 1 points), closed-form RHS cases."""
import math

import numpy as np
import pytest

import oracle
from synth import P0, pcg64_state

ORDERS = [1, 2, 3, 4]
# textbook central-difference weights (first and second derivative), i = 1..r
C1 = {1: (1 / 2,), 2: (2 / 3, -1 / 12), 3: (3 / 4, -3 / 20, 1 / 60), 4: (4 / 5, -1 / 5, 4 / 105, -1 / 280)}
D2 = {1: (1.0,), 2: (4 / 3, -1 / 12), 3: (3 / 2, -3 / 20, 1 / 90), 4: (8 / 5, -1 / 5, 8 / 315, -1 / 560)}
PSTRONG = dict(nu=0.3, zeta=0.2, eta=0.25, mu0=1.4, cs0=1.1, cp=1.5, gamma=5.0 / 3.0,
               K=0.35, H=0.3, C=0.1, lnrho0=0.2, lnT0=0.1)


def _filled(interior, r):
    return oracle.periodic_fill(oracle.with_halo(interior.astype(np.float64), r), r=r)


@pytest.mark.parametrize("r", ORDERS)
def test_fft_symbols(r):
    rng = np.random.default_rng(3 + r)
    shape = (12, 14, 18)
    f = rng.random(shape)
    ds = (0.31, 0.52, 0.77)
    g = _filled(f, r)
    F = np.fft.fftn(f)
    nz, ny, nx = shape
    th = [2 * np.pi * np.fft.fftfreq(nx)[None, None, :], 2 * np.pi * np.fft.fftfreq(ny)[None, :, None],
          2 * np.pi * np.fft.fftfreq(nz)[:, None, None]]
    for a in range(3):
        s1 = sum(2j * C1[r][i - 1] * np.sin(i * th[a]) for i in range(1, r + 1)) / ds[a]
        s2 = sum(2 * D2[r][i - 1] * (np.cos(i * th[a]) - 1) for i in range(1, r + 1)) / ds[a] ** 2
        np.testing.assert_allclose(oracle.apply_op(g, ds, "d1", a, r=r), np.fft.ifftn(F * s1).real, atol=1e-12)
        np.testing.assert_allclose(oracle.apply_op(g, ds, "d2", a, r=r), np.fft.ifftn(F * s2).real, atol=1e-11)
        b = (a + 1) % 3
        sx = sum(-D2[r][i - 1] * np.sin(i * th[a]) * np.sin(i * th[b]) for i in range(1, r + 1)) / (ds[a] * ds[b])
        np.testing.assert_allclose(oracle.apply_op(g, ds, "dx", a, b, r=r), np.fft.ifftn(F * sx).real, atol=1e-11)


def _poly(fun, r, n=7, ds=(0.37, 0.29, 0.23), origin=(0.11, -0.07, 0.05)):
    idx = np.arange(-r, n + r)
    X, Y, Z = np.broadcast_arrays(origin[0] + idx[None, None, :] * ds[0], origin[1] + idx[None, :, None] * ds[1],
                                  origin[2] + idx[:, None, None] * ds[2])
    pts = [a[r:-r, r:-r, r:-r].astype(np.float64) for a in (X, Y, Z)]
    L = np.longdouble
    return fun(X.astype(L), Y.astype(L), Z.astype(L)), pts, ds


@pytest.mark.parametrize("r", ORDERS)
def test_exactness_degree(r):
    """Order 2r: D1 exact to degree 2r (not 2r+1); D2 and the cross derivative exact to degree
    2r+1 (not 2r+2)."""
    for deg in range(0, 2 * r + 2):
        g, pts, ds = _poly(lambda X, Y, Z: X ** deg, r)
        got = oracle.apply_op(g, ds, "d1", 0, kind="ld", r=r).astype(np.float64)
        ex = deg * pts[0] ** max(deg - 1, 0)
        err = np.max(np.abs(got - ex)) / max(1.0, np.max(np.abs(ex)))
        assert (err < 1e-11) if deg <= 2 * r else (err > 1e-7), ("d1", deg, err)
    for deg in range(0, 2 * r + 3):
        g, pts, ds = _poly(lambda X, Y, Z: Y ** deg, r)
        got = oracle.apply_op(g, ds, "d2", 1, kind="ld", r=r).astype(np.float64)
        ex = deg * (deg - 1) * pts[1] ** max(deg - 2, 0)
        err = np.max(np.abs(got - ex)) / max(1.0, np.max(np.abs(ex)))
        assert (err < 1e-10) if deg <= 2 * r + 1 else (err > 1e-7), ("d2", deg, err)
    worst = 0.0
    for p in range(0, 2 * r + 3):
        for q in range(0, 2 * r + 3 - p):
            g, pts, ds = _poly(lambda X, Y, Z: X ** p * Z ** q, r)
            got = oracle.apply_op(g, ds, "dx", 0, 2, kind="ld", r=r).astype(np.float64)
            ex = p * q * pts[0] ** max(p - 1, 0) * pts[2] ** max(q - 1, 0)
            err = np.max(np.abs(got - ex)) / max(1.0, np.max(np.abs(ex)))
            if p + q <= 2 * r + 1:
                assert err < 1e-10, ("dx", p, q, err)
            else:
                worst = max(worst, err)
    assert worst > 1e-7


@pytest.mark.parametrize("r", ORDERS)
def test_convergence_order(r):
    errs = []
    ns = (16, 32) if r < 4 else (24, 48)
    for n in ns:
        ds = (2 * np.pi / n,) * 3
        x = np.arange(n) * ds[0]
        f = np.broadcast_to(np.sin(x[None, None, :] + 0.3) * np.cos(2 * x[None, :, None]), (n, n, n)).copy()
        g = _filled(f, r)
        ex = np.cos(x[None, None, :] + 0.3) * np.cos(2 * x[None, :, None])
        errs.append(np.max(np.abs(oracle.apply_op(g, ds, "d1", 0, r=r) - ex)))
    ratio = errs[0] / errs[1]
    assert 0.75 * 2 ** (2 * r) < ratio < 1.3 * 2 ** (2 * r), (r, errs)


@pytest.mark.parametrize("r", ORDERS)
def test_periodic_fill_and_footprint(r):
    nz, ny, nx = 9, 11, 10
    f = np.arange(nz * ny * nx, dtype=np.float64).reshape(nz, ny, nx)
    g = _filled(f, r)
    Z, Y, X = np.meshgrid(*(np.arange(v + 2 * r) for v in (nz, ny, nx)), indexing="ij")
    assert np.array_equal(g, (((Z - r) % nz) * ny + (Y - r) % ny) * nx + (X - r) % nx)
    # footprint: the RHS at a cell depends on exactly the Eq. 14 point set of radius r
    n = 16
    st = pcg64_state((n, n, n), seed=11)
    ds = (0.2, 0.25, 0.3)
    base = oracle.rhs(st, ds, P0, r=r)
    c = 8
    hit = set()
    for dz in range(-r - 1, r + 2):
        for dy in range(-r - 1, r + 2):
            for dx in range(-r - 1, r + 2):
                pert = st.copy()
                pert[:, c + dz, c + dy, c + dx] += 0.0625
                if not np.array_equal(oracle.rhs(pert, ds, P0, r=r)[:, c, c, c], base[:, c, c, c]):
                    hit.add((dx, dy, dz))
    expect = {(0, 0, 0)}
    for k in range(1, r + 1):
        for s in (k, -k):
            for ax in range(3):
                o = [0, 0, 0]
                o[ax] = s
                expect.add(tuple(o))
            for a, b in ((0, 1), (0, 2), (1, 2)):
                for t in (k, -k):
                    o = [0, 0, 0]
                    o[a], o[b] = s, t
                    expect.add(tuple(o))
    assert len(expect) == 18 * r + 1 and hit == expect


@pytest.mark.parametrize("r", ORDERS)
def test_uniform_state_and_beltrami(r):
    st = np.zeros((8, 6, 8, 10))
    for q, v in enumerate((0.37, 0.11, -0.23, 0.41, 0.29, 0.5, -0.6, 0.7)):
        st[q] = v
    assert np.all(oracle.rhs(st, (0.3, 0.4, 0.5), dict(PSTRONG, H=0.2, C=0.2), r=r) == 0.0)
    # Beltrami mode along z: dA/dt = -eta k2 A, du/dt = -nu k2 u with the order-2r symbol k2
    n = (24, 8, 8)
    L = 2 * math.pi
    dz = L / n[0]
    z = np.arange(n[0]) * dz
    sn = np.broadcast_to(np.sin(2 * z)[:, None, None], n)
    cs = np.broadcast_to(np.cos(2 * z)[:, None, None], n)
    st = np.zeros((8,) + n)
    st[0], st[4] = 0.15, 0.1
    st[1], st[2], st[5], st[6] = 0.6 * sn, 0.6 * cs, 0.8 * sn, 0.8 * cs
    th = 2 * dz
    k2 = 2 * sum(D2[r][i - 1] * (1 - math.cos(i * th)) for i in range(1, r + 1)) / dz ** 2
    out = oracle.rhs(st, (L / 8, L / 8, dz), PSTRONG, r=r)
    np.testing.assert_allclose(out[5:8], -PSTRONG["eta"] * k2 * st[5:8], atol=1e-12)
    np.testing.assert_allclose(out[1:4], -PSTRONG["nu"] * k2 * st[1:4], atol=1e-12)


@pytest.mark.parametrize("r", [1, 4])
def test_double_vs_long_double(r):
    n = (12, 12, 12)
    st = pcg64_state(n)
    ds = (2 * np.pi / 12,) * 3
    d = oracle.integrate(st, ds, P0, 1.19209e-7, 5, r=r)
    ld = oracle.integrate(st, ds, P0, 1.19209e-7, 5, kind="ld", r=r).astype(np.float64)
    assert np.max(np.abs(d - ld)) < 1e-13
