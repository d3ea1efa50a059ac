"""Pins of the CPU oracle against things other than itself (no GPU).

Each test names what it pins and the passage it follows.  None of these
re-types the oracle's own formulas: they use FFT symbols (library routine),
polynomial exactness and convergence orders (mathematics), closed-form
solutions (Beltrami mode, uniform state, linear ODE), a symbolic transcription
of the continuum equations B.1-B.4 with textbook vector calculus,
conservation laws, and the long-double build of the oracle.
"""
import math

import numpy as np
import pytest

import oracle
from synth import P0, pcg64_state

R = 3
# A parameter set where every term of B.1-B.4 is O(0.1-1), so that a dropped
# or mis-signed term is far above the discretisation error.
PSTRONG = dict(nu=0.3, zeta=0.2, eta=0.25, mu0=1.4, cs0=1.1, cp=1.5, gamma=5.0 / 3.0,
               K=0.35, H=0.3, C=0.1, lnrho0=0.2, lnT0=0.1)


def _filled(interior, kind="d"):
    return oracle.periodic_fill(oracle.with_halo(interior.astype(np.float64)), kind)


# ---------------------------------------------------------------------------------------------
# Derivative operators vs FFT symbols (circulant operators on a periodic grid)
# ---------------------------------------------------------------------------------------------
def _symbols(n, ds):
    k = 2 * np.pi * np.fft.fftfreq(n)  # theta = k * ds, grid angle per cell
    return k


@pytest.mark.parametrize("shape_zyx", [(12, 20, 24), (16, 16, 16)])
def test_operators_equal_fft_symbols(shape_zyx):
    """D1, D2, DX are circulant; the FFT of each equals its Fourier symbol built from the
    Taylor-series weights of 6th-order central differences.  The weights below
    are the textbook ones; the pin is that the oracle's *application* matches the
    spectral product on random data (catches index, sign and axis errors)."""
    rng = np.random.default_rng(1)
    f = rng.random(shape_zyx)
    ds = (0.3, 0.7, 1.1)  # x, y, z
    g = _filled(f)
    F = np.fft.fftn(f)
    th = [None] * 3
    nz, ny, nx = shape_zyx
    th[0] = 2 * np.pi * np.fft.fftfreq(nx)[None, None, :]
    th[1] = 2 * np.pi * np.fft.fftfreq(ny)[None, :, None]
    th[2] = 2 * np.pi * np.fft.fftfreq(nz)[:, None, None]
    c = (3 / 4, -3 / 20, 1 / 60)
    d = (3 / 2, -3 / 20, 1 / 90)
    e = (270 / 720, -27 / 720, 2 / 720)
    for a in range(3):
        s1 = sum(2j * c[i - 1] * np.sin(i * th[a]) for i in (1, 2, 3)) / ds[a]
        s2 = sum(2 * d[i - 1] * (np.cos(i * th[a]) - 1) for i in (1, 2, 3)) / ds[a] ** 2
        ref1 = np.fft.ifftn(F * s1).real
        ref2 = np.fft.ifftn(F * s2).real
        np.testing.assert_allclose(oracle.apply_op(g, ds, "d1", a), ref1, atol=1e-13 / ds[a])
        np.testing.assert_allclose(oracle.apply_op(g, ds, "d2", a), ref2, atol=1e-12 / ds[a] ** 2)
        for b in range(3):
            if b == a:
                continue
            sx = sum(-4 * e[i - 1] * np.sin(i * th[a]) * np.sin(i * th[b]) for i in (1, 2, 3)) / (ds[a] * ds[b])
            refx = np.fft.ifftn(F * sx).real
            np.testing.assert_allclose(oracle.apply_op(g, ds, "dx", a, b), refx, atol=1e-12 / (ds[a] * ds[b]))


# ---------------------------------------------------------------------------------------------
# Polynomial exactness (mathematics: order of the central differences)
# ---------------------------------------------------------------------------------------------
def _poly_grid(fun, n=9, ds=(0.37, 0.29, 0.23), origin=(0.11, -0.07, 0.05)):
    """Halo-inclusive grid of fun(x, y, z) (no periodic fill) for exactness tests."""
    idx = np.arange(-R, n + R)
    x = origin[0] + idx[None, None, :] * ds[0]
    y = origin[1] + idx[None, :, None] * ds[1]
    z = origin[2] + idx[:, None, None] * ds[2]
    X, Y, Z = np.broadcast_arrays(x, y, z)
    pts = [a[R:-R, R:-R, R:-R] for a in (X, Y, Z)]
    return fun(X.astype(np.longdouble), Y.astype(np.longdouble), Z.astype(np.longdouble)), pts, ds


@pytest.mark.parametrize("axis", [0, 1, 2])
def test_d1_exact_to_degree_6_not_7(axis):
    """6th-order D1 is exact for polynomials of degree <= 6 and not for 7 (BASELINE north star pin 1)."""
    for deg in range(0, 8):
        g, pts, ds = _poly_grid(lambda X, Y, Z: [X, Y, Z][axis] ** deg + 0.5 * X * Y * Z)
        got = oracle.apply_op(g, ds, "d1", axis, kind="ld").astype(np.float64)
        q = [p.astype(np.float64) for p in pts]
        exact = deg * q[axis] ** max(deg - 1, 0) + 0.5 * np.prod([q[i] for i in range(3) if i != axis], axis=0)
        err = np.max(np.abs(got - exact)) / max(1.0, np.max(np.abs(exact)))
        if deg <= 6:
            assert err < 1e-12, (deg, err)
        else:
            assert err > 1e-6, (deg, err)


@pytest.mark.parametrize("axis", [0, 1, 2])
def test_d2_exact_to_degree_7_not_8(axis):
    for deg in range(0, 9):
        g, pts, ds = _poly_grid(lambda X, Y, Z: [X, Y, Z][axis] ** deg)
        got = oracle.apply_op(g, ds, "d2", axis, kind="ld").astype(np.float64)
        q = pts[axis].astype(np.float64)
        exact = deg * (deg - 1) * q ** max(deg - 2, 0)
        err = np.max(np.abs(got - exact)) / max(1.0, np.max(np.abs(exact)))
        if deg <= 7:
            assert err < 1e-11, (deg, err)
        else:
            assert err > 1e-6, (deg, err)


@pytest.mark.parametrize("a,b", [(0, 1), (0, 2), (1, 2), (1, 0)])
def test_cross_exact_to_total_degree_7(a, b):
    """The bidiagonal cross derivative on Eq. 14's diagonal points is exact for
    every monomial x_a^p x_b^q with p + q <= 7 and fails for some p + q = 8."""
    worst8 = 0.0
    for p in range(0, 9):
        for q in range(0, 9 - p):
            g, pts, ds = _poly_grid(lambda X, Y, Z: [X, Y, Z][a] ** p * [X, Y, Z][b] ** q)
            got = oracle.apply_op(g, ds, "dx", a, b, kind="ld").astype(np.float64)
            xa, xb = pts[a].astype(np.float64), pts[b].astype(np.float64)
            exact = p * q * xa ** max(p - 1, 0) * xb ** max(q - 1, 0)
            err = np.max(np.abs(got - exact)) / max(1.0, np.max(np.abs(exact)))
            if p + q <= 7:
                assert err < 1e-11, (p, q, err)
            else:
                worst8 = max(worst8, err)
    assert worst8 > 1e-6


# ---------------------------------------------------------------------------------------------
# Convergence order on sin/cos (north-star pin 2)
# ---------------------------------------------------------------------------------------------
def test_sixth_order_convergence_on_trig():
    errs = {"d1": [], "d2": [], "dx": []}
    for n in (16, 32, 64):
        L = 2 * np.pi
        ds = (L / n,) * 3
        x = np.arange(n) * ds[0]
        X = x[None, None, :]
        Y = x[None, :, None]
        Z = x[:, None, None]
        f = np.sin(X + 0.3) * np.cos(2 * Y) * np.ones_like(Z)
        g = _filled(np.broadcast_to(f, (n, n, n)).copy())
        errs["d1"].append(np.max(np.abs(oracle.apply_op(g, ds, "d1", 0) - np.cos(X + 0.3) * np.cos(2 * Y))))
        errs["d2"].append(np.max(np.abs(oracle.apply_op(g, ds, "d2", 1) + 4 * np.sin(X + 0.3) * np.cos(2 * Y))))
        errs["dx"].append(np.max(np.abs(oracle.apply_op(g, ds, "dx", 0, 1) + 2 * np.cos(X + 0.3) * np.sin(2 * Y))))
    for k, e in errs.items():
        r1, r2 = e[0] / e[1], e[1] / e[2]
        assert 50 < r1 < 80 and 50 < r2 < 80, (k, e)  # 2^6 = 64


def test_sum_of_first_derivative_vanishes():
    """Antisymmetric periodic D1 telescopes: sum over cells of D1 f = 0 (to rounding)."""
    f = np.random.default_rng(2).random((16, 12, 20))
    g = _filled(f)
    for a in range(3):
        s = oracle.apply_op(g, (0.1, 0.2, 0.3), "d1", a).sum()
        assert abs(s) < 1e-11


# ---------------------------------------------------------------------------------------------
# Periodic halo: sentinel = global linear index, bitwise
# ---------------------------------------------------------------------------------------------
def test_periodic_fill_sentinel_bitwise():
    nz, ny, nx = 7, 9, 11
    f = np.arange(nz * ny * nx, dtype=np.float64).reshape(nz, ny, nx)
    g = _filled(f)
    Z, Y, X = np.meshgrid(np.arange(nz + 6), np.arange(ny + 6), np.arange(nx + 6), indexing="ij")
    # s' = ((s - r) mod n) + r, per axis, then back to interior coordinates
    zz = (Z - R) % nz
    yy = (Y - R) % ny
    xx = (X - R) % nx
    expect = (zz * ny + yy) * nx + xx
    assert np.array_equal(g, expect.astype(np.float64))


# ---------------------------------------------------------------------------------------------
# RK3: amplification factor of a 3-stage 3rd-order RK on y' = lambda y
# ---------------------------------------------------------------------------------------------
def test_rk3_linear_amplification_factor():
    for lam, dt in [(-1.0, 0.1), (-3.0, 0.05), (0.7, 0.2), (-0.25, 1.0)]:
        y = oracle.rk3_linear(np.array([1.0, -2.0, 0.5]), lam, dt, 7)
        z = lam * dt
        Rz = 1 + z + z * z / 2 + z ** 3 / 6
        np.testing.assert_allclose(y, np.array([1.0, -2.0, 0.5]) * Rz ** 7, rtol=1e-14)


def test_rk3_global_order_three():
    errs = []
    for n in (20, 40, 80, 160):
        dt = 1.0 / n
        y = oracle.rk3_linear(np.array([1.0]), -2.0, dt, n)
        errs.append(abs(y[0] - math.exp(-2.0)))
    slopes = [math.log2(errs[i] / errs[i + 1]) for i in range(3)]
    assert all(abs(s - 3.0) < 0.2 for s in slopes), slopes


# ---------------------------------------------------------------------------------------------
# RHS special cases with closed forms
# ---------------------------------------------------------------------------------------------
def test_uniform_state_is_fixed_point_bitwise():
    """Uniform state with H = C: every term of B.1-B.4 vanishes exactly."""
    n = (8, 10, 12)
    st = np.empty((8,) + n)
    vals = [0.37, 0.11, -0.23, 0.41, 0.29, 0.5, -0.6, 0.7]
    for q in range(8):
        st[q] = vals[q]
    p = dict(PSTRONG, H=0.2, C=0.2)
    r = oracle.rhs(st, (0.3, 0.4, 0.5), p)
    assert np.all(r == 0.0)


def test_uniform_state_heating_closed_form():
    """Uniform state, H != C: only the entropy equation is driven, ds/dt = (H - C)/(rho T) (B.3)
    with T from the ideal-gas reading R#5."""
    n = (6, 8, 10)
    st = np.zeros((8,) + n)
    lnrho, s = 0.37, 0.29
    st[0] = lnrho
    st[4] = s
    p = PSTRONG
    r = oracle.rhs(st, (0.3, 0.4, 0.5), p)
    lnT = p["lnT0"] + p["gamma"] * s / p["cp"] + (p["gamma"] - 1) * (lnrho - p["lnrho0"])
    expect = (p["H"] - p["C"]) / (math.exp(lnrho) * math.exp(lnT))
    assert np.all(r[[0, 1, 2, 3, 5, 6, 7]] == 0.0)
    np.testing.assert_allclose(r[4], expect, rtol=1e-14)


def _modified_wavenumbers(k, ds):
    th = k * ds
    c = (3 / 4, -3 / 20, 1 / 60)
    d = (3 / 2, -3 / 20, 1 / 90)
    k1 = 2 * sum(c[i - 1] * math.sin(i * th) for i in (1, 2, 3)) / ds
    k2 = 2 * sum(d[i - 1] * (1 - math.cos(i * th)) for i in (1, 2, 3)) / ds ** 2
    return k1, k2


@pytest.mark.parametrize("axis", [0, 1, 2])
def test_beltrami_mode_closed_form(axis):
    """Force-free Beltrami mode along one axis: A = a(sin, cos) in the two transverse components,
    u = b(sin, cos), uniform lnrho and s.  Then B = k1 A, j = (k2/mu0) A, j x B = u x B = 0,
    so dA/dt = -eta k2 A, du/dt = -nu k2 u, dlnrho/dt = 0, and
    ds/dt = (H - C + eta k2^2 a^2/mu0 + rho nu k1^2 b^2)/(rho T) — uniform (B.1-B.4).
    With a large dt, RK3 must give A_n = R(-eta k2 dt)^n A_0."""
    n = {0: (8, 8, 32), 1: (8, 32, 8), 2: (32, 8, 8)}[axis]  # (nz, ny, nx)
    nxyz = (n[2], n[1], n[0])
    L = 2 * math.pi
    ds = tuple(L / v for v in nxyz)
    kw = 2
    coord = np.arange(nxyz[axis]) * ds[axis] * kw
    a, b = 0.8, 0.6
    lnrho, s = 0.15, 0.1
    shape = [1, 1, 1]
    shape[2 - axis] = nxyz[axis]
    sn = np.broadcast_to(np.sin(coord).reshape(shape), n)
    cs = np.broadcast_to(np.cos(coord).reshape(shape), n)
    t1, t2 = (axis + 1) % 3, (axis + 2) % 3  # transverse components, cyclic
    st = np.zeros((8,) + n)
    st[0] = lnrho
    st[4] = s
    st[1 + t1], st[1 + t2] = b * sn, b * cs
    st[5 + t1], st[5 + t2] = a * sn, a * cs
    p = PSTRONG
    k1, k2 = _modified_wavenumbers(kw, ds[axis])
    r = oracle.rhs(st, ds, p)
    np.testing.assert_allclose(r[5:8], -p["eta"] * k2 * st[5:8], atol=1e-13)
    np.testing.assert_allclose(r[1:4], -p["nu"] * k2 * st[1:4], atol=1e-13)
    assert np.max(np.abs(r[0])) < 1e-13
    rho = math.exp(lnrho)
    T = math.exp(p["lnT0"] + p["gamma"] * s / p["cp"] + (p["gamma"] - 1) * (lnrho - p["lnrho0"]))
    heat = p["H"] - p["C"] + p["eta"] * k2 ** 2 * a ** 2 / p["mu0"] + rho * p["nu"] * k1 ** 2 * b ** 2
    np.testing.assert_allclose(r[4], heat / (rho * T), rtol=1e-12)
    # time integration with a large dt so that the z^2 and z^3 terms of R(z) are resolved
    # dt below the RK3 stability limit of the stiffest (longitudinal viscous) mode
    dt, steps = 0.02, 8
    out = oracle.integrate(st, ds, p, dt, steps)
    zA, zu = -p["eta"] * k2 * dt, -p["nu"] * k2 * dt
    RA = (1 + zA + zA ** 2 / 2 + zA ** 3 / 6) ** steps
    Ru = (1 + zu + zu ** 2 / 2 + zu ** 3 / 6) ** steps
    np.testing.assert_allclose(out[5:8], RA * st[5:8], atol=1e-13)
    np.testing.assert_allclose(out[1:4], Ru * st[1:4], atol=1e-13)


# ---------------------------------------------------------------------------------------------
# Continuum limit: symbolic B.1-B.4 with textbook vector calculus
# ---------------------------------------------------------------------------------------------
def _continuum_rhs(p):
    import sympy as sp
    X, Y, Z = sp.symbols("x y z", real=True)
    V = (X, Y, Z)
    lnrho = 0.3 * sp.sin(X + 0.2) * sp.cos(Y) + 0.2 * sp.cos(Z - 0.4) + 0.25
    u = [0.4 * sp.sin(Y + 0.3) * sp.cos(Z), 0.35 * sp.cos(X) * sp.sin(Z + 0.1), 0.3 * sp.sin(X - 0.2) + 0.2 * sp.cos(Y)]
    s = 0.25 * sp.cos(X + Y) + 0.15 * sp.sin(Z) * sp.cos(X)
    A = [0.5 * sp.cos(Z + 0.5) * sp.sin(Y), 0.45 * sp.sin(X) * sp.cos(Z - 0.3), 0.4 * sp.cos(Y + 0.1) * sp.sin(X)]

    def grad(f):
        return [sp.diff(f, v) for v in V]

    def div(w):
        return sum(sp.diff(w[i], V[i]) for i in range(3))

    def curl(w):
        return [sp.diff(w[2], Y) - sp.diff(w[1], Z), sp.diff(w[0], Z) - sp.diff(w[2], X),
                sp.diff(w[1], X) - sp.diff(w[0], Y)]

    def lap(f):
        return sum(sp.diff(f, v, 2) for v in V)

    def cross(a, b):
        return [a[1] * b[2] - a[2] * b[1], a[2] * b[0] - a[0] * b[2], a[0] * b[1] - a[1] * b[0]]

    def dot(a, b):
        return sum(a[i] * b[i] for i in range(3))

    rho = sp.exp(lnrho)
    B = curl(A)                                # Table B.2
    j = [c / p["mu0"] for c in curl(B)]        # Table B.2: j = mu0^-1 curl B
    divu = div(u)
    S = [[sp.Rational(1, 2) * (sp.diff(u[i], V[k]) + sp.diff(u[k], V[i])) - (divu / 3 if i == k else 0)
          for k in range(3)] for i in range(3)]
    lnT = p["lnT0"] + p["gamma"] * s / p["cp"] + (p["gamma"] - 1) * (lnrho - p["lnrho0"])  # reading R#5
    T = sp.exp(lnT)
    cs2 = p["cs0"] ** 2 * sp.exp(lnT - p["lnT0"])
    gdiv = grad(divu)
    glnrho = grad(lnrho)
    jxB = cross(j, B)
    out = []
    out.append(-dot(u, glnrho) - divu)  # B.1 with D/Dt = d/dt + u.grad
    pg = grad(s / p["cp"] + lnrho)
    for i in range(3):
        Du = (-cs2 * pg[i] + jxB[i] / rho
              + p["nu"] * (lap(u[i]) + gdiv[i] / 3 + 2 * sum(S[i][k] * glnrho[k] for k in range(3)))
              + p["zeta"] * gdiv[i])
        out.append(Du - dot(u, grad(u[i])))  # B.2
    SS = sum(S[i][k] ** 2 for i in range(3) for k in range(3))
    gT = grad(T)
    divKgradT = sum(sp.diff(p["K"] * gT[i], V[i]) for i in range(3))
    rhoTDs = (p["H"] - p["C"] + divKgradT + p["eta"] * p["mu0"] * dot(j, j) + 2 * rho * p["nu"] * SS
              + p["zeta"] * rho * divu ** 2)
    out.append(rhoTDs / (rho * T) - dot(u, grad(s)))  # B.3
    uxB = cross(u, B)
    for i in range(3):
        out.append(uxB[i] + p["eta"] * lap(A[i]))  # B.4
    fields = [lnrho, u[0], u[1], u[2], s, A[0], A[1], A[2]]
    fn = sp.lambdify(V, fields, "numpy")
    rn = sp.lambdify(V, out, "numpy")
    return fn, rn


def test_rhs_converges_to_symbolic_continuum_equations():
    """The discrete RHS converges at 6th order to B.1-B.4 evaluated symbolically on smooth
    periodic fields, with j = mu0^-1 curl curl A and div(K grad T) taken literally."""
    p = PSTRONG
    fn, rn = _continuum_rhs(p)
    errs = []
    for n in (24, 48):
        ds = (2 * np.pi / n,) * 3
        c = np.arange(n) * ds[0]
        Z, Y, X = np.meshgrid(c, c, c, indexing="ij")
        st = np.stack([np.broadcast_to(np.asarray(v, dtype=np.float64), X.shape) for v in fn(X, Y, Z)])
        ex = np.stack([np.broadcast_to(np.asarray(v, dtype=np.float64), X.shape) for v in rn(X, Y, Z)])
        got = oracle.rhs(st, ds, p)
        errs.append([np.max(np.abs(got[q] - ex[q])) / np.max(np.abs(ex[q])) for q in range(8)])
    errs = np.array(errs)
    assert np.all(errs[1] < 2e-6), errs
    ratio = errs[0] / errs[1]
    assert np.all(ratio > 40), ratio  # 2^6 = 64 for 6th order


def test_periodic_mass_conservation():
    """d/dt sum(rho) = sum(rho * dlnrho/dt) = -sum(div(rho u)) = 0 in the continuum (B.1,
    periodic P:418).  On smooth periodic fields the discrete drift is at roundoff; a dropped or
    mis-signed term in B.1 would make it O(0.1) relative to sum |rho dlnrho/dt|."""
    p = PSTRONG
    fn, _ = _continuum_rhs(p)
    drift = []
    for n in (24, 48):
        ds = (2 * np.pi / n,) * 3
        c = np.arange(n) * ds[0]
        Z, Y, X = np.meshgrid(c, c, c, indexing="ij")
        st = np.stack([np.broadcast_to(np.asarray(v, dtype=np.float64), X.shape) for v in fn(X, Y, Z)])
        r = oracle.rhs(st, ds, p)
        rho = np.exp(st[0])
        drift.append(abs(np.sum(rho * r[0])) / np.sum(np.abs(rho * r[0])))
    assert max(drift) < 1e-12, drift


# ---------------------------------------------------------------------------------------------
# Stencil footprint (Eq. 14): the RHS at a cell reads exactly the 55-point set
# ---------------------------------------------------------------------------------------------
def test_rhs_footprint_is_eq14_point_set():
    n = 16
    st = pcg64_state((n, n, n), seed=7)
    ds = (0.2, 0.25, 0.3)
    base = oracle.rhs(st, ds, P0)
    cz = cy = cx = 8
    inset = set()
    for zz in range(-3, 4):
        for ax in range(3):
            o = [0, 0, 0]
            o[ax] = zz
            inset.add(tuple(o))
        for a, b in ((0, 1), (0, 2), (1, 2)):
            for sgn in (1, -1):
                o = [0, 0, 0]
                o[a] = zz
                o[b] = sgn * zz
                inset.add(tuple(o))
    assert len(inset) == 55  # 1 + 18 r (r = 3)
    tested = [(1, 1, 1), (2, -1, 0), (3, 3, 3), (1, 2, 0), (-3, 0, 0), (2, -2, 0), (0, 3, -3), (0, 0, 0),
              (-1, 3, 2), (3, 0, 3), (0, -1, -1), (0, 4, 0), (4, 4, 0)]
    union = set()
    for q in range(8):
        for o in tested:
            pert = st.copy()
            pert[q, cz + o[2], cy + o[1], cx + o[0]] += 0.125
            r = oracle.rhs(pert, ds, P0)
            changed = not np.array_equal(r[:, cz, cy, cx], base[:, cz, cy, cx])
            on_axis = sum(v != 0 for v in o) <= 1 and max(abs(v) for v in o) <= 3
            # lnrho and s need only axis derivatives; component c of u or A needs the cross
            # derivatives d_c d_b (grad div), i.e. the two diagonal planes containing axis c
            if q in (0, 4):
                expect = on_axis
            else:
                c = (q - 1) % 4 if q < 4 else q - 5
                diag_c = o in inset and o[c] != 0 and sum(v != 0 for v in o) == 2
                expect = on_axis or diag_c
            assert changed == expect, (q, o)
            if changed:
                union.add(o)
    assert union == {o for o in tested if o in inset}


# ---------------------------------------------------------------------------------------------
# The oracle's own rounding: double vs long double after 10 steps of the parity workload
# ---------------------------------------------------------------------------------------------
def test_double_vs_long_double_oracle_rounding():
    n = (12, 12, 12)
    st = pcg64_state(n)
    ds = (2 * np.pi / 12,) * 3
    d = oracle.integrate(st, ds, P0, 1.19209e-7, 10)
    ld = oracle.integrate(st, ds, P0, 1.19209e-7, 10, kind="ld").astype(np.float64)
    for q in range(8):
        e = np.max(np.abs(d[q] - ld[q]) / np.maximum(np.abs(ld[q]), 1e-3 * np.max(np.abs(ld[q]))))
        assert e < 1e-13, (q, e)
        inc_d, inc_ld = d[q] - st[q], ld[q] - st[q]
        # floor: ~30 roundings of f (ulp ~ 1e-16) against an increment of ~5e-6 (lnrho) ~ 1e-9
        assert np.max(np.abs(inc_d - inc_ld)) / np.max(np.abs(inc_ld)) < 2e-9


# ---------------------------------------------------------------------------------------------
# The two-state RK3 form (reading R#4) is the explicit 2N scheme up to rounding
# ---------------------------------------------------------------------------------------------
def test_two_state_rk3_form_equals_explicit_form():
    n = (12, 12, 12)
    st = pcg64_state(n)
    ds = (2 * np.pi / 12,) * 3
    for kind, tol in (("d", 1e-13), ("ld", 1e-15)):  # ld: coefficients rounded to double, as on the GPU
        w = oracle.integrate(st, ds, P0, 1.19209e-7, 3, kind=kind).astype(np.float64)
        w2 = oracle.integrate(st, ds, P0, 1.19209e-7, 3, kind=kind, form="w2").astype(np.float64)
        for q in range(8):
            e = np.max(np.abs(w[q] - w2[q]) / np.maximum(np.abs(w[q]), 1e-3 * np.max(np.abs(w[q]))))
            assert e < tol, (kind, q, e)
    # and on y' = lambda y with a large lambda dt the two forms give the same amplification R(z)
    lam, dt = -2.0, 0.1
    z = lam * dt
    y0 = np.ones((1, 1, 1))
    st1 = np.zeros((8, 4, 4, 4))
    st1[0] = 1.0
    # a uniform state with H = C has RHS = 0 for every field: the state must be a bitwise fixed point
    p = dict(P0)
    p["H"] = p["C"] = 0.0
    fixed = oracle.integrate(st1, (0.5, 0.5, 0.5), p, 0.1, 2, form="w2")
    assert np.array_equal(fixed, st1)
    assert abs(float(oracle.rk3_linear(y0, lam, dt, 1)[0, 0, 0]) - (1 + z + z * z / 2 + z ** 3 / 6)) < 1e-15
