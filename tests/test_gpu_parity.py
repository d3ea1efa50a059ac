"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle on identical seeded inputs.

Tolerances (BASELINE.json north star):
  * halo exchange, load/store, indexing: bit-exact;
  * fields after 10 RK3 steps: max relative error <= 1e-11 (FP64), <= 1e-4 (FP32), with the
    per-field floor e = max|g - o| / max(|o|, 1e-3 ||o||_inf) (reading R#18);
  * RHS (debug_rhs): ||g - o||_inf / ||o||_inf <= 1e-12 (FP64), <= 1e-4 (FP32);
  * increments f(steps) - f(0): normwise <= 1e-9 against the long-double oracle (FP64; the
    double oracle's own floor, ~2e-9 at 12^3, tests/test_oracle_pins.py, is not in the way);
    FP32: <= 2e-2, or the bound FP32 state storage allows where the increment is smaller
    (_fp32_increment_ok).
"""
import math

import numpy as np
import pytest

import oracle
import synth

pytestmark = pytest.mark.gpu

PSTRONG = dict(nu=0.3, zeta=0.2, eta=0.25, mu0=1.4, cs0=1.1, cp=1.5, gamma=5.0 / 3.0,
               K=0.35, H=0.3, C=0.1, lnrho0=0.2, lnT0=0.1)


def _mesh(n_xyz, ds=None, params=synth.P0, dtype=None, **kw):
    import paper_2103_01597_b200 as b2
    import torch
    torch.cuda.set_device(0)
    ds = ds or synth.spacing(n_xyz)
    return b2.Mesh(n_xyz, ds, params, dtype or b2.MHD_F64, **kw), ds


def _field_err(g, o):
    return max(float(np.max(np.abs(g[q] - o[q]) / np.maximum(np.abs(o[q]), 1e-3 * np.max(np.abs(o[q])))))
               for q in range(8))


def _norm_err(g, o):
    return max(float(np.max(np.abs(g[q] - o[q])) / np.max(np.abs(o[q]))) for q in range(8))


def _fp32_increment_ok(got, ref, st, nsub):
    """FP32 increment parity per field: normwise <= 2e-2, or, where the increment is
    too small for that, the bound the FP32 state storage itself allows: every substep rounds f to
    FP32 (|error| <= 2^-24 |f| <= 2^-23 max|f|), so after nsub substeps the increment can be off
    by nsub 2^-23 max|f| against an exact-arithmetic reference."""
    for q in range(8):
        inc_g, inc_o = got[q] - st[q], ref[q] - st[q]
        den = np.max(np.abs(inc_o))
        e = float(np.max(np.abs(inc_g - inc_o)) / den)
        tol = max(2e-2, nsub * 2.0 ** -23 * float(np.max(np.abs(ref[q]))) / den)
        assert e <= tol, (q, e, tol)


# ---- bit-exact data movement --------------------------------------------------------------------
@pytest.mark.parametrize("dtype", [8, 4])
def test_load_store_roundtrip_bitwise(dtype):
    n = (37, 23, 19)
    m, _ = _mesh(n, dtype=dtype)
    st = synth.pcg64_state((n[2], n[1], n[0]), dtype=np.float64 if dtype == 8 else np.float32)
    m.load(st)
    got = m.store().cpu().numpy()
    assert np.array_equal(got, st)
    import torch
    pinned = torch.empty_like(torch.from_numpy(st)).pin_memory()
    m.store(out=pinned)
    assert np.array_equal(pinned.numpy(), st)
    # asynchronous store (staging + copy stream), interleaved with updates and reloads
    a = torch.empty_like(pinned).pin_memory()
    b = torch.empty_like(pinned).pin_memory()
    m.store_async(a)
    m.step(1e-4)
    ref = m.store().cpu().numpy()
    m.store_async(b)
    m.load(st)
    m.synchronize()
    assert np.array_equal(a.numpy(), st) and np.array_equal(b.numpy(), ref)
    # asynchronous load: a pipelined load -> step -> store sequence equals the blocking one
    src = torch.from_numpy(st).pin_memory()
    m.load_async(src)
    m.step(1e-4)
    m.store_async(a)
    m.load_async(src)
    m.store_async(b)
    m.synchronize()
    assert np.array_equal(a.numpy(), ref) and np.array_equal(b.numpy(), st)
    m.close()


@pytest.mark.parametrize("corners", [False, True])
@pytest.mark.parametrize("n", [(32, 32, 32), (37, 23, 19)])
def test_halo_exchange_sentinel_bitwise(corners, n):
    """Sentinel = global linear index; every halo cell must hold the wrapped index."""
    m, _ = _mesh(n, exchange_corners=corners)
    nz, ny, nx = n[2], n[1], n[0]
    st = (np.arange(8)[:, None, None, None] * 1e6 + np.arange(nz * ny * nx).reshape(nz, ny, nx)).astype(np.float64)
    m.load(st)
    m.halo_exchange()
    grid = m.store_grid().numpy()
    expect = np.stack([oracle.periodic_fill(oracle.with_halo(st[q])) for q in range(8)])
    mask = np.ones(grid.shape[1:], bool)
    if not corners:
        for zs in (slice(0, 3), slice(-3, None)):
            for ys in (slice(0, 3), slice(-3, None)):
                for xs in (slice(0, 3), slice(-3, None)):
                    mask[zs, ys, xs] = False
    assert np.array_equal(grid[:, mask], expect[:, mask])
    m.close()


@pytest.mark.parametrize("dtype", [8, 4])
@pytest.mark.parametrize("n,r", [((40, 24, 19), 3), ((37, 23, 16), 1), ((36, 20, 18), 4), ((64, 48, 40), 3),
                                 ((12, 20, 16), 3)])
def test_poison_halo_steps_bit_identical(dtype, n, r):
    """NaN-poison mode (MHD_DEBUG_POISON_HALO): before every update each halo cell of the state it
    writes is NaN, and each loaded field's halo too.  One rank keeps its halo by three mechanisms
    (x faces from the update epilogue, y rows copied, z planes fetched through the TMA coordinate
    wrap and never stored) and never exchanges corners: if any stencil read a cell
    none of them refreshed, NaN would spread.  The state after 2 RK3 steps is bit-identical to the
    run without poison (nx = 12: the direct kernel)."""
    import paper_2103_01597_b200 as b2
    st = synth.pcg64_state((n[2], n[1], n[0]), dtype=np.float64 if dtype == 8 else np.float32)
    outs = []
    for debug in (0, b2.MHD_DEBUG_POISON_HALO):
        m, _ = _mesh(n, radius=r, dtype=dtype)
        m.set_debug(debug)
        m.load(st)
        for _ in range(2):
            m.step(1e-4)
        outs.append(m.store().cpu().numpy())
        if debug:  # the poison is really there: the corners of the current state are NaN
            grid = m.store_grid().numpy()
            assert np.all(np.isnan(grid[:, :r, :r, :r]))
        m.close()
    assert np.all(np.isfinite(outs[1]))
    assert np.array_equal(outs[0], outs[1])


def test_poison_halo_exchange_bitwise():
    """With the poison on, an explicit exchange refills every non-corner halo cell bitwise."""
    import paper_2103_01597_b200 as b2
    n = (37, 23, 19)
    m, _ = _mesh(n)
    m.set_debug(b2.MHD_DEBUG_POISON_HALO)
    nz, ny, nx = n[2], n[1], n[0]
    st = (np.arange(8)[:, None, None, None] * 1e6 + np.arange(nz * ny * nx).reshape(nz, ny, nx)).astype(np.float64)
    m.load(st)
    m.halo_exchange()
    grid = m.store_grid().numpy()
    expect = np.stack([oracle.periodic_fill(oracle.with_halo(st[q])) for q in range(8)])
    mask = np.ones(grid.shape[1:], bool)
    for zs in (slice(0, 3), slice(-3, None)):
        for ys in (slice(0, 3), slice(-3, None)):
            for xs in (slice(0, 3), slice(-3, None)):
                mask[zs, ys, xs] = False
    assert np.array_equal(grid[:, mask], expect[:, mask])
    assert np.all(np.isnan(grid[:, ~mask]))
    m.close()


@pytest.mark.parametrize("n,r", [((64, 24, 19), 3), ((48, 20, 18), 4)])
def test_xface_wrap_store_bit_identical(n, r, monkeypatch):
    """One rank: the x/y halo written by the plain kernel's predicated epilogue stores and the z
    planes wrapped by TMA (the default, B2MHD_XWRAP=1) give the same state, bit for bit, as the
    self-copy schedule (B2MHD_XWRAP=0)."""
    st = synth.pcg64_state((n[2], n[1], n[0]))
    out = []
    for xw in ("0", "1"):
        monkeypatch.setenv("B2MHD_XWRAP", xw)
        m, _ = _mesh(n, radius=r)
        m.load(st)
        for _ in range(2):
            m.step(1e-3)
        out.append(m.store().cpu().numpy())
        m.close()
    assert np.array_equal(out[0], out[1])


@pytest.mark.parametrize("xwrap", ["0", "1"])
def test_debug_rhs_after_steps(xwrap, monkeypatch):
    """The RHS of a state reached by substeps (whose halo comes from the schedule's own
    machinery: x faces from the previous epilogue, y rows copied, z planes wrapped by TMA) equals
    the oracle's RHS of the stored interior; then stepping on gives the same state as a fresh
    load of that interior."""
    monkeypatch.setenv("B2MHD_XWRAP", xwrap)
    n = (64, 24, 19)
    m, ds = _mesh(n, params=PSTRONG)
    st = synth.pcg64_state((n[2], n[1], n[0]))
    m.load(st)
    m.step(1e-4)
    m.step(1e-4)
    cur = m.store().cpu().numpy()
    got = m.debug_rhs().cpu().numpy()
    ref = oracle.rhs(cur, ds, PSTRONG)
    assert _norm_err(got, ref) <= 1e-12
    m.step(1e-4)
    a = m.store().cpu().numpy()
    m.load(cur)
    m.step(1e-4)
    assert np.array_equal(m.store().cpu().numpy(), a)
    m.close()


def test_async_io_dtype_conversion():
    """store_async into an FP32 host buffer from an FP64 mesh and load_async of FP32 host data
    into it: the same values as the blocking calls with the same conversions."""
    import torch
    import paper_2103_01597_b200 as b2
    n = (40, 24, 19)
    m, _ = _mesh(n)
    st = synth.pcg64_state((n[2], n[1], n[0]))
    m.load(st)
    out32 = torch.empty((8, n[2], n[1], n[0]), dtype=torch.float32).pin_memory()
    m.store_async(out32)
    m.synchronize()
    assert np.array_equal(out32.numpy(), st.astype(np.float32))
    src32 = torch.from_numpy(st.astype(np.float32)).pin_memory()
    m.load_async(src32)
    m.synchronize()
    assert np.array_equal(m.store().cpu().numpy(), st.astype(np.float32).astype(np.float64))
    m.close()


# ---- RHS parity ------------------------------------------------------------------------------------
@pytest.mark.parametrize("params", [synth.P0, PSTRONG], ids=["P0", "strong"])
@pytest.mark.parametrize("n,box", [((32, 32, 32), None), ((40, 32, 24), (2 * math.pi, 4 * math.pi, 6 * math.pi)),
                                   ((37, 29, 19), None)])
def test_rhs_parity_fp64(params, n, box):
    ds = synth.spacing(n, box)
    m, _ = _mesh(n, ds, params)
    st = synth.pcg64_state((n[2], n[1], n[0]))
    m.load(st)
    got = m.debug_rhs().cpu().numpy()
    ref = oracle.rhs(st, ds, params)
    assert _norm_err(got, ref) <= 1e-12
    m.close()


def test_rhs_parity_fp32():
    n = (32, 24, 20)
    ds = synth.spacing(n)
    m, _ = _mesh(n, ds, dtype=4)
    st = synth.pcg64_state((n[2], n[1], n[0]), dtype=np.float32)
    m.load(st)
    got = m.debug_rhs().cpu().numpy().astype(np.float64)
    ref = oracle.rhs(st.astype(np.float64), ds, synth.P0)
    assert _norm_err(got, ref) <= 1e-4
    m.close()


# ---- 10 full RK3 steps (north star) -------------------------------------------------------------------
@pytest.mark.parametrize("n,box,steps", [((32, 32, 32), None, 10),
                                         ((40, 32, 24), (2 * math.pi, 4 * math.pi, 6 * math.pi), 4),
                                         ((37, 29, 19), None, 3)])
def test_steps_parity_fp64(n, box, steps):
    ds = synth.spacing(n, box)
    m, _ = _mesh(n, ds)
    st = synth.pcg64_state((n[2], n[1], n[0]))
    m.load(st)
    for _ in range(steps):
        m.step(synth.DT)
    got = m.store().cpu().numpy()
    ref = oracle.integrate(st, ds, synth.P0, synth.DT, steps)
    assert _field_err(got, ref) <= 1e-11
    ref_ld = oracle.integrate(st, ds, synth.P0, synth.DT, steps, kind="ld")
    inc = (ref_ld - st.astype(np.longdouble)).astype(np.float64)
    assert _norm_err(got - st, inc) <= 1e-9
    m.close()


def test_steps_parity_fp32():
    n = (32, 32, 32)
    ds = synth.spacing(n)
    m, _ = _mesh(n, ds, dtype=4)
    st = synth.pcg64_state((n[2], n[1], n[0]), dtype=np.float32)
    m.load(st)
    for _ in range(10):
        m.step(synth.DT)
    got = m.store().cpu().numpy().astype(np.float64)
    ref = oracle.integrate(st.astype(np.float64), ds, synth.P0, synth.DT, 10)
    assert _field_err(got, ref) <= 1e-4
    _fp32_increment_ok(got, ref, st.astype(np.float64), 30)
    m.close()


def test_fp32_128_multichunk():
    """FP32 at 128^3 on one GPU: the 32 x 16 FP32 tile over several 64-plane z chunks, in the
    launch configuration bench.py --dtype f32 uses; RHS, one RK3 step and its increment against
    the double oracle fed the FP32-rounded state (R#18)."""
    import os
    oracle.set_threads(os.cpu_count() or 1)
    n = (128, 128, 128)
    ds = synth.spacing(n)
    m, _ = _mesh(n, ds, dtype=4)
    st = synth.splitmix_state((128, 128, 128), (0, 0, 0), (128, 128, 128), dtype=np.float32)
    st64 = st.astype(np.float64)
    m.load(st)
    got_rhs = m.debug_rhs().cpu().numpy().astype(np.float64)
    assert _norm_err(got_rhs, oracle.rhs(st64, ds, synth.P0)) <= 1e-4
    m.step(synth.DT)
    got = m.store().cpu().numpy().astype(np.float64)
    m.close()
    ref = oracle.integrate(st64, ds, synth.P0, synth.DT, 1)
    assert _field_err(got, ref) <= 1e-4
    _fp32_increment_ok(got, ref, st64, 3)


def test_substep_level_parity_and_rk3_order():
    """After each single substep the state matches the oracle (exercises the reconstructed-w
    form for k = 1, 2 separately, reading R#4)."""
    n = (24, 24, 24)
    ds = synth.spacing(n)
    m, _ = _mesh(n, ds, PSTRONG)
    st = synth.pcg64_state((n[2], n[1], n[0]))
    m.load(st)
    dt = 1e-4
    for sub in range(1, 7):
        m.substep((sub - 1) % 3, dt)
        got = m.store().cpu().numpy()
        ref = oracle.integrate(st, ds, PSTRONG, dt, 0, substeps=sub)
        assert _norm_err(got - st, ref - st) <= 1e-10, sub
    m.close()


# ---- kernels agree bit for bit ---------------------------------------------------------------------------
@pytest.mark.parametrize("n", [(64, 48, 40), (70, 43, 150)])
def test_kernel_variants_bit_identical(n):
    """direct (1), z-marching (2) and warp-specialised z-marching (3) kernels: bit-identical RHS
    and states after two RK3 steps, on a tiled box and on a ragged one with several z chunks"""
    from paper_2103_01597_b200 import MhdError
    st = synth.pcg64_state((n[2], n[1], n[0]))
    outs, rhss = [], []
    for variant in (1, 2, 3):
        m, ds = _mesh(n)
        try:
            m.set_kernel(variant)
        except MhdError:
            m.close()
            if variant == 3:
                continue
            pytest.skip("z-marching kernel not available for this geometry")
        m.load(st)
        rhss.append(m.debug_rhs().cpu().numpy())
        for _ in range(2):
            m.step(synth.DT)
        outs.append(m.store().cpu().numpy())
        m.close()
    assert len(outs) == 3, "warp-specialised kernel unavailable for an FP64 order-6 mesh"
    for o, r in zip(outs[1:], rhss[1:]):
        assert np.array_equal(outs[0], o)
        assert np.array_equal(rhss[0], r)


# ---- ABI state machine, reductions --------------------------------------------------------------------
def test_substep_order_enforced():
    from paper_2103_01597_b200 import MhdError
    m, _ = _mesh((16, 16, 16))
    m.load(synth.pcg64_state((16, 16, 16)))
    with pytest.raises(MhdError) as e:
        m.substep(1, synth.DT)
    assert e.value.status == 9
    m.substep(0, synth.DT)
    with pytest.raises(MhdError):
        m.substep(2, synth.DT)
    m.close()


def test_reductions():
    import paper_2103_01597_b200 as b2
    n = (24, 20, 16)
    m, _ = _mesh(n)
    st = synth.pcg64_state((n[2], n[1], n[0]))
    m.load(st)
    for q in (0, 3, 7):
        assert m.reduce(q, b2.MHD_MIN) == st[q].min()
        assert m.reduce(q, b2.MHD_MAX) == st[q].max()
        assert abs(m.reduce(q, b2.MHD_SUM) - st[q].sum()) <= 1e-12 * st[q].size
        assert abs(m.reduce(q, b2.MHD_RMS) - math.sqrt((st[q] ** 2).mean())) <= 1e-13
        assert abs(m.reduce(q, b2.MHD_SUM_EXP) - np.exp(st[q]).sum()) <= 1e-12 * st[q].size
    bad = st.copy()
    bad[2, 3, 4, 5] = np.nan
    m.load(bad)
    with pytest.raises(b2.MhdError) as e:
        m.reduce(2, b2.MHD_SUM)
    assert e.value.status == 8
    m.close()


# ---- full size (BASELINE configs[1]: 256^3, the bench launch configuration) -------------------------------
def test_full_size_256_rhs_and_substep():
    """256^3 FP64 on one GPU, in the configuration bench.py times: the RHS of every cell and one
    substep k = 0 against the oracle (OpenMP over z on the host cores)."""
    import os
    oracle.set_threads(os.cpu_count() or 1)
    n = (256, 256, 256)
    ds = synth.spacing(n)
    m, _ = _mesh(n, ds)
    st = synth.splitmix_state((256, 256, 256), (0, 0, 0), (256, 256, 256))
    m.load(st)
    got_rhs = m.debug_rhs().cpu().numpy()
    ref, ref_rhs = oracle.integrate(st, ds, synth.P0, synth.DT, 0, substeps=1, return_rhs=True)
    assert _norm_err(got_rhs, ref_rhs) <= 1e-12
    del got_rhs, ref_rhs
    m.substep(0, synth.DT)
    got = m.store().cpu().numpy()
    assert _field_err(got, ref) <= 1e-11
    assert _norm_err(got - st, ref - st) <= 1e-10
    m.close()


def test_full_size_512_rhs_and_substep():
    """512^3 FP64 on one GPU (BASELINE configs[2] at N = 1, 17.8 GB of state) in bench.py's launch
    configuration: the RHS of every cell and one substep k = 0 against the oracle on the host cores
    (≈ 50 GB of host memory)."""
    import os
    oracle.set_threads(os.cpu_count() or 1)
    n = (512, 512, 512)
    ds = synth.spacing(n)
    m, _ = _mesh(n, ds)
    st = synth.splitmix_state((512, 512, 512), (0, 0, 0), (512, 512, 512))
    m.load(st)
    got_rhs = m.debug_rhs().cpu().numpy()
    ref, ref_rhs = oracle.integrate(st, ds, synth.P0, synth.DT, 0, substeps=1, return_rhs=True)
    assert _norm_err(got_rhs, ref_rhs) <= 1e-12
    del got_rhs, ref_rhs
    m.substep(0, synth.DT)
    got = m.store().cpu().numpy()
    m.close()
    assert _field_err(got, ref) <= 1e-11
    assert _norm_err(got - st, ref - st) <= 1e-10


def test_paper_ulp_analog_256():
    """The paper's own verification: one RK3 step of a 256^3 grid of random [0, 1]
    values against the single-core CPU model, error in ulps of the model value (Eqs. 15-16,
    p = 53).  The paper reports <= 2 ulps everywhere for a logically identical CPU solver; ours
    evaluates w in another algebraic form (R#4), so the bar is >= 99.5 % of values within 2 ulps
    in every field and <= 4 ulps everywhere for A (whose increment is small).  Measured on B200:
    A <= 3, lnrho <= 6 ulps; u and s exceed 2 ulps on 0.3 % / 0.2 % of cells, where the large
    j x B / rho and ohmic-heating increments at 256^3 cancel against f (tools/ulp_check.py).
    The binding checks at this size are the north-star ones: fields <= 1e-11 (R#18) and
    increments <= 1e-9 against the long-double oracle."""
    import os
    oracle.set_threads(os.cpu_count() or 1)
    n = (256, 256, 256)
    ds = synth.spacing(n)
    st = synth.pcg64_state(n)
    m, _ = _mesh(n, ds)
    m.load(st)
    m.step(synth.DT)
    got = m.store().cpu().numpy()
    m.close()
    ref = oracle.integrate(st, ds, synth.P0, synth.DT, 1)
    # the north-star tolerances at the benched size (R#18): fields vs the double oracle,
    # increments vs the long-double oracle
    assert _field_err(got, ref) <= 1e-11
    ref_ld = oracle.integrate(st, ds, synth.P0, synth.DT, 1, kind="ld")
    inc_ld = (ref_ld - st.astype(np.longdouble)).astype(np.float64)
    del ref_ld
    assert _norm_err(got - st, inc_ld) <= 1e-9
    del inc_ld
    # the same step with the oracle's arithmetic but the two-state RK3 form the GPU stores (R#4)
    w2 = oracle.integrate(st, ds, synth.P0, synth.DT, 1, form="w2")

    def ulps_of(model, cand):
        eps = np.exp2(np.floor(np.log2(np.abs(model))) - 52)  # Eq. 15
        return np.abs(model - cand) / eps                       # Eq. 16

    for q in range(8):
        mq, cq = ref[q].ravel(), got[q].ravel()
        assert np.all(mq != 0)
        ulps = ulps_of(mq, cq)
        assert np.mean(ulps <= 2.0) >= 0.995, (q, float(np.mean(ulps <= 2.0)))
        if q >= 5:
            assert ulps.max() <= 4.0, (q, float(ulps.max()))
        # attribution of the > 2-ulp values: they sit where f + dt RHS cancels; the oracle's own
        # arithmetic, only rearranged into the two-state RK3 form (R#4), misses the 2-ulp bar at
        # such cells too (measured: u 0.17 %, up to 4.6e4 ulps; s 0.03 %; GPU: u 0.28 %, s 0.19 %,
        # profiles/r02/ulp_check_w2.json), so the bar is a property of the arrangement of the
        # arithmetic, not of the GPU path
        out_gpu = int(np.sum(ulps > 2.0))
        out_w2 = int(np.sum(ulps_of(mq, w2[q].ravel()) > 2.0))
        if out_gpu >= 1000:
            assert out_w2 >= 0.1 * out_gpu, (q, out_gpu, out_w2)


# ---- stencil orders 2, 4, 6, 8 -------------------------------------------------------------
@pytest.mark.parametrize("r", [1, 2, 3, 4])
def test_orders_rhs_steps_and_kernels(r):
    """Every order: RHS parity, 3 RK3 steps parity, and the direct, z-marching and (radius 3, 4)
    warp-specialised kernels agree bit for bit."""
    import paper_2103_01597_b200 as b2
    from paper_2103_01597_b200 import MhdError
    n = (40, 28, 24)
    ds = synth.spacing(n)
    st = synth.pcg64_state((n[2], n[1], n[0]))
    outs = []
    for variant in (1, 2, 3):
        m, _ = _mesh(n, ds, PSTRONG, radius=r)
        try:
            m.set_kernel(variant)
        except MhdError:
            # z-march single group at FP64 radius 4 runs on a 32 x 4 tile; the warp-specialised
            # kernel exists for radius 3 and 4 only
            assert (variant == 2 and r == 4) or (variant == 3 and r < 3)
            m.close()
            continue
        m.load(st)
        got = m.debug_rhs().cpu().numpy()
        ref = oracle.rhs(st, ds, PSTRONG, r=r)
        assert _norm_err(got, ref) <= 1e-12, (r, variant)
        for _ in range(3):
            m.step(1e-5)
        outs.append(m.store().cpu().numpy())
        m.close()
    ref = oracle.integrate(st, ds, PSTRONG, 1e-5, 3, r=r)
    for o in outs:
        assert _field_err(o, ref) <= 1e-11
        assert _norm_err(o - st, ref - st) <= 1e-9
    for o in outs[1:]:
        assert np.array_equal(outs[0], o)


@pytest.mark.parametrize("r", [1, 2, 3, 4])
@pytest.mark.parametrize("n", [(40, 28, 24), (37, 23, 70)])
def test_fp32_kernels_bit_identical(r, n):
    """FP32: the z-marching kernel (two cells per thread in FP32x2 instructions at r <= 3) and the
    direct kernel (one cell per thread, scalar FP32) give bit-identical RHS and states, on a tiled
    box and on a ragged one whose tile rows are half empty and whose z spans several chunks"""
    ds = synth.spacing(n)
    st = synth.pcg64_state((n[2], n[1], n[0]), dtype=np.float32)
    outs, rhss = [], []
    for variant in (1, 2):
        m, _ = _mesh(n, ds, PSTRONG, dtype=4, radius=r)
        m.set_kernel(variant)
        m.load(st)
        rhss.append(m.debug_rhs().cpu().numpy())
        for _ in range(2):
            m.step(1e-5)
        outs.append(m.store().cpu().numpy())
        m.close()
    assert np.array_equal(rhss[0], rhss[1])
    assert np.array_equal(outs[0], outs[1])


@pytest.mark.parametrize("r", [1, 4])
def test_orders_halo_sentinel_bitwise(r):
    n = (20, 18, 16)
    m, _ = _mesh(n, radius=r, exchange_corners=True)
    nz, ny, nx = n[2], n[1], n[0]
    st = (np.arange(8)[:, None, None, None] * 1e6 + np.arange(nz * ny * nx).reshape(nz, ny, nx)).astype(np.float64)
    m.load(st)
    m.halo_exchange()
    grid = m.store_grid().numpy()
    expect = np.stack([oracle.periodic_fill(oracle.with_halo(st[q], r), r=r) for q in range(8)])
    assert np.array_equal(grid, expect)
    m.close()


def test_order8_fp32_zmarch():
    n = (40, 24, 20)
    ds = synth.spacing(n)
    m, _ = _mesh(n, ds, dtype=4, radius=4)
    m.set_kernel(2)
    st = synth.pcg64_state((n[2], n[1], n[0]), dtype=np.float32)
    m.load(st)
    got = m.debug_rhs().cpu().numpy().astype(np.float64)
    ref = oracle.rhs(st.astype(np.float64), ds, synth.P0, r=4)
    assert _norm_err(got, ref) <= 1e-4
    m.close()
