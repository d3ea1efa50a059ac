"""Multi-rank hot path on ONE GPU: every rank of a 2/4/8-rank Morton decomposition driven by one
process (`Group`, mhd_group_*).  The ranks run the multi-GPU schedules and kernels of P:765-782 —
pack / transfer / unpack (a1-a3; the transfer is a copy-engine pull instead of NCCL), the
peer-memory boundary copy (8(f)1), the inner/outer split (a7) — on one device, ordered by CUDA
events instead of the cross-process flags, so the driver's 1-GPU box exercises them.

Checks (SURVEY 8(c) "Halo / indexing", R#19): the halo exchange of a sentinel field is bitwise the
global periodic wrap on every rank, repeated with fresh values; P ranks reproduce
the 1-rank result bit for bit; and the oracle within the north-star tolerance.  The NaN-poison
mode (MHD_DEBUG_POISON_HALO) runs underneath several of them: every halo cell of the state an
update writes is NaN beforehand, so a cell that the schedule fails to refresh before a stencil
reads it (or a corner, which P:937 says is never needed) would show."""
import numpy as np
import pytest

import oracle
import synth
from oracle import geometry as G

pytestmark = pytest.mark.gpu

# (x, y, z) grids per rank count: local extents of several tiles with an inner segment
GRID = {2: (40, 36, 48), 4: (40, 48, 48), 8: (64, 48, 48)}


def _group(N, nranks, exchange, dtype=None, **kw):
    import torch

    import paper_2103_01597_b200 as b2
    torch.cuda.set_device(0)
    return b2.Group(N, synth.spacing(N), kw.pop("params", synth.P0), dtype or b2.MHD_F64, nranks=nranks,
                    exchange=exchange, **kw)


def _single(N, st, steps, dt, dtype=None, radius=3, params=synth.P0):
    import torch

    import paper_2103_01597_b200 as b2
    torch.cuda.set_device(0)
    m = b2.Mesh(N, synth.spacing(N), params, dtype or b2.MHD_F64, radius=radius)
    m.load(st)
    for _ in range(steps):
        m.step(dt)
    out = m.store().cpu().numpy()
    m.close()
    return out


def _field_err(g, o):
    return max(float(np.max(np.abs(g[q] - o[q]) / np.maximum(np.abs(o[q]), 1e-3 * np.max(np.abs(o[q])))))
               for q in range(8))


def _corner_mask(shape, r):
    mask = np.ones(shape, bool)
    for zs in (slice(0, r), slice(-r, None)):
        for ys in (slice(0, r), slice(-r, None)):
            for xs in (slice(0, r), slice(-r, None)):
                mask[zs, ys, xs] = False
    return mask


def _sentinel(N, rep, f32=False):
    Nx, Ny, Nz = N
    idx = np.arange(Nz * Ny * Nx).reshape(Nz, Ny, Nx)[None]
    if f32:
        return (np.arange(8)[:, None, None, None] * 1e5 + idx + rep * 1e6).astype(np.float32)
    return (np.arange(8)[:, None, None, None] * 1e7 + idx + rep * 1e9).astype(np.float64)


@pytest.mark.parametrize("nranks", [2, 4, 8])
@pytest.mark.parametrize("exchange", ["packed", "p2p"])
@pytest.mark.parametrize("corners", [False, True])
def test_group_halo_sentinel_bitwise(nranks, exchange, corners):
    """Sentinel = global linear index; after the exchange every halo cell of every rank holds the
    wrapped global value, bitwise (8 repetitions with fresh values: a race shows as a stale cell).
    With corners off the corner cells are left poisoned (NaN) and excluded."""
    import paper_2103_01597_b200 as b2
    N = GRID[nranks]
    g = _group(N, nranks, exchange, exchange_corners=corners, debug=b2.MHD_DEBUG_POISON_HALO)
    for rep in range(8):
        glob = _sentinel(N, rep)
        g.load(glob)
        g.halo_exchange()
        for m, grid in zip(g.meshes, g.store_grids()):
            grid = grid.numpy()
            expect = G.local_subgrid_with_halo(glob, tuple(reversed(m.P)), tuple(reversed(m.coord)), r=3)
            mask = np.ones(grid.shape[1:], bool) if corners else _corner_mask(grid.shape[1:], 3)
            assert np.array_equal(grid[:, mask], expect[:, mask]), (rep, m.coord)
            if not corners:
                assert np.all(np.isnan(grid[:, ~mask])), "corners are not exchanged: they stay poisoned"
    g.close()


@pytest.mark.parametrize("nranks", [2, 4, 8])
@pytest.mark.parametrize("exchange", ["packed", "p2p"])
def test_group_steps_bit_identical_and_oracle(nranks, exchange):
    """3 RK3 steps on P ranks (halos poisoned before every update) = the 1-rank run bit for bit,
    and the oracle within 1e-11 (R#18)."""
    import paper_2103_01597_b200 as b2
    N = GRID[nranks]
    st = synth.pcg64_state((N[2], N[1], N[0]))
    g = _group(N, nranks, exchange, debug=b2.MHD_DEBUG_POISON_HALO)
    g.load(st)
    for _ in range(3):
        g.step(synth.DT)
    got = g.store()
    g.close()
    one = _single(N, st, 3, synth.DT)
    assert np.array_equal(got, one)
    ref = oracle.integrate(st, synth.spacing(N), synth.P0, synth.DT, 3)
    assert _field_err(got, ref) <= 1e-11


@pytest.mark.parametrize("nranks", [4, 8])
def test_group_p2p_coarse_arrival_same_bits(nranks, monkeypatch):
    """The round-1 peer-memory schedule (one wait for every neighbour before the first boundary
    slab, B2MHD_FINE_ARRIVAL=0) and the per-slab arrival schedule give the same bits."""
    import paper_2103_01597_b200 as b2
    N = GRID[nranks]
    st = synth.pcg64_state((N[2], N[1], N[0]))
    outs = []
    for fine in ("0", "1"):
        monkeypatch.setenv("B2MHD_FINE_ARRIVAL", fine)
        g = _group(N, nranks, "p2p", debug=b2.MHD_DEBUG_POISON_HALO)
        g.load(st)
        for _ in range(2):
            g.step(synth.DT)
        outs.append(g.store())
        g.close()
    assert np.array_equal(outs[0], outs[1])


@pytest.mark.parametrize("exchange", ["packed", "p2p"])
def test_group_corners_on_same_result(exchange):
    """Exchanging the corner segments changes nothing (Eq. 14 has no 3-D corner points)."""
    N = GRID[8]
    st = synth.pcg64_state((N[2], N[1], N[0]))
    outs = []
    for corners in (False, True):
        g = _group(N, 8, exchange, exchange_corners=corners)
        g.load(st)
        for _ in range(2):
            g.step(1e-4)
        outs.append(g.store())
        g.close()
    assert np.array_equal(outs[0], outs[1])


def test_group_thin_x_direct_kernel():
    """local nx' = 12 is too narrow for the z-marching kernel, so every region
    runs the direct kernel, which must also write the periodic x faces it claims (x_valid).  2 and
    4 ranks, both exchanges: bitwise equal to one rank, and the oracle."""
    import paper_2103_01597_b200 as b2
    for nranks, N in ((2, (12, 40, 32)), (4, (12, 48, 48))):
        st = synth.pcg64_state((N[2], N[1], N[0]))
        one = _single(N, st, 2, 1e-4)
        for exchange in ("packed", "p2p"):
            g = _group(N, nranks, exchange, debug=b2.MHD_DEBUG_POISON_HALO)
            g.load(st)
            for _ in range(2):
                g.step(1e-4)
            got = g.store()
            g.close()
            assert np.array_equal(got, one), (nranks, exchange)
        ref = oracle.integrate(st, synth.spacing(N), synth.P0, 1e-4, 2)
        assert _field_err(one, ref) <= 1e-11


@pytest.mark.parametrize("exchange", ["packed", "p2p"])
def test_group_rhs_and_reductions(exchange):
    """RHS of every rank (mhd_group_debug_rhs) against the oracle's (<= 1e-12), then global
    reductions combined over the ranks."""
    import paper_2103_01597_b200 as b2
    N = GRID[4]
    ds = synth.spacing(N)
    st = synth.pcg64_state((N[2], N[1], N[0]))
    g = _group(N, 4, exchange)
    g.load(st)
    got = g.debug_rhs()
    ref = oracle.rhs(st, ds, synth.P0)
    assert max(float(np.max(np.abs(got[q] - ref[q])) / np.max(np.abs(ref[q]))) for q in range(8)) <= 1e-12
    g.step(1e-4)  # the RHS pass did not disturb the state machine
    cur = g.store()
    for q in (0, 4, 7):
        assert g.reduce(q, b2.MHD_MIN) == cur[q].min()
        assert g.reduce(q, b2.MHD_MAX) == cur[q].max()
        assert abs(g.reduce(q, b2.MHD_SUM) - cur[q].sum()) <= 1e-12 * cur[q].size
        assert abs(g.reduce(q, b2.MHD_SUM_EXP) - np.exp(cur[q]).sum()) <= 1e-12 * cur[q].size
    g.close()


@pytest.mark.parametrize("radius", [1, 2, 4])
def test_group_other_orders(radius):
    """Orders 2, 4, 8 on 4 ranks, peer-memory exchange: bitwise halo and 1-rank identity."""
    import paper_2103_01597_b200 as b2
    N = (40, 48, 48)
    g = _group(N, 4, "p2p", radius=radius, debug=b2.MHD_DEBUG_POISON_HALO)
    glob = _sentinel(N, 0)
    g.load(glob)
    g.halo_exchange()
    for m, grid in zip(g.meshes, g.store_grids()):
        grid = grid.numpy()
        expect = G.local_subgrid_with_halo(glob, tuple(reversed(m.P)), tuple(reversed(m.coord)), r=radius)
        mask = _corner_mask(grid.shape[1:], radius)
        assert np.array_equal(grid[:, mask], expect[:, mask])
    st = synth.pcg64_state((N[2], N[1], N[0]))
    g.load(st)
    for _ in range(2):
        g.step(1e-5)
    got = g.store()
    g.close()
    assert np.array_equal(got, _single(N, st, 2, 1e-5, radius=radius))


@pytest.mark.parametrize("nranks,exchange", [(2, "p2p"), (4, "packed"), (8, "p2p")])
def test_group_fp32(nranks, exchange):
    """FP32: bitwise halo (FP32-exact sentinels), P ranks = 1 rank bit for bit, oracle within 1e-4
    (R#18: the oracle is fed the FP32-rounded state)."""
    import paper_2103_01597_b200 as b2
    N = GRID[nranks]
    g = _group(N, nranks, exchange, dtype=b2.MHD_F32, debug=b2.MHD_DEBUG_POISON_HALO)
    glob = _sentinel(N, 1, f32=True)
    g.load(glob)
    g.halo_exchange()
    for m, grid in zip(g.meshes, g.store_grids()):
        grid = grid.numpy()
        expect = G.local_subgrid_with_halo(glob, tuple(reversed(m.P)), tuple(reversed(m.coord)), r=3)
        mask = _corner_mask(grid.shape[1:], 3)
        assert np.array_equal(grid[:, mask], expect[:, mask])
    st = synth.pcg64_state((N[2], N[1], N[0]), dtype=np.float32)
    g.load(st)
    for _ in range(3):
        g.step(synth.DT)
    got = g.store()
    g.close()
    assert np.array_equal(got, _single(N, st, 3, synth.DT, dtype=b2.MHD_F32))
    ref = oracle.integrate(st.astype(np.float64), synth.spacing(N), synth.P0, synth.DT, 3)
    assert _field_err(got.astype(np.float64), ref) <= 1e-4


def test_group_substep_order_and_exclusivity():
    """The group enforces k = 0, 1, 2 on every rank; a grouped mesh refuses per-mesh hot-path calls."""
    from paper_2103_01597_b200 import MhdError
    N = GRID[2]
    g = _group(N, 2, "p2p")
    g.load(synth.pcg64_state((N[2], N[1], N[0])))
    with pytest.raises(MhdError) as e:
        g.substep(1, synth.DT)
    assert e.value.status == 9
    with pytest.raises(MhdError) as e:
        g.meshes[0].substep(0, synth.DT)
    assert e.value.status == 1
    g.substep(0, synth.DT)
    g.close()


@pytest.mark.parametrize("nranks,exchange", [(1, None), (2, "p2p"), (4, "packed"), (8, "p2p")])
def test_minimal_subdomains(nranks, exchange):
    """The degenerate sizes: every subdomain axis n' = 2r + 1 = 7 (the smallest the method allows,
    n'_i > 2r; the inner segment is then empty along split axes and every update runs on the direct
    kernel), with every halo cell of an update's output poisoned: 2 RK3 steps against the oracle
    (R#18) and, for P > 1, bit for bit against one rank."""
    import paper_2103_01597_b200 as b2
    P = {1: (1, 1, 1), 2: (1, 1, 2), 4: (1, 2, 2), 8: (2, 2, 2)}[nranks]  # (x, y, z), Morton P:557
    N = tuple(7 * p for p in P)
    st = synth.pcg64_state((N[2], N[1], N[0]))
    one = _single(N, st, 2, synth.DT)
    ref = oracle.integrate(st, synth.spacing(N), synth.P0, synth.DT, 2)
    assert _field_err(one, ref) <= 1e-11
    if nranks > 1:
        g = _group(N, nranks, exchange, debug=b2.MHD_DEBUG_POISON_HALO)
        g.load(st)
        for _ in range(2):
            g.step(synth.DT)
        got = g.store()
        g.close()
        assert np.array_equal(got, one)


@pytest.mark.parametrize("radius", [1, 2, 4])
@pytest.mark.parametrize("nranks", [2, 8])
def test_group_fp32_other_orders(radius, nranks):
    """FP32 orders 2, 4, 8 on 2 and 8 ranks (peer memory, poisoned halos): P ranks = 1 rank bit for
    bit, and the oracle within 1e-4 (R#18)."""
    import paper_2103_01597_b200 as b2
    N = GRID[nranks]
    st = synth.pcg64_state((N[2], N[1], N[0]), dtype=np.float32)
    g = _group(N, nranks, "p2p", dtype=b2.MHD_F32, radius=radius, debug=b2.MHD_DEBUG_POISON_HALO)
    g.load(st)
    for _ in range(2):
        g.step(1e-5)
    got = g.store()
    g.close()
    assert np.array_equal(got, _single(N, st, 2, 1e-5, dtype=b2.MHD_F32, radius=radius))
    ref = oracle.integrate(st.astype(np.float64), synth.spacing(N), synth.P0, 1e-5, 2, r=radius)
    assert _field_err(got.astype(np.float64), ref) <= 1e-4


@pytest.mark.parametrize("nranks", [2, 8])
def test_group_warp_specialised_order6(nranks, monkeypatch):
    """The warp-specialised kernel (B2MHD_ZSPLIT=1) on the boundary slabs and inner segments of a
    multi-rank order-6 decomposition gives the same bits as the single-group kernel."""
    import paper_2103_01597_b200 as b2
    N = GRID[nranks]
    st = synth.pcg64_state((N[2], N[1], N[0]))
    outs = []
    for split in ("0", "1"):
        monkeypatch.setenv("B2MHD_ZSPLIT", split)
        g = _group(N, nranks, "p2p", debug=b2.MHD_DEBUG_POISON_HALO)
        g.load(st)
        for _ in range(2):
            g.step(synth.DT)
        outs.append(g.store())
        g.close()
    assert np.array_equal(outs[0], outs[1])
