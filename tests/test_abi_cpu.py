"""C ABI checks that need no GPU: the library loads and exports every symbol include/b2mhd.h
declares; host-side decomposition and segment logic against the paper's definitions."""
import os
import re

import numpy as np
import pytest

import synth
from oracle import geometry as G

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _native():
    from paper_2103_01597_b200 import _native
    return _native


def test_library_exports_every_header_symbol():
    nat = _native()
    hdr = open(os.path.join(ROOT, "include", "b2mhd.h")).read()
    declared = set(re.findall(r"^(?:mhd_status|const char\*|int32_t)\s+(mhd_\w+)\s*\(", hdr, re.M))
    assert declared == set(nat.SYMBOLS), declared ^ set(nat.SYMBOLS)
    for name in declared:
        assert hasattr(nat.lib, name), name
    assert nat.mhd_abi_version() == nat.MHD_ABI_VERSION


def test_library_links_no_torch_and_is_sm100a():
    nat = _native()
    import subprocess
    deps = subprocess.run(["ldd", nat.LIB_PATH], capture_output=True, text=True).stdout
    assert "torch" not in deps and "libc10" not in deps
    sass = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", nat.LIB_PATH], capture_output=True,
                          text=True).stdout
    assert "sm_100a" in sass


def _info(n, nranks=1, corners=False, **kw):
    nat = _native()
    return nat.make_info(n, (0.1, 0.1, 0.1), synth.P0, nranks=nranks, exchange_corners=corners, **kw)


def test_decompose_matches_morton_p557():
    nat = _native()
    for cp in (1, 2, 4, 8, 16, 32, 64):
        info = _info((256, 256, 256), cp)
        Pm = G.partition(cp)  # Morton order: coordinate 0 -> z
        for r in range(cp):
            P, c, n = nat.mhd_decompose(info, r)
            assert P == (Pm[2], Pm[1], Pm[0])
            cm = G.morton_inverse(r)
            assert c == (cm[2], cm[1], cm[0])
            assert n == tuple(256 // p for p in P)


@pytest.mark.parametrize("n,nranks,status", [((256, 256, 256), 3, 2), ((255, 256, 256), 8, 2),
                                             ((12, 12, 12), 2, 3), ((7, 7, 7), 1, 0)])
def test_decompose_errors(n, nranks, status):
    nat = _native()
    import ctypes
    info = _info(n, nranks)
    st = nat.lib.mhd_decompose(ctypes.byref(info), 0, None, None, None)
    assert st == status, nat.mhd_last_error()


def test_unsupported_radius_and_dtype():
    nat = _native()
    import ctypes
    b = ctypes.c_size_t()
    for r, st in ((0, 4), (5, 4), (1, 0), (2, 0), (3, 0), (4, 0)):
        info = _info((32, 32, 32))
        info.radius = r  # orders 2, 4, 6, 8 are built
        assert nat.lib.mhd_workspace_bytes(ctypes.byref(info), ctypes.byref(b)) == st
    info = _info((32, 32, 32))
    info.dtype = 2
    assert nat.lib.mhd_workspace_bytes(ctypes.byref(info), ctypes.byref(b)) == 4


@pytest.mark.parametrize("n", [(64, 64, 64), (40, 32, 24), (256, 256, 256)])
@pytest.mark.parametrize("corners", [True, False])
def test_segments_tile_the_halo(n, corners):
    """26 segments (6 sides, 12 edges, 8 corners), disjoint, covering C_M' - C_N'
    (Eqs. 2-3); without corners the count drops by 8 r^3 = 216."""
    nat = _native()
    segs = nat.mhd_segment_table(_info(n, 1, corners), 0)
    kinds = [s["kind"] for s in segs]
    assert kinds.count(1) == 6 and kinds.count(2) == 12 and kinds.count(3) == (8 if corners else 0)
    total = sum(int(np.prod(s["extent"])) for s in segs)
    halo = G.halo_cells((n[2], n[1], n[0]))
    assert total == (halo if corners else halo - 216)
    # disjoint cover of the shell and the P:705 map s' = ((s - r) mod n') + r on every axis
    if max(n) <= 64:
        cover = np.zeros((n[2] + 6, n[1] + 6, n[0] + 6), dtype=np.int32)
        for s in segs:
            sl = tuple(slice(s["dst_first"][a] + 3, s["dst_first"][a] + 3 + s["extent"][a]) for a in (2, 1, 0))
            cover[sl] += 1
            for a in range(3):
                for i in range(s["extent"][a]):
                    dst = s["dst_first"][a] + i + 3  # halo-inclusive index s
                    src = s["src_first"][a] + i + 3
                    assert src == ((dst - 3) % n[a]) + 3
        assert cover[3:-3, 3:-3, 3:-3].sum() == 0
        shell = cover.copy()
        shell[3:-3, 3:-3, 3:-3] = 1
        if corners:
            assert np.all(shell == 1)
        else:
            assert np.all(shell <= 1) and (shell == 0).sum() == 216


@pytest.mark.parametrize("r", [1, 2, 4])
def test_segments_other_orders(r):
    """Segment extents follow the radius: the halo of width r is tiled exactly (Eqs. 2-3)."""
    nat = _native()
    n = (20, 18, 16)
    info = nat.make_info(n, (0.1,) * 3, synth.P0, exchange_corners=True, radius=r)
    segs = nat.mhd_segment_table(info, 0)
    total = sum(int(np.prod(s["extent"])) for s in segs)
    assert total == (n[0] + 2 * r) * (n[1] + 2 * r) * (n[2] + 2 * r) - n[0] * n[1] * n[2]
    assert all(e in (r, nv) for s in segs for e, nv in zip(s["extent"], n))


def test_largest_segment_is_12MiB_at_256():
    """the largest individual halo segment at 256^3 is 12 MiB (8 fields x 8 B)."""
    nat = _native()
    segs = nat.mhd_segment_table(_info((256, 256, 256), 1), 0)
    assert max(int(np.prod(s["extent"])) for s in segs) * 8 * 8 == 12 * 2 ** 20


@pytest.mark.parametrize("nranks", [2, 4, 8])
@pytest.mark.parametrize("corners", [True, False])
def test_send_and_recv_lists_match_across_ranks(nranks, corners):
    """What rank A sends to B is, segment by segment and in order, what B expects from A."""
    nat = _native()
    info = _info((64, 64, 64), nranks, corners)
    tables = [nat.mhd_segment_table(info, r) for r in range(nranks)]
    for a in range(nranks):
        for b in range(nranks):
            if a == b:
                continue
            sends = [s for s in tables[a] if s["send_peer"] == b and s["send_peer"] != a]
            recvs = [s for s in tables[b] if s["recv_peer"] == a and s["recv_peer"] != b]
            assert [s["offset"] for s in sends] == [s["offset"] for s in recvs]
            assert [s["extent"] for s in sends] == [s["extent"] for s in recvs]
            assert [s["send_buf_cell"] for s in sends] == [s["recv_buf_cell"] for s in recvs]


def test_distinct_peers_per_rank():
    """Morton (2,1,1)/(2,2,1)/(2,2,2) gives 1/3/7 distinct remote peers per rank."""
    nat = _native()
    for nranks, peers in ((2, 1), (4, 3), (8, 7)):
        for corners in (True, False):
            segs = nat.mhd_segment_table(_info((64, 64, 64), nranks, corners), 0)
            got = {s["send_peer"] for s in segs if s["send_peer"] != 0}
            # the diagonal (1,1,1) neighbour at 8 ranks is reached only through corners
            assert len(got) == (peers if (corners or nranks < 8) else 6)
