"""N > 1 host logic on CPU: world_size 2/4/8 gloo processes exchange halos driven by the
library's own segment tables (mhd_segment_table: Morton mapping P:557, 26 segments P:705,
per-peer concatenation), with the staging-buffer layout the CUDA pack/unpack kernels use
(per segment: field-major, then z, y, x).  The resulting halo-inclusive subgrid of every rank
must equal the oracle's periodic wrap of the global grid, bit for bit."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, N_xyz, corners, q_out):
    import sys
    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist

    import synth
    from oracle import geometry as G
    from paper_2103_01597_b200 import _native as nat

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        info = nat.make_info(N_xyz, (0.1, 0.1, 0.1), synth.P0, nranks=world, rank=rank, exchange_corners=corners)
        P, c, n = nat.mhd_decompose(info, rank)
        segs = nat.mhd_segment_table(info, rank)
        Nz, Ny, Nx = N_xyz[2], N_xyz[1], N_xyz[0]
        glob = (np.arange(8)[:, None, None, None] * (Nz * Ny * Nx)
                + np.arange(Nz * Ny * Nx).reshape(Nz, Ny, Nx)[None]).astype(np.float64)
        Pz, cz = (P[2], P[1], P[0]), (c[2], c[1], c[0])
        grid = np.full((8, n[2] + 6, n[1] + 6, n[0] + 6), np.nan)
        grid[:, 3:-3, 3:-3, 3:-3] = G.local_interior(glob, Pz, cz)

        def box(first, ext):
            return (slice(None),) + tuple(slice(first[a] + 3, first[a] + 3 + ext[a]) for a in (2, 1, 0))

        sendbufs, recvbufs = {}, {}
        for s in segs:
            if s["send_peer"] == rank:
                grid[box(s["dst_first"], s["extent"])] = grid[box(s["src_first"], s["extent"])]
                continue
            cnt = int(np.prod(s["extent"]))
            sendbufs.setdefault(s["send_peer"], []).append((s["send_buf_cell"], grid[box(s["src_first"], s["extent"])].reshape(8, cnt)))
            recvbufs.setdefault(s["recv_peer"], []).append((s["recv_buf_cell"], s))
        reqs, rbufs = [], {}
        for peer, parts in sorted(sendbufs.items()):
            total = sum(p[1].shape[1] for p in parts)
            buf = np.empty(8 * total)
            for cell0, data in parts:
                buf[8 * cell0: 8 * cell0 + data.size] = data.reshape(-1)  # field-major per segment
            reqs.append(dist.isend(torch.from_numpy(buf), peer))
        for peer, parts in sorted(recvbufs.items()):
            total = sum(int(np.prod(s["extent"])) for _, s in parts)
            rbufs[peer] = torch.empty(8 * total, dtype=torch.float64)
            reqs.append(dist.irecv(rbufs[peer], peer))
        for r in reqs:
            r.wait()
        for peer, parts in recvbufs.items():
            b = rbufs[peer].numpy()
            for cell0, s in parts:
                cnt = int(np.prod(s["extent"]))
                ext = s["extent"]
                grid[box(s["dst_first"], ext)] = b[8 * cell0: 8 * cell0 + 8 * cnt].reshape(8, ext[2], ext[1], ext[0])
        expect = G.local_subgrid_with_halo(glob, Pz, cz)
        mask = np.ones(grid.shape[1:], bool)
        if not corners:
            for zs in (slice(0, 3), slice(-3, None)):
                for ys in (slice(0, 3), slice(-3, None)):
                    for xs in (slice(0, 3), slice(-3, None)):
                        mask[zs, ys, xs] = False
        ok = bool(np.array_equal(grid[:, mask], expect[:, mask]))
        q_out.put((rank, ok, P))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,N", [(2, (12, 10, 16)), (4, (12, 14, 16)), (8, (14, 16, 18))])
@pytest.mark.parametrize("corners", [False, True])
def test_gloo_halo_exchange_matches_periodic_wrap(world, N, corners):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, N, corners, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    assert all(ok for _, ok, _ in res), res
