"""Multi-GPU checks, run under torchrun (one process per GPU):

  1. halo exchange of a sentinel field (global linear index) is bit-exact against the oracle's
     periodic wrap of the global grid, on every rank;
  2. after `steps` RK3 steps the gathered P-GPU state is bit-identical to a 1-GPU run of the
     same global grid done by rank 0 on its own device, and matches the oracle (<= 1e-11 FP64;
     FP32 (MGPU_DTYPE=f32): <= 1e-4 against the oracle fed the FP32-rounded state, R#18).

Prints one JSON line per rank; exit code 0 iff every check passed.
"""
from __future__ import annotations

import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import numpy as np
    import torch
    import torch.distributed as dist

    import synth
    import paper_2103_01597_b200 as b2
    from oracle import geometry as G

    rank = int(os.environ["RANK"])
    world = int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    N = tuple(int(v) for v in os.environ.get("MGPU_N", "48,40,32").split(","))  # (x, y, z)
    steps = int(os.environ.get("MGPU_STEPS", "3"))
    corners = bool(int(os.environ.get("MGPU_CORNERS", "0")))
    exchange = os.environ.get("MGPU_EXCHANGE", "p2p")
    radius = int(os.environ.get("MGPU_RADIUS", "3"))
    f32 = os.environ.get("MGPU_DTYPE", "f64") == "f32"
    mdt, npdt = (b2.MHD_F32, np.float32) if f32 else (b2.MHD_F64, np.float64)
    ds = synth.spacing(N)
    res = {"rank": rank, "world": world, "N": N}
    ok = True

    mesh = b2.Mesh(N, ds, synth.P0, mdt, rank=rank, nranks=world, exchange_corners=corners,
                   exchange=exchange, radius=radius)
    res["exchange"] = exchange
    Pz = tuple(reversed(mesh.P))
    cz = tuple(reversed(mesh.coord))
    res["P_xyz"], res["coord_xyz"] = mesh.P, mesh.coord

    # 1. sentinel halo exchange, repeated with fresh values (races would show as stale halo cells)
    Nz, Ny, Nx = N[2], N[1], N[0]
    reps = int(os.environ.get("MGPU_HALO_REPS", "8"))
    mask = None
    res["halo_bitwise"] = True
    for rep in range(reps):
        glob = (np.arange(8)[:, None, None, None] * 1e7 + np.arange(Nz * Ny * Nx).reshape(Nz, Ny, Nx)[None]
                + rep * 1e9).astype(np.float64)
        if f32:  # sentinels exactly representable in FP32
            glob = (np.arange(8)[:, None, None, None] * 1e5 + np.arange(Nz * Ny * Nx).reshape(Nz, Ny, Nx)[None]
                    + rep * 1e6).astype(np.float32)
        mesh.load(np.ascontiguousarray(G.local_interior(glob, Pz, cz)))
        mesh.halo_exchange()
        grid = mesh.store_grid().numpy()
        expect = G.local_subgrid_with_halo(glob, Pz, cz, r=radius)
        if mask is None:
            mask = np.ones(grid.shape[1:], bool)
            if not corners:
                for zs in (slice(0, radius), slice(-radius, None)):
                    for ys in (slice(0, radius), slice(-radius, None)):
                        for xs in (slice(0, radius), slice(-radius, None)):
                            mask[zs, ys, xs] = False
        okh = bool(np.array_equal(grid[:, mask], expect[:, mask]))
        if not okh and res["halo_bitwise"]:
            bad = np.argwhere((grid != expect) & mask[None])
            res["halo_bad_rep"] = rep
            res["halo_bad_cells"] = int(len(bad))
            res["halo_bad_first"] = bad[:6].tolist()
            res["halo_bad_vals"] = [[float(grid[tuple(b)]), float(expect[tuple(b)])] for b in bad[:3]]
        res["halo_bitwise"] &= okh
    ok &= res["halo_bitwise"]

    # 2. RK3 steps: P GPUs vs 1 GPU (bit-identical) vs oracle
    st = synth.pcg64_state((Nz, Ny, Nx), dtype=npdt)
    mesh.load(np.ascontiguousarray(G.local_interior(st, Pz, cz)))
    for _ in range(steps):
        mesh.step(synth.DT)
    mine = mesh.store().cpu().numpy()
    parts = [None] * world if rank == 0 else None
    dist.gather_object((cz, mine), parts, dst=0)
    if rank == 0:
        full = np.empty_like(st)
        for c, part in parts:
            n = part.shape[1:]
            full[:, c[0] * n[0]:(c[0] + 1) * n[0], c[1] * n[1]:(c[1] + 1) * n[1], c[2] * n[2]:(c[2] + 1) * n[2]] = part
        single = b2.Mesh(N, ds, synth.P0, mdt, radius=radius)
        single.load(st)
        for _ in range(steps):
            single.step(synth.DT)
        one = single.store().cpu().numpy()
        single.close()
        res["bit_identical_vs_1gpu"] = bool(np.array_equal(full, one))
        ok &= res["bit_identical_vs_1gpu"]
        if os.environ.get("MGPU_ORACLE", "1") == "1":
            import oracle
            ref = oracle.integrate(st, ds, synth.P0, synth.DT, steps, r=radius)
            e = max(float(np.max(np.abs(full[q] - ref[q]) / np.maximum(np.abs(ref[q]), 1e-3 * np.max(np.abs(ref[q])))))
                    for q in range(8))
            res["oracle_field_err"] = e
            ok &= e <= (1e-4 if f32 else 1e-11)
    res["ok"] = bool(ok)
    print(json.dumps(res), flush=True)
    flag = torch.tensor([1 if ok else 0], device="cuda")
    dist.all_reduce(flag, op=dist.ReduceOp.MIN)
    mesh.close()
    dist.destroy_process_group()
    sys.exit(0 if flag.item() == 1 else 1)


if __name__ == "__main__":
    main()
