"""Full-size multi-GPU check in the launch configuration bench.py times (run under torchrun, one
process per GPU): the BASELINE 512^3 strong-scaling grid split over the ranks, the
counter-based random state of bench.py, one RK3 step with the chosen exchange; every rank's
result must equal, bit for bit, the same region of a 1-GPU run of the whole grid done by rank 0
(decomposition invariance, a property that holds at any size; the 1-GPU path itself is checked
against the oracle at full size by tests/test_gpu_parity.py::test_full_size_256_rhs_and_substep).

    MGPU_N=512,512,512 MGPU_EXCHANGE=p2p torchrun --nproc-per-node 4 tools/mgpu_full.py
Prints one JSON line (rank 0); exit code 0 iff identical.
"""
from __future__ import annotations

import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def checksum(t):
    """Bit-sensitive digest of a float64 tensor block: wrapping int64 sums of the bit patterns and
    of a position-mixed hash of them (any flipped bit changes it, barring a 2^-64 collision)."""
    import torch
    b = t.contiguous().view(torch.int64).flatten()
    idx = torch.arange(b.numel(), device=b.device, dtype=torch.int64)
    mixed = (b ^ (b >> 29)) * -7046029254386353131 + idx * 0x632BE59BD9B4E019  # odd constants
    return (int(b.sum().item()), int((mixed ^ (mixed >> 31)).sum().item()))


def main():
    import torch
    import torch.distributed as dist

    import synth
    import paper_2103_01597_b200 as b2

    rank = int(os.environ["RANK"])
    world = int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    N = tuple(int(v) for v in os.environ.get("MGPU_N", "512,512,512").split(","))  # (x, y, z)
    exchange = os.environ.get("MGPU_EXCHANGE", "p2p")
    steps = int(os.environ.get("MGPU_STEPS", "1"))
    ds = synth.spacing(N)
    Nzyx = (N[2], N[1], N[0])

    mesh = b2.Mesh(N, ds, synth.P0, b2.MHD_F64, rank=rank, nranks=world, exchange=exchange)
    nz, ny, nx = mesh.shape
    lo = tuple(c * n for c, n in zip(reversed(mesh.coord), (nz, ny, nx)))
    mesh.load(torch.from_numpy(synth.splitmix_state(Nzyx, lo, (nz, ny, nx))))
    for _ in range(steps):
        mesh.step(synth.DT)
    mine = mesh.store()  # device (8, nz', ny', nx')
    torch.cuda.synchronize()
    mesh.close()

    ok = True
    res = {"N": N, "world": world, "exchange": exchange, "steps": steps, "local": [nx, ny, nz]}
    los = [None] * world
    dist.all_gather_object(los, lo)
    if os.environ.get("MGPU_CHECKSUM") == "1":
        # grids whose whole 1-GPU state cannot also be held as a copy (1024^3: 137 GB of mesh
        # workspace on one B200): compare bit-sensitive checksums of every rank's block per field
        sums = [checksum(mine[q]) for q in range(8)]
        del mine, mesh  # free this rank's workspace before rank 0 builds the 1-GPU mesh
        torch.cuda.empty_cache()
        allsums = [None] * world
        dist.all_gather_object(allsums, sums)
        if rank == 0:
            single = b2.Mesh(N, ds, synth.P0, b2.MHD_F64)
            for q in range(8):  # one field at a time on the host (8.6 GB each at 1024^3)
                f = synth.splitmix_state(Nzyx, (0, 0, 0), Nzyx, fields=(q,))[0]
                b2._native.mhd_load(single.handle, q, f.ctypes.data, b2.MHD_F64, False)
                del f
            single.synchronize()
            for _ in range(steps):
                single.step(synth.DT)
            res["ranks_identical"] = [True] * world
            buf = torch.empty(Nzyx, dtype=torch.float64, device="cuda")
            finite = True
            for q in range(8):
                b2._native.mhd_store(single.handle, q, buf.data_ptr(), b2.MHD_F64, True)
                torch.cuda.synchronize()
                finite &= bool(torch.isfinite(buf).all().item())
                for r in range(world):
                    z0, y0, x0 = los[r]
                    same = checksum(buf[z0:z0 + nz, y0:y0 + ny, x0:x0 + nx]) == allsums[r][q]
                    res["ranks_identical"][r] &= same
                    ok &= same
            single.close()
            res["finite"] = finite
            res["mode"] = "checksums (sum of the int64 bit patterns and of a mixed hash, per rank and field)"
            ok &= finite
        res["ok"] = bool(ok)
        if rank == 0:
            print(json.dumps(res), flush=True)
        flag = torch.tensor([1 if ok else 0], device="cuda")
        dist.broadcast(flag, src=0)
        dist.destroy_process_group()
        sys.exit(0 if flag.item() == 1 else 1)
    if rank == 0:
        single = b2.Mesh(N, ds, synth.P0, b2.MHD_F64)
        single.load(torch.from_numpy(synth.splitmix_state(Nzyx, (0, 0, 0), Nzyx)))
        for _ in range(steps):
            single.step(synth.DT)
        one = single.store()
        torch.cuda.synchronize()
        single.close()
        res["ranks_identical"] = []
        for r in range(world):
            if r == 0:
                part = mine
            else:
                part = torch.empty_like(mine)
                dist.recv(part, src=r)
            z0, y0, x0 = los[r]
            ref = one[:, z0:z0 + nz, y0:y0 + ny, x0:x0 + nx]
            same = bool(torch.equal(part, ref))
            res["ranks_identical"].append(same)
            ok &= same
        res["finite"] = bool(torch.isfinite(one).all().item())
        ok &= res["finite"]
    else:
        dist.send(mine, dst=0)
    res["ok"] = bool(ok)
    if rank == 0:
        print(json.dumps(res), flush=True)
    flag = torch.tensor([1 if ok else 0], device="cuda")
    dist.broadcast(flag, src=0)
    dist.destroy_process_group()
    sys.exit(0 if flag.item() == 1 else 1)


if __name__ == "__main__":
    main()
