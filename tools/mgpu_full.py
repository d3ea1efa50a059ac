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
