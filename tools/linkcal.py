"""Link calibration (the analog of the paper's 12 MiB block measurement):
time NCCL point-to-point send/recv between every GPU pair of one box at the halo message sizes,
then all pairs concurrently, and print GB/s per direction.  Measurement tool only (torch.distributed
send/recv over NCCL); the exchange itself lives in libb2mhd.so.

    torchrun --nproc-per-node N --master-addr 127.0.0.1 tools/linkcal.py [--reps 20]
"""
import argparse
import json
import os

import torch
import torch.distributed as dist

SIZES = {
    "corners_13.5KiB": 13824,
    "edges_576KiB": 589824,
    "side_12MiB": 12 * 2 ** 20,          # one 3 x 256^2 side, 8 fields x 8 B
    "side_pair_24MiB": 24 * 2 ** 20,     # per-peer sides at n' = 256^3
    "side_pair_100.7MB": 2 * 3 * 518 * 518 * 64,  # per-peer sides at n' = 512^3 (with edges)
}


def timed(fn, reps, warm=3):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    dist.barrier()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    t = torch.tensor([a.elapsed_time(b) / reps], device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return t.item() * 1e-3


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=20)
    a = ap.parse_args()
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", rank)))
    dist.init_process_group("nccl")
    out = {"world": world, "pairs": {}, "all_peers": {}}
    for name, nbytes in SIZES.items():
        n = nbytes // 8
        send = torch.ones(n, dtype=torch.float64, device="cuda")
        recv = [torch.empty(n, dtype=torch.float64, device="cuda") for _ in range(world)]
        # every pair (i, j), i < j, bidirectional exchange; the other ranks idle
        for i in range(world):
            for j in range(i + 1, world):
                def pair():
                    if rank in (i, j):
                        peer = j if rank == i else i
                        ops = [dist.P2POp(dist.isend, send, peer), dist.P2POp(dist.irecv, recv[peer], peer)]
                        for w in dist.batch_isend_irecv(ops):
                            w.wait()
                t = timed(pair, a.reps)
                out["pairs"].setdefault(name, {})[f"{i}-{j}"] = round(nbytes / t / 1e9, 1)

        # every rank exchanges with every other rank at once (the 7-peer case at 8 GPUs)
        def allp():
            ops = []
            for p in range(world):
                if p != rank:
                    ops += [dist.P2POp(dist.isend, send, p), dist.P2POp(dist.irecv, recv[p], p)]
            for w in dist.batch_isend_irecv(ops):
                w.wait()
        if world > 1:
            t = timed(allp, a.reps)
            out["all_peers"][name] = {"per_peer_GBs": round(nbytes / t / 1e9, 1),
                                      "per_gpu_out_GBs": round(nbytes * (world - 1) / t / 1e9, 1)}
    if rank == 0:
        print(json.dumps(out))
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
