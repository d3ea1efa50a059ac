#!/usr/bin/env python
"""Benchmark of the B200 hot path of arXiv 2103.01597: RK3 substeps of FP64 MHD.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]
    python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 bench.py --gpus N ...

A bench "step" is one full RK3 step = 3 ISL iterations, each one pass of the whole
hot path: the halo exchange (one GPU: periodic y rows copied, x faces written by
the previous update's epilogue, z planes wrapped by TMA; N > 1: fused peer-memory stores by
the boundary-slab kernels at N = 2, 4, or NCCL pack -> send/recv -> unpack) overlapped with the
inner update, and the boundary-slab update.  Metric (BASELINE.json): Gcell-updates/s per RK3
substep = global interior cells x substeps / time.

Default workload: 256^3 FP64 per GPU (BASELINE configs[1] at N = 1; configs[3] weak scaling
for N > 1: global grid = 256^3 x Morton partition, 512^3 at N = 8).  --scaling strong
--grid 512 runs configs[2].  ICs: counter-based splitmix64 uniform [0, 1),
dt = 1.19209e-7, parameters P0 (reading R#12).  Inputs (2.3 GB per GPU) are far
larger than the 126 MB L2, so no L2 flush is needed between steps.

Prints ONE JSON line on rank 0.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "Gcell-updates/s per RK3 substep (FP64 MHD)"
UNIT = "Gcell-updates/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", choices=("b200", "reference"), default="b200")
    ap.add_argument("--grid", type=int, default=256, help="per-GPU n (weak) or global n (strong)")
    ap.add_argument("--scaling", choices=("weak", "strong"), default="weak")
    ap.add_argument("--dtype", choices=("f64", "f32"), default="f64")
    ap.add_argument("--kernel", type=int, default=0, help="0 auto, 1 direct, 2 z-marching")
    ap.add_argument("--e2e-steps", type=int, default=10)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--corners", action="store_true")
    ap.add_argument("--order", type=int, choices=(2, 4, 6, 8), default=6,
                    help="stencil order 2r (P:829-830); the paper's benchmarks use 6")
    ap.add_argument("--exchange", choices=("auto", "p2p", "nccl"), default="auto",
                    help="N > 1: boundary results stored into the neighbours' halos over NVLink peer memory "
                         "(p2p) or NCCL send/recv of packed segments; auto = p2p (measured faster at N = 2, 4: "
                         "DESIGN.md 10; the 8-rank peer-memory protocol is validated by the one-GPU virtual-rank "
                         "tests), falling back to NCCL if peer memory cannot be opened on every rank")
    return ap.parse_args()


# ---- clocks during the timed region (B200_PROFILING.md clocks line) -------------------------------
class ClockSampler:
    """SM clock, power and throttle reasons sampled every 20 ms by NVML while the timed region
    runs; the memory clock is read once at the end (a per-sample memory-clock query measurably
    slowed the launch-heavy multi-GPU schedule)."""

    REASONS = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
               "sw_power_cap": 0x4, "hw_power_brake_slowdown": 0x80}

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.samples = []
        self.stop = threading.Event()
        self.t = threading.Thread(target=self.run, daemon=True)
        self.err = None
        self.mem = None

    def run(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.gpu)
            mx = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
            while not self.stop.is_set():
                sm = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
                pw = pynvml.nvmlDeviceGetPowerUsage(h) / 1000.0
                rs = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                self.samples.append((sm, mx, pw, rs))
                self.stop.wait(0.02)
            self.mem = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_MEM)
        except Exception as e:  # pragma: no cover
            self.err = str(e)

    def __enter__(self):
        self.t.start()
        return self

    def __exit__(self, *a):
        self.stop.set()
        self.t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvml unavailable: %s" % self.err]}
        reasons = sorted({n for s in self.samples for n, bit in self.REASONS.items() if s[3] & bit})
        return {"sm_mhz": statistics.median(s[0] for s in self.samples), "sm_max_mhz": max(s[1] for s in self.samples),
                "mem_mhz_end": self.mem, "power_w_max": max(s[2] for s in self.samples), "samples": len(self.samples),
                "reasons": reasons}


def numa_bind(gpu_index: int) -> None:
    """N > 1: run this rank on the host cores next to its GPU (NVML CPU affinity), so that its
    pinned host buffers are first touched on the GPU's own NUMA node; the end-to-end copies of
    several ranks then do not cross the socket interconnect.  (N = 1 keeps every core for the
    CPU baseline.)"""
    try:
        import pynvml
        pynvml.nvmlInit()
        h = pynvml.nvmlDeviceGetHandleByIndex(gpu_index)
        words = pynvml.nvmlDeviceGetCpuAffinity(h, 16)
        cpus = {w * 64 + b for w, m in enumerate(words) for b in range(64) if (m >> b) & 1}
        cpus &= os.sched_getaffinity(0)
        if cpus:
            os.sched_setaffinity(0, cpus)
    except Exception:
        pass


def peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {}


# FP64 issue peak measured on this pool's B200 with a DFMA microbenchmark
# (tools/microbench/fp64_peak.cu, profiles/r01_fp64_lds_microbench.txt): 17.09 T DFMA-lane/s.
FP64_PEAK_LANE_OPS = 17.09e12
# executed FP64 lane operations (DADD + DMUL + DFMA) per cell-substep of zmarch_kernel<double, r>
# by stencil order 2r (ncu smsp__sass_thread_inst_executed_op_d*_pred_on.sum over a k = 2 launch
# at 256^3 / 256^3 cells; profiles/r01/ncu_dp_counts.txt)
DP_PER_CELL = {2: 368.25, 4: 501.0, 6: 634.25, 8: 768.0}
NF_BYTES = {"f64": 64, "f32": 32}  # 8 fields x sizeof(T)


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def cpu_baseline(n_glob, ds, params, dt, seconds_hint=True):
    """The oracle as it stands, on the host cores: one RK3 step (3 substeps) of a periodic slab of
    the bench workload of about 8 M cells (256 x 256 x 128 at 256^3; same cells, same per-cell
    work; a bounded sample of a few seconds on the host cores); and the same on ONE core (the
    paper's CPU model solver was single-core) on a 16-plane slab."""
    import numpy as np

    import oracle
    import synth
    cores = len(os.sched_getaffinity(0))
    oracle.set_threads(cores)
    nz = max(16, min(n_glob[2], (8 << 20) // (n_glob[0] * n_glob[1])))
    st = synth.splitmix_state((n_glob[2], n_glob[1], n_glob[0]), (0, 0, 0), (nz, n_glob[1], n_glob[0]))
    oracle.integrate(st[:, :8], ds, params, dt, 0, substeps=1)  # warm the thread pool
    t0 = time.perf_counter()
    oracle.integrate(st, ds, params, dt, 1)
    el = time.perf_counter() - t0
    cells = nz * n_glob[1] * n_glob[0]
    oracle.set_threads(1)
    nz1 = min(16, n_glob[2])
    t1 = time.perf_counter()
    oracle.integrate(st[:, :nz1], ds, params, dt, 1)
    el1 = time.perf_counter() - t1
    oracle.set_threads(cores)
    cells1 = nz1 * n_glob[1] * n_glob[0]
    return {"value": cells * 3 / el / 1e9, "unit": UNIT, "cores": cores, "kind": "oracle", "cpu": cpu_model(),
            "sample": f"1 RK3 step (3 substeps) of a {n_glob[0]}x{n_glob[1]}x{nz} periodic slab of the "
                      f"workload, {el:.2f} s wall, OpenMP over z",
            "one_core": {"value": cells1 * 3 / el1 / 1e9, "unit": UNIT, "cores": 1,
                         "sample": f"1 RK3 step of a {n_glob[0]}x{n_glob[1]}x{nz1} slab, {el1:.2f} s"}}


def perf_model(n_glob, world, P_xyz, local_cells, substep_ms, prof, r, cell_bytes):
    """The paper's model (Eq. 4, tau_0 = 0 as P:406; tools/perfmodel.py) at device level for this
    run: tau_W = W pi^-1 with pi^-1 the per-cell time of this rank's update kernels (inner +
    boundary slabs, their device time per substep), tau_Q = Q beta^-1 with Q the remote halo
    cells of Eq. 7 (both directions) and beta^-1 = bytes per halo cell / NVLink per-direction
    bandwidth (full duplex).  The driver computes the measured efficiency from the per-N values;
    efficiency_model is what the model predicts for this N."""
    sys.path.insert(0, os.path.join(ROOT, "tools"))
    import perfmodel
    P = tuple(reversed(P_xyz))  # Morton coordinate order (z first, reading R#16)
    n = tuple(reversed(n_glob))
    upd = prof["update"]["ms"] + prof["outer"]["ms"]
    nsub = max(prof["update"]["launches"], 1)
    pi_inv = upd / nsub * 1e-3 / local_cells  # s per cell (device time of the update kernels)
    link = 770e9  # B200_PROFILING.md peer-copy reference, per direction
    beta_inv = cell_bytes / link / 2.0
    q = perfmodel.halo_q(n, P, r, periodic_self=True)
    tau_w = local_cells * pi_inv
    tau_q = q * beta_inv
    return {"equation": "T = max(W pi^-1, Q beta^-1) (Eq. 4, P:331; tau_0 = 0, P:406)", "P": list(P),
            "pi_inv_ns": pi_inv * 1e9, "beta_inv_ps": beta_inv * 1e12, "remote_halo_cells_Q": q,
            "tau_w_ms": tau_w * 1e3, "tau_q_ms": tau_q * 1e3, "efficiency_model": tau_w / max(tau_w, tau_q),
            "substep_ms_measured": substep_ms}


def run_reference(args, n_glob, rank):
    """--impl reference: the oracle (the paper's 'single-core CPU solver logically equivalent',
    P:899, here with OpenMP) as it stands, one bounded sample per step."""
    import numpy as np

    import oracle
    import synth
    if rank != 0:
        return
    ds = synth.spacing(n_glob)
    cores = len(os.sched_getaffinity(0))
    oracle.set_threads(cores)
    nz = max(8, min(n_glob[2], (2 << 20) // (n_glob[0] * n_glob[1])))  # ~2 M cells per sample
    st = synth.splitmix_state((n_glob[2], n_glob[1], n_glob[0]), (0, 0, 0), (nz, n_glob[1], n_glob[0]))
    oracle.integrate(st[:, :4], ds, synth.P0, synth.DT, 0, substeps=1)
    cur = st
    for _ in range(args.warmup):
        cur = oracle.integrate(cur, ds, synth.P0, synth.DT, 0, substeps=1)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        cur = oracle.integrate(cur, ds, synth.P0, synth.DT, 0, substeps=1)
    el = time.perf_counter() - t0
    cells = nz * n_glob[1] * n_glob[0]
    value = cells * args.steps / el / 1e9
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": el / args.steps * 1e3,
            "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": {"workload": f"{n_glob[0]}^3 FP64 MHD RK3 substep" if n_glob[0] == n_glob[1] == n_glob[2]
                       else f"{n_glob} FP64 MHD RK3 substep", "grid": list(n_glob)},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle", "cpu": cpu_model(),
                             "sample": f"per step: 1 substep of a {n_glob[0]}x{n_glob[1]}x{nz} periodic slab"},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    emit(line)


_JSON_OUT = None


def emit(line: dict) -> None:
    """The one JSON line, on the real stdout (everything else, e.g. the NCCL version banner some
    environments print at communicator creation, goes to stderr)."""
    out = _JSON_OUT if _JSON_OUT is not None else sys.stdout
    out.write(json.dumps(line) + "\n")
    out.flush()


def main():
    global _JSON_OUT
    # keep stdout for the JSON line alone: fd 1 is pointed at stderr for the libraries
    sys.stdout.flush()
    _JSON_OUT = os.fdopen(os.dup(1), "w")
    os.dup2(2, 1)
    sys.stdout = sys.stderr
    args = parse()
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    if world != args.gpus:
        args.gpus = world

    # decomposition for the weak-scaling global grid
    def morton_partition(nr):
        P = [1, 1, 1]
        v = nr - 1
        k = 0
        while v >> (3 * k):
            for j in range(3):
                P[2 - j] += ((v >> (3 * k + j)) & 1) << k
            k += 1
        return P  # (x, y, z)

    P = morton_partition(world)
    n_glob = tuple(args.grid * p for p in P) if args.scaling == "weak" else (args.grid,) * 3

    if args.impl == "reference":
        run_reference(args, n_glob, rank)
        return

    import numpy as np
    import torch

    import synth
    import paper_2103_01597_b200 as b2

    torch.cuda.set_device(local)
    if world > 1:
        numa_bind(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dtype = b2.MHD_F64 if args.dtype == "f64" else b2.MHD_F32
    es = 8 if dtype == b2.MHD_F64 else 4
    ds = synth.spacing(n_glob)
    exchange = args.exchange if args.exchange != "auto" else "p2p"

    def make_mesh(ex):
        return b2.Mesh(n_glob, ds, synth.P0, dtype, rank=rank, nranks=world, exchange_corners=args.corners,
                       kernel=args.kernel, exchange=ex, radius=args.order // 2)

    if world > 1 and args.exchange == "auto":
        # peer memory on every rank, else NCCL everywhere (the ranks must agree)
        mesh, err = None, None
        try:
            mesh = make_mesh("p2p")
        except Exception as e:  # pragma: no cover - hardware dependent
            err = e
        ok = torch.tensor([0 if mesh is None else 1], dtype=torch.int32, device="cuda")
        dist.all_reduce(ok, op=dist.ReduceOp.MIN)
        if not int(ok.item()):
            if mesh is not None:
                mesh.close()
            if rank == 0:
                print(f"bench: peer-memory exchange unavailable ({err}); using NCCL", file=sys.stderr)
            mesh = make_mesh("nccl")
    else:
        mesh = make_mesh(exchange)
    nz, ny, nx = mesh.shape
    lo = tuple(c * n for c, n in zip(reversed(mesh.coord), (nz, ny, nx)))
    npdt = np.float64 if dtype == b2.MHD_F64 else np.float32
    host = torch.from_numpy(synth.splitmix_state((n_glob[2], n_glob[1], n_glob[0]), lo, (nz, ny, nx),
                                                 dtype=npdt)).pin_memory()
    mesh.load(host)
    dt = synth.DT

    def barrier():
        if dist is not None:
            dist.barrier()

    def max_over_ranks(v):
        if dist is None:
            return v
        t = torch.tensor([v], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    for _ in range(args.warmup):
        mesh.step(dt)
    mesh.synchronize()

    # ---- timed region: K full RK3 steps, device-timed on the mesh stream ----
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    l0 = mesh.launch_count()
    mesh.profile(True)
    barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        ev0.record(mesh.stream)
        for _ in range(args.steps):
            mesh.step(dt)
        ev1.record(mesh.stream)
        torch.cuda.synchronize()
    barrier()
    launches = mesh.launch_count() - l0
    ms_total = max_over_ranks(ev0.elapsed_time(ev1))
    prof = mesh.profile_read()
    mesh.profile(False)
    cells = n_glob[0] * n_glob[1] * n_glob[2]
    value = cells * 3 * args.steps / (ms_total * 1e-3) / 1e9

    # per-substep time by k (k = 0 moves 128 B/cell, k = 1, 2 192 B/cell), from a few
    # extra steps after the timed region, events between the substeps on the mesh stream
    nk = max(1, min(10, args.steps))
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(nk)]
    barrier()
    torch.cuda.synchronize()
    for i in range(nk):
        evs[i][0].record(mesh.stream)
        for k in range(3):
            mesh.substep(k, dt)
            evs[i][k + 1].record(mesh.stream)
    torch.cuda.synchronize()
    per_k = [max_over_ranks(sum(evs[i][k].elapsed_time(evs[i][k + 1]) for i in range(nk)) / nk) for k in range(3)]
    per_k_gcells = [cells / (t * 1e-3) / 1e9 for t in per_k]

    # finiteness over the timed window: any NaN/Inf invalidates the run
    finite = True
    for q in range(8):
        try:
            mesh.reduce(q, b2.MHD_MAX)
        except b2.MhdError:
            finite = False

    # ---- roofline of the dominant kernel (the fused update), from its live launch times ----
    up = prof["update"]
    upd_ms = up["ms"] / max(up["launches"], 1)
    hbm_peak = peaks().get("hbm_gbs", 6650.0)
    achieved_gbs = up["bytes"] / (up["ms"] * 1e-3) / 1e9 if up["ms"] > 0 else None
    local_cells = nx * ny * nz
    # FP64 lane operations per cell-substep executed by the update kernel (DFMA + DADD + DMUL,
    # ncu source counters of zmarch_kernel<double>, profiles/r01/ncu_zmarch_*.txt)
    dp_per_cell = DP_PER_CELL[args.order] if dtype == b2.MHD_F64 else None
    ncu = {}
    try:
        ncu = json.load(open(os.path.join(ROOT, "profiles", "ncu_latest.json")))
    except Exception:
        pass
    substep_ms = ms_total / (3 * args.steps)
    traffic = ncu.get("dram_bytes_per_launch") if ncu.get("dtype") == args.dtype and world == 1 else None
    roofline = {"bound": "hbm", "achieved": achieved_gbs, "peak": hbm_peak, "unit": "GB/s",
                "frac": achieved_gbs / hbm_peak if achieved_gbs else None, "traffic": traffic,
                "traffic_note": ncu.get("note") if traffic else None,
                "kernel": "update (fused stencil + RHS + RK3)", "avg_launch_ms": upd_ms,
                "peak_source": "MEASURED_PEAKS.json hbm_gbs (measured copy)"}
    step_share = up["ms"] / max(ms_total, 1e-9)
    phases = {k: {"launches": v["launches"], "ms_per_substep": v["ms"] / (3 * args.steps)} for k, v in prof.items()}

    # ---- end to end through the public API with host buffers ----
    e2e = None
    if args.e2e_steps > 0:
        out_host = torch.empty_like(host).pin_memory()
        mesh.load(host)
        barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(args.e2e_steps):
            mesh.load_async(host)         # H2D of the step's input state (pinned), own copy stream
            mesh.step(dt)
            mesh.store_async(out_host)    # D2H of the step's result, own copy stream
        mesh.synchronize()                # every step's result is on the host
        torch.cuda.synchronize()
        el = max_over_ranks(time.perf_counter() - t0)
        e2e = {"value": cells * 3 * args.e2e_steps / el / 1e9, "unit": UNIT,
               "h2d_bytes_per_step": int(host.numel() * es), "d2h_bytes_per_step": int(out_host.numel() * es)}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(n_glob, ds, synth.P0, dt)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_total / args.steps, "higher_is_better": True,
            "scaling": args.scaling if world > 1 else "weak", "vs_baseline": None, "dtype": args.dtype,
            "data": "synthetic",
            "config": {"workload": (f"{n_glob[0]}^3" if len(set(n_glob)) == 1 else "x".join(map(str, n_glob)))
                       + f" {args.dtype.upper()} MHD, 1 RK3 step (3 substeps) per bench step",
                       "grid": list(n_glob), "local_grid": [nx, ny, nz], "partition": list(mesh.P),
                       "substeps_per_step": 3, "dt": dt, "params": "P0",
                       "l2": "inputs larger than L2 (no flush)", "kernel": args.kernel,
                       "exchange_corners": bool(args.corners),
                       "exchange": mesh.exchange, "order": args.order},
            "ms_per_substep": substep_ms,
            "per_k": {"ms": per_k, "gcells": per_k_gcells, "steps": nk},
            "gpu_launches": launches,
            "clocks": clk.summary(),
            "roofline": roofline,
            "update_share_of_step": step_share,
            "phases": phases,
            "finite": finite,
            "e2e": e2e,
            "cpu_baseline": cpu,
        }
        if world > 1:
            # several ranks: the inner launch and the boundary slabs (side stream) run concurrently,
            # so the roofline counts every cell this rank updates over the whole device-timed
            # substep (inner + outer + exchange): a lower bound on the kernels' own rate
            sub_s = substep_ms * 1e-3
            line["roofline_substep"] = {
                "bound": "alu" if dp_per_cell else "hbm",
                "achieved": (dp_per_cell * local_cells / sub_s) if dp_per_cell else
                            (NF_BYTES[args.dtype] * (2 + 3 + 3) / 3 * local_cells / sub_s / 1e9),
                "peak": FP64_PEAK_LANE_OPS if dp_per_cell else hbm_peak,
                "unit": "DP lane-ops/s" if dp_per_cell else "GB/s",
                "scope": "all update kernels of one rank (inner + boundary slabs) over the device-timed substep"}
            line["roofline_substep"]["frac"] = line["roofline_substep"]["achieved"] / line["roofline_substep"]["peak"]
            line["model"] = perf_model(n_glob, world, P, local_cells, substep_ms, prof, args.order // 2,
                                       NF_BYTES[args.dtype])
        if dtype == b2.MHD_F64 and args.order == 6 and up["ms"] > 0 and world == 1:
            # the binding on-chip resource: shared-memory wavefronts of the LSU pipe,
            # 14.91 per cell-substep (ncu l1tex__data_pipe_lsu_wavefronts_mem_shared over a k = 2
            # launch / cells, profiles/r02/ncu_zmarch_final.txt; TMA writes not included), 128 B
            # each, against the measured LDS.64 rate of 127.4 B/clk/SM (profiles/r02/
            # microbench_mio_fp64.txt) at the SM clock sampled during the timed region
            upd_cells = up["bytes"] / (NF_BYTES[args.dtype] * (2 + 3 + 3) / 3)
            sm_mhz = line["clocks"].get("sm_mhz") or 1965
            ach = 14.91 * 128 * upd_cells / (up["ms"] * 1e-3) / 1e9
            peak = 127.4 * 148 * sm_mhz * 1e6 / 1e9
            line["roofline_smem"] = {"bound": "smem", "achieved": ach, "peak": peak, "unit": "GB/s",
                                     "frac": ach / peak, "wavefronts_per_cell": 14.91,
                                     "peak_source": "LDS.64 microbenchmark 127.4 B/clk/SM x 148 SM x sampled SM clock"}
        if dtype == b2.MHD_F32 and up["ms"] > 0:
            # FP32: the same canonical arithmetic as FP64 (mhd_math.cuh), so the same executed
            # operation count per cell (ncu FP64 counters; FP32x2 pairs count two lane-ops); peak
            # nominal 148 SM x 128 FP32 lanes x 1.965 GHz (not measured)
            upd_cells = up["bytes"] / (NF_BYTES[args.dtype] * (2 + 3 + 3) / 3)
            ach = DP_PER_CELL[args.order] * upd_cells / (up["ms"] * 1e-3)
            peak32 = 148 * 128 * 1.965e9
            line["roofline_alu_fp32"] = {"bound": "alu", "achieved": ach, "peak": peak32, "unit": "FP32 lane-ops/s",
                                         "frac": ach / peak32, "ops_per_cell": DP_PER_CELL[args.order],
                                         "peak_source": "nominal 148 x 128 x 1.965 GHz",
                                         "note": "the FP32 kernel is bound by the LSU instruction rate "
                                                 "(DESIGN.md 7), not by the FP32 pipe"}
        if dp_per_cell and up["ms"] > 0:
            # FP64: the kernel is bound by on-chip work (FP64 pipe and shared-memory wavefronts,
            # DESIGN.md 7), not by HBM, so the FP64 roof is the primary one and HBM secondary.
            upd_cells = up["bytes"] / (NF_BYTES[args.dtype] * (2 + 3 + 3) / 3)  # cells x substeps updated
            ach = dp_per_cell * upd_cells / (up["ms"] * 1e-3)
            line["roofline_hbm"] = roofline
            line["roofline"] = {"bound": "alu", "achieved": ach, "peak": FP64_PEAK_LANE_OPS,
                                "unit": "DP lane-ops/s", "frac": ach / FP64_PEAK_LANE_OPS,
                                "traffic": traffic, "dp_per_cell": dp_per_cell,
                                "kernel": roofline["kernel"], "avg_launch_ms": upd_ms,
                                "peak_source": "measured DFMA microbenchmark, 17.09e12 lane-ops/s = 92 % of "
                                               "148 SM x 64 FP64 lanes x 1.965 GHz (profiles/r01_fp64_lds_microbench.txt)"}
        emit(line)
    mesh.close()
    if dist is not None:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
