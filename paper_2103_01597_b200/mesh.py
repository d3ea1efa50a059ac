"""`Mesh`: one rank's subdomain, its device workspace and stream; `Group`: every rank of a
decomposition driven by one process (argument marshalling only).

All arithmetic runs in libb2mhd.so; these classes allocate the caller-owned workspaces
(torch uint8 tensors), pick the streams, broadcast the NCCL unique id over the torch
process group, and move tensors in and out through the C ABI.
"""
from __future__ import annotations

import numpy as np

from . import _native as native

_TORCH_DT = {native.MHD_F64: "float64", native.MHD_F32: "float32"}


class Mesh:
    def __init__(self, n_xyz, ds_xyz, params: dict, dtype: int = native.MHD_F64, rank: int = 0, nranks: int = 1,
                 exchange_corners: bool = False, stream=None, process_group=None, kernel: int = 0,
                 exchange: str = "nccl", radius: int = 3, group_member: bool = False, debug: int = 0):
        """exchange (nranks > 1): "p2p" = boundary results stored straight into the neighbours' halos
        over NVLink (CUDA IPC peer memory); "nccl" = pack, NCCL send/recv, unpack.
        radius: stencil radius r, order 2r = 2, 4, 6 (default, the paper's benchmarks) or 8.
        group_member: created for a `Group` (no NCCL communicator, no IPC; the group wires it).
        debug: mhd_set_debug flags (MHD_DEBUG_POISON_HALO)."""
        import torch

        if not torch.cuda.is_available():
            raise RuntimeError("b2mhd needs a CUDA device (no CPU fallback)")
        self.torch = torch
        self.dtype = int(dtype)
        self.tdtype = getattr(torch, _TORCH_DT[self.dtype])
        self.radius = int(radius)
        self.info = native.make_info(n_xyz, ds_xyz, params, dtype, rank, nranks, exchange_corners, radius)
        self.nbytes = native.mhd_workspace_bytes(self.info)
        self.device = torch.device("cuda", torch.cuda.current_device())
        self.stream = stream if stream is not None else torch.cuda.Stream(self.device)
        self.workspace = torch.empty(self.nbytes, dtype=torch.uint8, device=self.device)
        self.handle = native.mhd_mesh_create(self.info, self.workspace.data_ptr(), self.nbytes,
                                             self.stream.cuda_stream)
        self.P, self.coord, self.local_n, _ = native.mhd_mesh_query(self.handle)
        self.shape = (self.local_n[2], self.local_n[1], self.local_n[0])  # (nz', ny', nx')
        self.process_group = process_group
        self._barrier_on_close = False
        if debug:
            native.mhd_set_debug(self.handle, debug)
        if nranks > 1 and not group_member:
            import torch.distributed as dist
            obj = [native.mhd_nccl_unique_id() if rank == 0 else None]
            dist.broadcast_object_list(obj, src=0, group=process_group)
            native.mhd_comm_init(self.handle, obj[0])  # reductions (and the "nccl" exchange)
            if exchange == "p2p":
                blobs = [None] * nranks
                dist.all_gather_object(blobs, native.mhd_p2p_export(self.handle), group=process_group)
                err = None
                try:
                    native.mhd_p2p_open(self.handle, blobs)
                except native.MhdError as e:
                    err = e
                # every rank learns whether every rank opened its neighbours' memory, so that a
                # failure raises everywhere (no rank is left waiting in a collective)
                flag = torch.tensor([0 if err else 1], dtype=torch.int32, device=self.device)
                dist.all_reduce(flag, op=dist.ReduceOp.MIN, group=process_group)
                if not int(flag.item()):
                    native.mhd_mesh_destroy(self.handle)
                    self.handle = None
                    raise RuntimeError(f"peer-memory exchange unavailable on some rank ({err or 'remote'})")
                dist.barrier(group=process_group)
                self._barrier_on_close = True
            elif exchange != "nccl":
                raise ValueError(f"exchange must be 'p2p' or 'nccl', not {exchange!r}")
        self.exchange = exchange if nranks > 1 and not group_member else ("group" if group_member else "local")
        if kernel:
            native.mhd_set_kernel(self.handle, kernel)

    # ---- state I/O ----------------------------------------------------------------------------
    def _dt_of(self, t) -> int:
        return native.MHD_F64 if t.dtype in (self.torch.float64, np.float64) else native.MHD_F32

    def load(self, state) -> None:
        """state: (8, nz', ny', nx') torch tensor (device or host) or numpy array, C-contiguous."""
        torch = self.torch
        if isinstance(state, np.ndarray):
            state = torch.from_numpy(np.ascontiguousarray(state))
        assert tuple(state.shape) == (8,) + tuple(self.shape), (state.shape, self.shape)
        state = state.contiguous()
        on_dev = state.is_cuda
        if on_dev:
            self.stream.wait_stream(torch.cuda.current_stream(self.device))
        dt = self._dt_of(state)
        for q in range(8):
            native.mhd_load(self.handle, q, state[q].data_ptr(), dt, on_dev)
        if not on_dev:
            self.synchronize()  # the host buffer may be reused by the caller
        self._keep = state

    def store(self, out=None, dtype=None):
        """Returns (8, nz', ny', nx'); `out` may be a device or (pinned) host tensor."""
        torch = self.torch
        if out is None:
            out = torch.empty((8,) + tuple(self.shape), dtype=dtype or self.tdtype, device=self.device)
        on_dev = out.is_cuda
        dt = self._dt_of(out)
        for q in range(8):
            native.mhd_store(self.handle, q, out[q].data_ptr(), dt, on_dev)
        if on_dev:
            torch.cuda.current_stream(self.device).wait_stream(self.stream)
        return out

    def load_async(self, state):
        """Enqueue the load of a host tensor (8, nz', ny', nx') (pinned for overlap); the caller
        keeps it alive and unmodified until synchronize()."""
        assert not state.is_cuda and state.is_contiguous()
        assert tuple(state.shape) == (8,) + tuple(self.shape), (state.shape, self.shape)
        dt = self._dt_of(state)
        for q in range(8):
            native.mhd_load_async(self.handle, q, state[q].data_ptr(), dt)
        self._keep = state

    def store_async(self, out):
        """Enqueue the store of the current state into the host tensor `out` (8, nz', ny', nx'),
        pinned for overlap; `out` is complete after synchronize()."""
        assert not out.is_cuda
        dt = self._dt_of(out)
        for q in range(8):
            native.mhd_store_async(self.handle, q, out[q].data_ptr(), dt)
        return out

    def store_grid(self):
        """Halo-inclusive local grids, (8, nz'+2r, ny'+2r, nx'+2r), on the host (test hook)."""
        sh = tuple(v + 2 * self.radius for v in self.shape)
        out = self.torch.empty((8,) + sh, dtype=self.tdtype).pin_memory()
        for q in range(8):
            native.mhd_store_grid(self.handle, q, out[q].data_ptr(), False)
        return out

    # ---- hot path -------------------------------------------------------------------------------
    def halo_exchange(self) -> None:
        native.mhd_halo_exchange(self.handle)

    def substep(self, k: int, dt: float) -> None:
        native.mhd_integrate_substep(self.handle, k, dt)

    def step(self, dt: float) -> None:
        native.mhd_integrate_step(self.handle, dt)

    def reduce(self, field: int, op: int, allow_nonfinite: bool = False) -> float:
        return native.mhd_reduce(self.handle, field, op, allow_nonfinite)

    def debug_rhs(self):
        out = self.torch.empty((8,) + tuple(self.shape), dtype=self.tdtype, device=self.device)
        native.mhd_debug_rhs(self.handle, out.data_ptr())
        self.torch.cuda.current_stream(self.device).wait_stream(self.stream)
        return out

    def set_exchange(self, mode: str) -> None:
        native.mhd_set_exchange(self.handle, {"nccl": 0, "p2p": 1}[mode])
        self.exchange = mode

    def set_kernel(self, variant: int) -> None:
        native.mhd_set_kernel(self.handle, variant)

    def set_debug(self, flags: int) -> None:
        native.mhd_set_debug(self.handle, flags)

    def synchronize(self) -> None:
        native.mhd_synchronize(self.handle)

    def profile(self, enable: bool) -> None:
        native.mhd_profile_enable(self.handle, enable)

    def profile_read(self) -> dict:
        out = {}
        for i, name in enumerate(native.PHASES):
            n, ms, by = native.mhd_profile_read(self.handle, i)
            out[name] = dict(launches=n, ms=ms, bytes=by)
        return out

    def launch_count(self) -> int:
        return native.mhd_launch_count(self.handle)

    def close(self) -> None:
        if getattr(self, "handle", None):
            native.mhd_mesh_destroy(self.handle)  # waits for the neighbours' last stores (p2p)
            self.handle = None
            if self._barrier_on_close:
                # no rank releases its IPC-exported workspace while a neighbour may still write it
                import torch.distributed as dist
                if dist.is_available() and dist.is_initialized():
                    dist.barrier(group=self.process_group)

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Group:
    """Every rank of an `nranks` decomposition, driven by this one process (mhd_group_*).

    The ranks run the same schedules and kernels as with one process per rank;
    the ranks are placed round-robin on `devices` (default: the current device), so 8 ranks
    can run on 1, 2 or 4 GPUs.  exchange: "packed" (pack -> copy-engine pull of the
    neighbours' send buffers -> unpack: the NCCL schedule with the transfer done by
    cudaMemcpyAsync) or "p2p" (peer-memory stores of the new boundary cells).  Cross-rank
    ordering uses CUDA events; no kernel waits on another.
    """

    def __init__(self, n_xyz, ds_xyz, params: dict, dtype: int = native.MHD_F64, nranks: int = 2,
                 exchange: str = "p2p", exchange_corners: bool = False, radius: int = 3, devices=None,
                 debug: int = 0):
        import torch

        if exchange not in ("packed", "p2p"):
            raise ValueError(f"group exchange must be 'packed' or 'p2p', not {exchange!r}")
        self.torch = torch
        devices = list(devices) if devices else [torch.cuda.current_device()]
        prev = torch.cuda.current_device()
        self.meshes = []
        try:
            for r in range(nranks):
                torch.cuda.set_device(devices[r % len(devices)])
                self.meshes.append(Mesh(n_xyz, ds_xyz, params, dtype, rank=r, nranks=nranks,
                                        exchange_corners=exchange_corners, radius=radius, group_member=True,
                                        debug=debug))
        finally:
            torch.cuda.set_device(prev)
        self.handle = native.mhd_group_create([m.handle for m in self.meshes], {"packed": 0, "p2p": 1}[exchange])
        self.exchange = exchange
        self.n = tuple(int(v) for v in n_xyz)
        self.radius = radius
        self.tdtype = self.meshes[0].tdtype

    def _block(self, m):
        nz, ny, nx = m.shape
        cx, cy, cz = m.coord
        return (slice(cz * nz, (cz + 1) * nz), slice(cy * ny, (cy + 1) * ny), slice(cx * nx, (cx + 1) * nx))

    def load(self, state) -> None:
        """state: the GLOBAL (8, Nz, Ny, Nx) array (numpy or host torch); each rank gets its block."""
        import numpy as np
        for m in self.meshes:
            bz, by, bx = self._block(m)
            m.load(np.ascontiguousarray(np.asarray(state)[:, bz, by, bx]))

    def store(self):
        """The global (8, Nz, Ny, Nx) state gathered from every rank, as a numpy array."""
        import numpy as np
        parts = [(m, m.store().cpu().numpy()) for m in self.meshes]
        out = np.empty((8, self.n[2], self.n[1], self.n[0]), dtype=parts[0][1].dtype)
        for m, part in parts:
            bz, by, bx = self._block(m)
            out[:, bz, by, bx] = part
        return out

    def store_grids(self):
        """Per rank, the halo-inclusive local grid (8, nz'+2r, ny'+2r, nx'+2r) on the host."""
        return [m.store_grid() for m in self.meshes]

    def halo_exchange(self) -> None:
        native.mhd_group_halo_exchange(self.handle)

    def substep(self, k: int, dt: float) -> None:
        native.mhd_group_integrate_substep(self.handle, k, dt)

    def step(self, dt: float) -> None:
        native.mhd_group_integrate_step(self.handle, dt)

    def debug_rhs(self):
        """The global RHS (8, Nz, Ny, Nx) of the current state, as a numpy array."""
        import numpy as np
        outs = [self.torch.empty((8,) + tuple(m.shape), dtype=m.tdtype, device=m.device) for m in self.meshes]
        native.mhd_group_debug_rhs(self.handle, [o.data_ptr() for o in outs])
        self.synchronize()
        full = np.empty((8, self.n[2], self.n[1], self.n[0]), dtype=outs[0].cpu().numpy().dtype)
        for m, o in zip(self.meshes, outs):
            bz, by, bx = self._block(m)
            full[:, bz, by, bx] = o.cpu().numpy()
        return full

    def reduce(self, field: int, op: int, allow_nonfinite: bool = False) -> float:
        return native.mhd_group_reduce(self.handle, field, op, allow_nonfinite)

    def synchronize(self) -> None:
        native.mhd_group_synchronize(self.handle)

    def launch_count(self) -> int:
        return sum(m.launch_count() for m in self.meshes)

    def close(self) -> None:
        if getattr(self, "handle", None):
            native.mhd_group_destroy(self.handle)
            self.handle = None
        for m in getattr(self, "meshes", []):
            m.close()
        self.meshes = []

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
