"""ctypes binding of libb2mhd.so (include/b2mhd.h).  Argument marshalling only.

Every entry point of the header has a Python function of the same name.  There is
no fallback: if the library cannot be loaded, importing this module raises.
"""
from __future__ import annotations

import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("B2MHD_LIB") or os.path.join(HERE, "libb2mhd.so")

MHD_ABI_VERSION = 1
MHD_RADIUS = 3
MHD_NFIELDS = 8
MHD_F32, MHD_F64 = 4, 8
MHD_P2P_HANDLE_BYTES = 80
MHD_MIN, MHD_MAX, MHD_SUM, MHD_RMS, MHD_SUM_EXP = range(5)
STATUS = {0: "MHD_OK", 1: "MHD_EINVAL", 2: "MHD_EDECOMP", 3: "MHD_ESMALL", 4: "MHD_EUNSUPPORTED",
          5: "MHD_ECUDA", 6: "MHD_ENCCL", 7: "MHD_ENOMEM", 8: "MHD_ENONFINITE", 9: "MHD_ESTATE"}

# every symbol include/b2mhd.h declares
SYMBOLS = ("mhd_decompose", "mhd_segment_table", "mhd_workspace_bytes", "mhd_mesh_create", "mhd_nccl_unique_id",
           "mhd_comm_init", "mhd_p2p_export", "mhd_p2p_open", "mhd_set_exchange", "mhd_mesh_destroy", "mhd_load", "mhd_store", "mhd_store_async", "mhd_load_async", "mhd_store_grid", "mhd_halo_exchange",
           "mhd_integrate_substep", "mhd_integrate_step", "mhd_reduce", "mhd_debug_rhs", "mhd_synchronize",
           "mhd_set_kernel", "mhd_set_debug", "mhd_mesh_query", "mhd_launch_count", "mhd_profile_enable", "mhd_profile_read",
           "mhd_group_create", "mhd_group_halo_exchange", "mhd_group_integrate_substep", "mhd_group_integrate_step",
           "mhd_group_debug_rhs", "mhd_group_reduce", "mhd_group_synchronize", "mhd_group_destroy",
           "mhd_status_str", "mhd_last_error", "mhd_abi_version")
MHD_DEBUG_POISON_HALO = 1


class MhdError(RuntimeError):
    def __init__(self, status: int, where: str, detail: str):
        super().__init__(f"{where}: {STATUS.get(status, status)} ({detail})")
        self.status = status


class mhd_params(ctypes.Structure):
    _fields_ = [(n, ctypes.c_double) for n in
                ("nu", "zeta", "eta", "mu0", "cs0", "cp", "gamma", "K", "H", "C", "lnrho0", "lnT0")]


class mhd_mesh_info(ctypes.Structure):
    _fields_ = [("abi_version", ctypes.c_int32), ("n", ctypes.c_int64 * 3), ("radius", ctypes.c_int32),
                ("ds", ctypes.c_double * 3), ("dtype", ctypes.c_int32), ("rank", ctypes.c_int32),
                ("nranks", ctypes.c_int32), ("exchange_corners", ctypes.c_int32), ("phys", mhd_params)]


class mhd_segment(ctypes.Structure):
    _fields_ = [("offset", ctypes.c_int32 * 3), ("kind", ctypes.c_int32), ("src_first", ctypes.c_int32 * 3),
                ("dst_first", ctypes.c_int32 * 3), ("extent", ctypes.c_int32 * 3), ("send_peer", ctypes.c_int32),
                ("recv_peer", ctypes.c_int32), ("send_buf_cell", ctypes.c_int64), ("recv_buf_cell", ctypes.c_int64)]


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: run `python __graft_entry__.py build` (no CPU fallback exists)")
    lib = ctypes.CDLL(LIB_PATH, mode=ctypes.RTLD_GLOBAL)
    P = ctypes.POINTER
    sig = {
        "mhd_decompose": [P(mhd_mesh_info), ctypes.c_int32, P(ctypes.c_int32), P(ctypes.c_int32), P(ctypes.c_int64)],
        "mhd_segment_table": [P(mhd_mesh_info), ctypes.c_int32, P(mhd_segment), ctypes.c_int32, P(ctypes.c_int32)],
        "mhd_workspace_bytes": [P(mhd_mesh_info), P(ctypes.c_size_t)],
        "mhd_mesh_create": [P(mhd_mesh_info), ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p, P(ctypes.c_void_p)],
        "mhd_nccl_unique_id": [ctypes.c_void_p],
        "mhd_comm_init": [ctypes.c_void_p, ctypes.c_void_p],
        "mhd_mesh_destroy": [ctypes.c_void_p],
        "mhd_p2p_export": [ctypes.c_void_p, ctypes.c_void_p],
        "mhd_p2p_open": [ctypes.c_void_p, ctypes.c_void_p],
        "mhd_set_exchange": [ctypes.c_void_p, ctypes.c_int32],
        "mhd_load": [ctypes.c_void_p, ctypes.c_int32, ctypes.c_void_p, ctypes.c_int32, ctypes.c_int32],
        "mhd_store": [ctypes.c_void_p, ctypes.c_int32, ctypes.c_void_p, ctypes.c_int32, ctypes.c_int32],
        "mhd_store_async": [ctypes.c_void_p, ctypes.c_int32, ctypes.c_void_p, ctypes.c_int32],
        "mhd_load_async": [ctypes.c_void_p, ctypes.c_int32, ctypes.c_void_p, ctypes.c_int32],
        "mhd_store_grid": [ctypes.c_void_p, ctypes.c_int32, ctypes.c_void_p, ctypes.c_int32],
        "mhd_halo_exchange": [ctypes.c_void_p],
        "mhd_integrate_substep": [ctypes.c_void_p, ctypes.c_int32, ctypes.c_double],
        "mhd_integrate_step": [ctypes.c_void_p, ctypes.c_double],
        "mhd_reduce": [ctypes.c_void_p, ctypes.c_int32, ctypes.c_int32, P(ctypes.c_double)],
        "mhd_debug_rhs": [ctypes.c_void_p, ctypes.c_void_p],
        "mhd_synchronize": [ctypes.c_void_p],
        "mhd_set_kernel": [ctypes.c_void_p, ctypes.c_int32],
        "mhd_set_debug": [ctypes.c_void_p, ctypes.c_int32],
        "mhd_group_create": [P(ctypes.c_void_p), ctypes.c_int32, ctypes.c_int32, P(ctypes.c_void_p)],
        "mhd_group_halo_exchange": [ctypes.c_void_p],
        "mhd_group_integrate_substep": [ctypes.c_void_p, ctypes.c_int32, ctypes.c_double],
        "mhd_group_integrate_step": [ctypes.c_void_p, ctypes.c_double],
        "mhd_group_debug_rhs": [ctypes.c_void_p, P(ctypes.c_void_p)],
        "mhd_group_reduce": [ctypes.c_void_p, ctypes.c_int32, ctypes.c_int32, P(ctypes.c_double)],
        "mhd_group_synchronize": [ctypes.c_void_p],
        "mhd_group_destroy": [ctypes.c_void_p],
        "mhd_mesh_query": [ctypes.c_void_p, P(ctypes.c_int32), P(ctypes.c_int32), P(ctypes.c_int64), P(ctypes.c_int32)],
        "mhd_launch_count": [ctypes.c_void_p, P(ctypes.c_int64)],
        "mhd_profile_enable": [ctypes.c_void_p, ctypes.c_int32],
        "mhd_profile_read": [ctypes.c_void_p, ctypes.c_int32, P(ctypes.c_int64), P(ctypes.c_double), P(ctypes.c_double)],
    }
    for name, args in sig.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = ctypes.c_int
    lib.mhd_status_str.argtypes = [ctypes.c_int]
    lib.mhd_status_str.restype = ctypes.c_char_p
    lib.mhd_last_error.argtypes = []
    lib.mhd_last_error.restype = ctypes.c_char_p
    lib.mhd_abi_version.argtypes = []
    lib.mhd_abi_version.restype = ctypes.c_int32
    if lib.mhd_abi_version() != MHD_ABI_VERSION:
        raise ImportError("libb2mhd ABI version mismatch")
    return lib


lib = _load()


def check(status: int, where: str) -> None:
    if status != 0:
        raise MhdError(status, where, lib.mhd_last_error().decode())


def make_info(n_xyz, ds_xyz, params: dict, dtype: int = MHD_F64, rank: int = 0, nranks: int = 1,
              exchange_corners: bool = False, radius: int = MHD_RADIUS) -> mhd_mesh_info:
    info = mhd_mesh_info()
    info.abi_version = MHD_ABI_VERSION
    for a in range(3):
        info.n[a] = int(n_xyz[a])
        info.ds[a] = float(ds_xyz[a])
    info.radius = int(radius)  # stencil order 2r: 2, 4, 6 or 8
    info.dtype = int(dtype)
    info.rank = int(rank)
    info.nranks = int(nranks)
    info.exchange_corners = int(bool(exchange_corners))
    info.phys = mhd_params(**{k: float(v) for k, v in params.items()})
    return info


# ---- thin wrappers, same names as the C ABI ------------------------------------------------------
def mhd_decompose(info: mhd_mesh_info, rank: int):
    P = (ctypes.c_int32 * 3)()
    c = (ctypes.c_int32 * 3)()
    n = (ctypes.c_int64 * 3)()
    check(lib.mhd_decompose(ctypes.byref(info), rank, P, c, n), "mhd_decompose")
    return tuple(P), tuple(c), tuple(n)


def mhd_segment_table(info: mhd_mesh_info, rank: int):
    arr = (mhd_segment * 26)()
    cnt = ctypes.c_int32()
    check(lib.mhd_segment_table(ctypes.byref(info), rank, arr, 26, ctypes.byref(cnt)), "mhd_segment_table")
    out = []
    for i in range(cnt.value):
        s = arr[i]
        out.append(dict(offset=tuple(s.offset), kind=s.kind, src_first=tuple(s.src_first),
                        dst_first=tuple(s.dst_first), extent=tuple(s.extent), send_peer=s.send_peer,
                        recv_peer=s.recv_peer, send_buf_cell=s.send_buf_cell, recv_buf_cell=s.recv_buf_cell))
    return out


def mhd_workspace_bytes(info: mhd_mesh_info) -> int:
    b = ctypes.c_size_t()
    check(lib.mhd_workspace_bytes(ctypes.byref(info), ctypes.byref(b)), "mhd_workspace_bytes")
    return b.value


def mhd_mesh_create(info: mhd_mesh_info, workspace_ptr: int, nbytes: int, stream_ptr: int) -> int:
    m = ctypes.c_void_p()
    check(lib.mhd_mesh_create(ctypes.byref(info), ctypes.c_void_p(workspace_ptr), nbytes,
                              ctypes.c_void_p(stream_ptr), ctypes.byref(m)), "mhd_mesh_create")
    return m.value


def mhd_nccl_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    check(lib.mhd_nccl_unique_id(buf), "mhd_nccl_unique_id")
    return buf.raw


def mhd_comm_init(mesh: int, uid: bytes) -> None:
    buf = ctypes.create_string_buffer(bytes(uid), 128)
    check(lib.mhd_comm_init(ctypes.c_void_p(mesh), buf), "mhd_comm_init")


def mhd_p2p_export(mesh: int) -> bytes:
    buf = ctypes.create_string_buffer(MHD_P2P_HANDLE_BYTES)
    check(lib.mhd_p2p_export(ctypes.c_void_p(mesh), buf), "mhd_p2p_export")
    return buf.raw


def mhd_p2p_open(mesh: int, blobs) -> None:
    raw = b"".join(bytes(b) for b in blobs)
    buf = ctypes.create_string_buffer(raw, len(raw))
    check(lib.mhd_p2p_open(ctypes.c_void_p(mesh), buf), "mhd_p2p_open")


def mhd_set_exchange(mesh: int, mode: int) -> None:
    check(lib.mhd_set_exchange(ctypes.c_void_p(mesh), mode), "mhd_set_exchange")


def mhd_mesh_destroy(mesh: int) -> None:
    check(lib.mhd_mesh_destroy(ctypes.c_void_p(mesh)), "mhd_mesh_destroy")


def mhd_load(mesh: int, field: int, ptr: int, dtype: int, on_device: bool) -> None:
    check(lib.mhd_load(ctypes.c_void_p(mesh), field, ctypes.c_void_p(ptr), dtype, int(on_device)), "mhd_load")


def mhd_store(mesh: int, field: int, ptr: int, dtype: int, on_device: bool) -> None:
    check(lib.mhd_store(ctypes.c_void_p(mesh), field, ctypes.c_void_p(ptr), dtype, int(on_device)), "mhd_store")


def mhd_load_async(mesh: int, field: int, ptr: int, dtype: int) -> None:
    check(lib.mhd_load_async(ctypes.c_void_p(mesh), field, ctypes.c_void_p(ptr), dtype), "mhd_load_async")


def mhd_store_async(mesh: int, field: int, ptr: int, dtype: int) -> None:
    check(lib.mhd_store_async(ctypes.c_void_p(mesh), field, ctypes.c_void_p(ptr), dtype), "mhd_store_async")


def mhd_store_grid(mesh: int, field: int, ptr: int, on_device: bool) -> None:
    check(lib.mhd_store_grid(ctypes.c_void_p(mesh), field, ctypes.c_void_p(ptr), int(on_device)), "mhd_store_grid")


def mhd_halo_exchange(mesh: int) -> None:
    check(lib.mhd_halo_exchange(ctypes.c_void_p(mesh)), "mhd_halo_exchange")


def mhd_integrate_substep(mesh: int, k: int, dt: float) -> None:
    check(lib.mhd_integrate_substep(ctypes.c_void_p(mesh), k, dt), "mhd_integrate_substep")


def mhd_integrate_step(mesh: int, dt: float) -> None:
    check(lib.mhd_integrate_step(ctypes.c_void_p(mesh), dt), "mhd_integrate_step")


def mhd_reduce(mesh: int, field: int, op: int, allow_nonfinite: bool = False) -> float:
    out = ctypes.c_double()
    st = lib.mhd_reduce(ctypes.c_void_p(mesh), field, op, ctypes.byref(out))
    if not (allow_nonfinite and st == 8):
        check(st, "mhd_reduce")
    return out.value


def mhd_debug_rhs(mesh: int, dev_ptr: int) -> None:
    check(lib.mhd_debug_rhs(ctypes.c_void_p(mesh), ctypes.c_void_p(dev_ptr)), "mhd_debug_rhs")


def mhd_synchronize(mesh: int) -> None:
    check(lib.mhd_synchronize(ctypes.c_void_p(mesh)), "mhd_synchronize")


def mhd_set_kernel(mesh: int, variant: int) -> None:
    check(lib.mhd_set_kernel(ctypes.c_void_p(mesh), variant), "mhd_set_kernel")


def mhd_set_debug(mesh: int, flags: int) -> None:
    check(lib.mhd_set_debug(ctypes.c_void_p(mesh), flags), "mhd_set_debug")


# ---- several ranks in one process ----
def mhd_group_create(meshes, exchange: int) -> int:
    arr = (ctypes.c_void_p * len(meshes))(*meshes)
    g = ctypes.c_void_p()
    check(lib.mhd_group_create(arr, len(meshes), exchange, ctypes.byref(g)), "mhd_group_create")
    return g.value


def mhd_group_halo_exchange(group: int) -> None:
    check(lib.mhd_group_halo_exchange(ctypes.c_void_p(group)), "mhd_group_halo_exchange")


def mhd_group_integrate_substep(group: int, k: int, dt: float) -> None:
    check(lib.mhd_group_integrate_substep(ctypes.c_void_p(group), k, dt), "mhd_group_integrate_substep")


def mhd_group_integrate_step(group: int, dt: float) -> None:
    check(lib.mhd_group_integrate_step(ctypes.c_void_p(group), dt), "mhd_group_integrate_step")


def mhd_group_debug_rhs(group: int, dev_ptrs) -> None:
    arr = (ctypes.c_void_p * len(dev_ptrs))(*dev_ptrs)
    check(lib.mhd_group_debug_rhs(ctypes.c_void_p(group), arr), "mhd_group_debug_rhs")


def mhd_group_reduce(group: int, field: int, op: int, allow_nonfinite: bool = False) -> float:
    out = ctypes.c_double()
    st = lib.mhd_group_reduce(ctypes.c_void_p(group), field, op, ctypes.byref(out))
    if not (allow_nonfinite and st == 8):
        check(st, "mhd_group_reduce")
    return out.value


def mhd_group_synchronize(group: int) -> None:
    check(lib.mhd_group_synchronize(ctypes.c_void_p(group)), "mhd_group_synchronize")


def mhd_group_destroy(group: int) -> None:
    check(lib.mhd_group_destroy(ctypes.c_void_p(group)), "mhd_group_destroy")


def mhd_mesh_query(mesh: int):
    P = (ctypes.c_int32 * 3)()
    c = (ctypes.c_int32 * 3)()
    n = (ctypes.c_int64 * 3)()
    k = ctypes.c_int32()
    check(lib.mhd_mesh_query(ctypes.c_void_p(mesh), P, c, n, ctypes.byref(k)), "mhd_mesh_query")
    return tuple(P), tuple(c), tuple(n), k.value


def mhd_launch_count(mesh: int) -> int:
    c = ctypes.c_int64()
    check(lib.mhd_launch_count(ctypes.c_void_p(mesh), ctypes.byref(c)), "mhd_launch_count")
    return c.value


PHASES = ("update", "self", "pack", "exchange", "unpack", "outer")


def mhd_profile_enable(mesh: int, enable: bool) -> None:
    check(lib.mhd_profile_enable(ctypes.c_void_p(mesh), int(enable)), "mhd_profile_enable")


def mhd_profile_read(mesh: int, phase: int):
    n = ctypes.c_int64()
    ms = ctypes.c_double()
    by = ctypes.c_double()
    check(lib.mhd_profile_read(ctypes.c_void_p(mesh), phase, ctypes.byref(n), ctypes.byref(ms), ctypes.byref(by)),
          "mhd_profile_read")
    return n.value, ms.value, by.value


def mhd_status_str(s: int) -> str:
    return lib.mhd_status_str(s).decode()


def mhd_last_error() -> str:
    return lib.mhd_last_error().decode()


def mhd_abi_version() -> int:
    return lib.mhd_abi_version()
