/*
 * b2mhd — C ABI of the B200-native hot path of arXiv 2103.01597
 * (Pekkilä et al., "Scalable communication for high-order stencil
 * computations using CUDA-aware MPI"): one third-order Runge–Kutta substep of
 * compressible MHD on a periodic 3-D grid (fused 6th-order stencil + RHS +
 * RK3 update) and the radius-3 halo exchange over a Morton-ordered 3-D
 * decomposition, one process per GPU.
 *
 * Citations: PAPER.md line numbers P:n with the section / equation.  Readings
 * of passages where the paper is silent are DESIGN.md "Readings" R#n.
 *
 * Conventions (all entry points)
 *   - Axis order in every array argument of this header is (x, y, z); x is the
 *     fastest memory axis (R#16).  The Morton coordinate 0 of P:557 maps to z.
 *   - "Local interior" buffers are nz' * ny' * nx' values, x fastest, no halo,
 *     in the dtype named by the call.  Field order is mhd_field (Table B.1).
 *   - Every call returns mhd_status; no call aborts or throws across the ABI.
 *     On failure, mhd_last_error() returns a thread-local message.
 *   - Pointers named dev_* are CUDA device pointers; on_device = 0 means a
 *     host pointer (pinned memory gives the fastest copies).
 *   - All device work of a mesh is issued on the CUDA stream passed to
 *     mhd_mesh_create (internal comm streams join it with events).  Calls are
 *     asynchronous with respect to the host unless documented as blocking.
 *   - One mesh per host thread.  Ranks run one process per GPU (torchrun; the NCCL or
 *     peer-memory exchange), or several ranks in one process (mhd_group_*, for fewer GPUs
 *     than ranks or a single-process driver).
 *   - Where a call has no passage of its own, the reading it implements is SURVEY §8(b)
 *     ("the field state loaded and stored per rank", "an ISL iteration = halo exchange +
 *     update", "verification by comparing stored state") over the problem statement P:194-212.
 */
#ifndef B2MHD_H
#define B2MHD_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MHD_ABI_VERSION 1
#define MHD_RADIUS 3      /* default stencil radius r (Eq. 1); 6th order: k = 2r.
                             mhd_mesh_info.radius may be 1..4 (orders 2, 4, 6, 8) */
#define MHD_NSEGMENTS 26  /* 6 sides + 12 edges + 8 corners */

typedef enum {
  MHD_OK = 0,
  MHD_EINVAL = 1,       /* bad argument (null pointer, field index, k out of range, ...) */
  MHD_EDECOMP = 2,      /* p_i does not divide n_i, or nranks is not a power of two */
  MHD_ESMALL = 3,       /* local extent n'_i <= 2r: no inner segment */
  MHD_EUNSUPPORTED = 4, /* radius outside 1..4, unknown dtype, ABI version mismatch, > 7 neighbours */
  MHD_ECUDA = 5,        /* a CUDA runtime call failed */
  MHD_ENCCL = 6,        /* an NCCL call failed, or comm used before mhd_comm_init */
  MHD_ENOMEM = 7,       /* workspace smaller than mhd_workspace_bytes */
  MHD_ENONFINITE = 8,   /* a reduction found a NaN or Inf */
  MHD_ESTATE = 9        /* substeps called out of order (k must go 0, 1, 2, 0, ...) */
} mhd_status;

/* The eight scalar fields of Table B.1; order is reading R#14. */
typedef enum {
  MHD_LNRHO = 0, MHD_UX = 1, MHD_UY = 2, MHD_UZ = 3,
  MHD_SS = 4, MHD_AX = 5, MHD_AY = 6, MHD_AZ = 7,
  MHD_NFIELDS = 8
} mhd_field;

/* Arithmetic type of the mesh state ("single and double precision"). */
typedef enum { MHD_F32 = 4, MHD_F64 = 8 } mhd_dtype;

typedef enum {
  MHD_MIN = 0, MHD_MAX = 1, MHD_SUM = 2,
  MHD_RMS = 3,     /* sqrt(sum f^2 / C_N) over the global interior */
  MHD_SUM_EXP = 4  /* sum e^f over the global interior (mass for f = lnrho) */
} mhd_reduce_op;

/* Physical parameters of Eqs. B.1-B.4 (Table B.2; values are not
 * given by the paper, reading R#12).  lnrho0/lnT0 are the reference state of
 * the ideal-gas relation lnT = lnT0 + gamma s/cp + (gamma-1)(lnrho - lnrho0)
 * (reading R#5); cs0 is the sound speed at that state. */
typedef struct {
  double nu, zeta, eta, mu0, cs0, cp, gamma, K, H, C, lnrho0, lnT0;
} mhd_params;

typedef struct {
  int32_t abi_version;      /* must be MHD_ABI_VERSION */
  int64_t n[3];             /* global computational domain N (x, y, z) */
  int32_t radius;           /* stencil radius r = 1..4 (order 2r); MHD_RADIUS = 3 is the paper's */
  double ds[3];             /* grid spacing (x, y, z) */
  int32_t dtype;            /* mhd_dtype */
  int32_t rank, nranks;     /* this process and C_P; C_P a power of two */
  int32_t exchange_corners; /* 0: skip the 8 corner segments (never read by Eq. 14) */
  mhd_params phys;
} mhd_mesh_info;

typedef struct mhd_mesh mhd_mesh; /* opaque */

/* One halo segment of a rank, as exchanged (host-side query).
 * offset o in {-1,0,1}^3 \ {0}.  The rank RECEIVES dst region (halo cells at
 * offset o) from recv_peer = rank of coord + o, and SENDS src region (its own
 * interior cells that neighbour coord - o needs) to send_peer.  Coordinates are
 * interior-relative: 0 .. n'-1 is the interior, -r .. -1 and n' .. n'+r-1 the halo.
 * Segments to one peer are concatenated in canonical order (sides, edges,
 * corners; lexicographic offset within a class) at buffer offsets in cells. */
typedef struct {
  int32_t offset[3];
  int32_t kind;              /* 1 side, 2 edge, 3 corner: number of nonzero offsets */
  int32_t src_first[3], dst_first[3], extent[3];
  int32_t send_peer, recv_peer;
  int64_t send_buf_cell, recv_buf_cell; /* cell offset inside that peer's buffer (-1: self copy) */
} mhd_segment;

/* ---- pure host functions (no device, no mesh) ---------------------------- */

/* P = morton^-1(C_P - 1) + (1,1,1); rank -> coord = morton^-1(rank);
 * n'_i = n_i / p_i.  P, coord, local_n in (x, y, z) order. */
mhd_status mhd_decompose(const mhd_mesh_info* info, int32_t rank, int32_t P[3],
                         int32_t coord[3], int64_t local_n[3]);

/* Writes up to max_segments segments of `rank` into out (26, or 18 without
 * corners) and their number into *count. */
mhd_status mhd_segment_table(const mhd_mesh_info* info, int32_t rank, mhd_segment* out,
                             int32_t max_segments, int32_t* count);

/* Bytes of device workspace a mesh needs: two pitched states (8 fields of (n'+2r)^3 cells, R#4:
 * f_k and f_{k-1}), the send/recv buffers of the P:705 segments, reduction scratch and the
 * peer-memory flags.  Pure host function. */
mhd_status mhd_workspace_bytes(const mhd_mesh_info* info, size_t* bytes);

/* ---- mesh lifecycle ------------------------------------------------------ */

/* The subdomain of `rank` on the current CUDA device.
 * dev_workspace: caller-owned device memory of >= mhd_workspace_bytes, borrowed
 * until mhd_mesh_destroy.  cuda_stream: a cudaStream_t (0 = legacy default).
 * Checks divisibility (EDECOMP), n'_i > 2r (ESMALL), radius/dtype (EUNSUPPORTED).
 * The state is zero after create.  Environment knobs read here (A/B measurements only):
 * B2MHD_XWRAP, B2MHD_PERSIST, B2MHD_SLAB, B2MHD_SLAB_ZCHUNK, B2MHD_POISON (= mhd_set_debug),
 * B2MHD_SPIN_TIMEOUT_S (peer-memory flag waits, default 60 s). */
mhd_status mhd_mesh_create(const mhd_mesh_info* info, void* dev_workspace, size_t bytes,
                           void* cuda_stream, mhd_mesh** out);

/* Multi-GPU, one process per rank (the paper's MPI ranks): nccl_unique_id is the
 * 128-byte ncclUniqueId created by rank 0 (mhd_nccl_unique_id) and broadcast by the caller.
 * Collective over all ranks.  Needed for reductions and the NCCL exchange. */
mhd_status mhd_nccl_unique_id(void* out128);
mhd_status mhd_comm_init(mhd_mesh* mesh, const void* nccl_unique_id);

/* Peer-memory halo exchange over NVLink / NVSwitch (all ranks on one box).  Each rank exports
 * its workspace as a CUDA IPC handle blob of MHD_P2P_HANDLE_BYTES; the caller all-gathers the
 * blobs in rank order and passes them to mhd_p2p_open (collective, after every rank created its
 * mesh; follow it with a host barrier).  From then on the outer-shell update kernels store their
 * boundary results directly into the neighbours' halos (no pack, send/recv or unpack), ordered by
 * system-scope flags in the workspaces (the paper's P:765-782 pipeline without the
 * pack/unpack copies).  Ranks must call the same substeps in lockstep; a flag wait that outlasts
 * B2MHD_SPIN_TIMEOUT_S gives up and the next blocking call (mhd_synchronize, mhd_store to host,
 * mhd_reduce) returns MHD_ECUDA.  mhd_set_exchange(mesh, 0) returns to NCCL. */
#define MHD_P2P_HANDLE_BYTES 80
mhd_status mhd_p2p_export(mhd_mesh* mesh, void* out_blob);
mhd_status mhd_p2p_open(mhd_mesh* mesh, const void* blobs);
mhd_status mhd_set_exchange(mhd_mesh* mesh, int32_t mode); /* 0: NCCL, 1: peer memory */

/* Releases the mesh (not the caller's workspace).  With the peer-memory exchange it first waits
 * until the neighbours' stores of their last operation into this workspace have landed; the
 * caller should also barrier across ranks before freeing the workspace.  A mesh in a group:
 * MHD_EINVAL until mhd_group_destroy. */
mhd_status mhd_mesh_destroy(mhd_mesh* mesh);

/* ---- state I/O ------------------------------------------------------------ */

/* Copy a local interior buffer into the current state (converting dtype if it
 * differs from the mesh dtype).  Resets the RK3 substep counter to 0: a loaded
 * state is a step boundary, where the 2N register w is zero (alpha_0 = 0, R#3).
 * The paper's initial condition is random values in [0, 1] loaded per rank. */
mhd_status mhd_load(mhd_mesh* mesh, int32_t field, const void* src, int32_t src_dtype,
                    int32_t on_device);

/* Copy the current state's local interior into dst (the paper verifies by comparing stored
 * state against the CPU model).  Blocking when on_device == 0 (synchronises the mesh
 * stream); see mhd_store_async. */
mhd_status mhd_store(mhd_mesh* mesh, int32_t field, void* dst, int32_t dst_dtype,
                     int32_t on_device);

/* Asynchronous store into HOST memory, for snapshot pipelines: the interior of the
 * current state's field is copied on the device (in stream order, after every
 * update already enqueued) into an internal staging buffer owned by the mesh
 * (allocated on first use: 8 * nx'*ny'*nz' * dst_dtype bytes), and the
 * device->host transfer then runs on a separate copy stream, overlapping the
 * calls that follow (the next mhd_load's host->device copy, the next updates).
 * dst must stay valid and must not be read until mhd_synchronize returns; a
 * second store_async of the same field first waits for the first one's transfer.
 * Page-locked dst gives full-duplex overlap.  Errors as mhd_store. */
mhd_status mhd_store_async(mhd_mesh* mesh, int32_t field, void* dst_host, int32_t dst_dtype);

/* Asynchronous load from HOST memory, the mirror of mhd_store_async: the
 * host->device copy runs on the load copy stream into a second staging buffer
 * (allocated on first use), overlapping the updates and transfers enqueued
 * before it; the scatter into the current state then runs on the mesh stream in
 * order.  Resets the substep counter like mhd_load.  src must stay valid and
 * unmodified until mhd_synchronize returns. */
mhd_status mhd_load_async(mhd_mesh* mesh, int32_t field, const void* src_host, int32_t src_dtype);

/* Test hook: copy the halo-inclusive local grid M' of one field of the current
 * state, (nz'+6) * (ny'+6) * (nx'+6) values in the mesh dtype, x fastest, to
 * dst.  Halo cells never written (corners when exchange_corners = 0) hold
 * whatever the workspace held (zero after create).  Blocking when on_device = 0. */
mhd_status mhd_store_grid(mhd_mesh* mesh, int32_t field, void* dst, int32_t on_device);

/* ---- the hot path ---------------------------------------------------------- */

/* Fill the halo of the current state: periodic along unsplit axes, and
 * the 26-segment exchange with neighbours.  Bit-exact copies.
 * A mesh in a group: MHD_EINVAL (use mhd_group_halo_exchange). */
mhd_status mhd_halo_exchange(mhd_mesh* mesh);

/* One ISL iteration = RK3 substep k: halo exchange overlapped
 * with the inner-segment update, then the outer segments; the update is the
 * fused 6th-order stencil + RHS (B.1-B.4) + Williamson 2N RK3 (R#3):
 *   w_k = alpha_k w_{k-1} + dt RHS(f_k),  f_{k+1} = f_k + beta_k w_k,
 * with w_{k-1} reconstructed as (f_k - f_{k-1}) / beta_{k-1} (reading R#4).
 * k must follow 0, 1, 2, 0, ... after a load (else MHD_ESTATE). */
mhd_status mhd_integrate_substep(mhd_mesh* mesh, int32_t k, double dt);

/* Three substeps (one full RK3 step). */
mhd_status mhd_integrate_step(mhd_mesh* mesh, double dt);

/* Global reduction of one field of the current state over all ranks
 * (NCCL allreduce when nranks > 1).  Blocking; *out on the host.
 * MHD_ENONFINITE if the field holds a NaN/Inf (the value is still written). */
mhd_status mhd_reduce(mhd_mesh* mesh, int32_t field, int32_t op, double* out);

/* Test hook: RHS (B.1-B.4) of the current state, all 8 fields, written to
 * dev_dst as 8 consecutive local-interior arrays in the mesh dtype.  Performs a
 * halo exchange first.  Does not change the state or the substep counter. */
mhd_status mhd_debug_rhs(mhd_mesh* mesh, void* dev_dst);

/* Block the host until all work of the mesh has completed (the per-iteration device
 * synchronisation of P:782, which the substeps themselves replace by stream order).  Reports a
 * timed-out peer-memory flag wait (MHD_ECUDA). */
mhd_status mhd_synchronize(mhd_mesh* mesh);

/* ---- configuration and introspection --------------------------------------- */

/* Update kernel: 0 = auto (fastest), 1 = direct (one thread per cell, loads via
 * the read-only path), 2 = z-marching shared-memory kernel, 3 = warp-specialised z-marching
 * kernel (two threads per cell: magnetic and flow warp groups; FP64, radius 3 only, else
 * MHD_EUNSUPPORTED).  Every variant gives bit-identical results. */
mhd_status mhd_set_kernel(mhd_mesh* mesh, int32_t variant);

/* Local geometry of the mesh: P, coord, local n', and the substep counter. */
mhd_status mhd_mesh_query(const mhd_mesh* mesh, int32_t P[3], int32_t coord[3],
                          int64_t local_n[3], int32_t* next_k);

/* Debug flags.  MHD_DEBUG_POISON_HALO: before every update, every halo cell of the state the
 * update writes (and, at load, of the loaded field) is set to NaN, so that a stencil reading a
 * halo cell the schedule did not refresh (e.g. a corner, which P:937 says is never needed)
 * produces NaN.  Results are bit-identical with and without it when the schedule is right. */
#define MHD_DEBUG_POISON_HALO 1
mhd_status mhd_set_debug(mhd_mesh* mesh, int32_t flags);

/* Number of kernels the library launched on this mesh since create. */
mhd_status mhd_launch_count(const mhd_mesh* mesh, int64_t* count);

/* Per-phase device timing with CUDA events recorded on the stream each phase is
 * launched on (compute stream for the inner update and self copies; comm stream for
 * pack, exchange, unpack and the outer slabs).  enable = 1 starts recording (and clears), 0 stops. */
typedef enum {
  MHD_PHASE_UPDATE = 0,   /* fused stencil + RHS + RK3 kernel over the inner segment, or over
                             the whole subdomain when it is not split */
  MHD_PHASE_SELF = 1,     /* periodic self-copy of the halo */
  MHD_PHASE_PACK = 2,     /* pack kernel */
  MHD_PHASE_EXCHANGE = 3, /* NCCL grouped send/recv */
  MHD_PHASE_UNPACK = 4,   /* unpack kernel */
  MHD_PHASE_OUTER = 5,    /* the same update kernels over the outer-shell slabs,
                             launched on the comm stream after the halo arrives */
  MHD_NPHASES = 6
} mhd_phase;
mhd_status mhd_profile_enable(mhd_mesh* mesh, int32_t enable);

/* Blocking (synchronises the mesh).  For one phase: number of launches recorded,
 * their summed device time in ms, and the algorithmic bytes they moved (updates:
 * interior cells x 8 fields x sizeof(T) x (2 for k = 0, else 3); copies: halo
 * cells x 8 fields x sizeof(T) x 2). */
mhd_status mhd_profile_read(mhd_mesh* mesh, int32_t phase, int64_t* launches, double* ms,
                            double* algorithmic_bytes);

/* ---- several ranks in one process ---------------------------------------------------------
 * A group drives every rank of an n-rank decomposition from one host thread: meshes created
 * with nranks = n and rank = 0..n-1 (each on the CUDA device current at its create; several on
 * one device allowed), passed in rank order, without mhd_comm_init / mhd_p2p_open.  The same
 * schedules and kernels run as with one process per rank; the transfer of
 * exchange = 0 is a copy-engine pull of each neighbour's packed send buffer (cudaMemcpyAsync)
 * instead of NCCL, exchange = 1 the peer-memory stores, and cross-rank ordering uses CUDA events
 * recorded phase by phase across the ranks, so no kernel waits on another.  While grouped, the
 * per-mesh hot-path calls return MHD_EINVAL; load/store/store_grid stay per mesh.  Peer access is
 * enabled between the devices of neighbouring ranks. */
typedef struct mhd_group mhd_group; /* opaque */
mhd_status mhd_group_create(mhd_mesh* const* meshes, int32_t n, int32_t exchange, mhd_group** out);
mhd_status mhd_group_halo_exchange(mhd_group* group);
mhd_status mhd_group_integrate_substep(mhd_group* group, int32_t k, double dt);
mhd_status mhd_group_integrate_step(mhd_group* group, double dt);
/* dev_dst[i]: the RHS destination of rank i, as mhd_debug_rhs. */
mhd_status mhd_group_debug_rhs(mhd_group* group, void* const* dev_dst);
/* Global reduction: per-rank partials combined on the host in rank order. */
mhd_status mhd_group_reduce(mhd_group* group, int32_t field, int32_t op, double* out);
mhd_status mhd_group_synchronize(mhd_group* group);
/* Synchronises every rank and releases the grouping (not the meshes). */
mhd_status mhd_group_destroy(mhd_group* group);

const char* mhd_status_str(mhd_status s);
const char* mhd_last_error(void);
int32_t mhd_abi_version(void);

#ifdef __cplusplus
}
#endif
#endif /* B2MHD_H */
