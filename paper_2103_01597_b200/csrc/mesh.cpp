// Host runtime and C ABI of b2mhd (include/b2mhd.h).
//
//  * decomposition: Morton mapping P:557 (Z-order, rank -> subdomain), n' = n / p
//  * halo segments: 6 sides, 12 edges, 8 corners; segments to one peer are
//    concatenated in canonical order, so one NCCL send/recv pair per distinct peer
//    replaces the paper's per-segment MPI_Isend/Irecv with tags
//  * the ISL iteration pipeline: pack on a high-priority comm stream, exchange
//    there, the inner-segment update concurrently on the compute stream, then unpack -> outer
//    segments -> event.  Stream order replaces the paper's per-iteration
//    cudaDeviceSynchronize + MPI_Barrier.
//  * ranks run either one per process (torchrun; cross-rank ordering by system-scope flags in
//    peer memory) or several in one process (mhd_group_*: every rank's work is enqueued phase by
//    phase and ordered by CUDA events, so no kernel ever waits for another).
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

// How the periodic (self) halo of unsplit axes is kept:
//  * one rank: z planes through the TMA plane wrap (never stored), x faces by the update
//    kernels' epilogue (Geom::xwrap), y rows by a copy launch;
//  * several ranks (z always split): x faces by the epilogue when x is unsplit, y rows copied.
// (Round 1 also had a "storing" kernel variant that wrote every self and remote halo cell from
// its epilogue; measured slower, it was removed: DESIGN.md 2, profiles/r01/bench_pcopy*.)

#include "../../include/b2mhd.h"
#include "kernels.h"

using namespace b2;

namespace {

thread_local std::string g_err;

mhd_status fail(mhd_status s, const std::string& msg) {
  g_err = msg;
  return s;
}

#define CU(call)                                                                                  \
  do {                                                                                            \
    cudaError_t e_ = (call);                                                                      \
    if (e_ != cudaSuccess) return fail(MHD_ECUDA, std::string(#call ": ") + cudaGetErrorString(e_)); \
  } while (0)
#define NC(call)                                                                                   \
  do {                                                                                             \
    ncclResult_t r_ = (call);                                                                      \
    if (r_ != ncclSuccess) return fail(MHD_ENCCL, std::string(#call ": ") + ncclGetErrorString(r_)); \
  } while (0)

// ---- Morton mapping: bit 3k + j of the index is bit k of coordinate j ----------------
void morton_decode(uint32_t idx, int c[3]) {
  c[0] = c[1] = c[2] = 0;
  for (int k = 0; k < 10; ++k)
    for (int j = 0; j < 3; ++j) c[j] |= (int)(((idx >> (3 * k + j)) & 1u) << k);
}
uint32_t morton_encode(const int c[3]) {
  uint32_t idx = 0;
  for (int k = 0; k < 10; ++k)
    for (int j = 0; j < 3; ++j) idx |= (uint32_t)((c[j] >> k) & 1) << (3 * k + j);
  return idx;
}
// Morton coordinate j maps to memory axis (2 - j): coordinate 0 -> z (reading R#16).
void partition_xyz(int nranks, int P[3]) {
  int m[3];
  morton_decode((uint32_t)(nranks - 1), m);
  for (int j = 0; j < 3; ++j) P[2 - j] = m[j] + 1;
}
void coord_xyz(int rank, int c[3]) {
  int m[3];
  morton_decode((uint32_t)rank, m);
  for (int j = 0; j < 3; ++j) c[2 - j] = m[j];
}
int rank_of_xyz(const int c[3]) {
  int m[3] = {c[2], c[1], c[0]};
  return (int)morton_encode(m);
}

mhd_status check_info(const mhd_mesh_info* info) {
  if (!info) return fail(MHD_EINVAL, "info is null");
  if (info->abi_version != MHD_ABI_VERSION) return fail(MHD_EUNSUPPORTED, "ABI version mismatch");
  if (info->radius < 1 || info->radius > 4)
    return fail(MHD_EUNSUPPORTED, "radius must be 1..4 (orders 2, 4, 6, 8; P:829-830)");
  if (info->dtype != MHD_F32 && info->dtype != MHD_F64) return fail(MHD_EUNSUPPORTED, "dtype must be F32 or F64");
  if (info->nranks < 1 || (info->nranks & (info->nranks - 1)) != 0)
    return fail(MHD_EDECOMP, "nranks must be a power of two (Morton partition, P:557)");
  if (info->rank < 0 || info->rank >= info->nranks) return fail(MHD_EINVAL, "rank out of range");
  for (int a = 0; a < 3; ++a) {
    if (info->n[a] < 1) return fail(MHD_EINVAL, "n must be positive");
    if (!(info->ds[a] > 0)) return fail(MHD_EINVAL, "ds must be positive");
  }
  int P[3];
  partition_xyz(info->nranks, P);
  for (int a = 0; a < 3; ++a) {
    if (info->n[a] % P[a] != 0) return fail(MHD_EDECOMP, "p_i does not divide n_i (P:207)");
    if (info->n[a] / P[a] <= 2 * info->radius) return fail(MHD_ESMALL, "local extent n'_i <= 2r (P:705)");
  }
  return MHD_OK;
}

struct SegInfo {
  mhd_segment s;
  bool self;
};

// Segments of one rank in canonical order: sides, edges, corners; lexicographic (oz, oy, ox).
std::vector<SegInfo> build_segments(const mhd_mesh_info* info, int rank) {
  int P[3], c[3];
  partition_xyz(info->nranks, P);
  coord_xyz(rank, c);
  int64_t n[3];
  for (int a = 0; a < 3; ++a) n[a] = info->n[a] / P[a];
  const int rad = info->radius;
  std::vector<SegInfo> out;
  for (int kind = 1; kind <= 3; ++kind) {
    if (kind == 3 && !info->exchange_corners) continue;
    for (int oz = -1; oz <= 1; ++oz)
      for (int oy = -1; oy <= 1; ++oy)
        for (int ox = -1; ox <= 1; ++ox) {
          const int o[3] = {ox, oy, oz};
          if ((ox != 0) + (oy != 0) + (oz != 0) != kind) continue;
          SegInfo si;
          memset(&si, 0, sizeof(si));
          mhd_segment& s = si.s;
          s.kind = kind;
          int rc[3], sc[3];
          for (int a = 0; a < 3; ++a) {
            s.offset[a] = o[a];
            // halo cells at offset o (receiver side) and the interior cells that fill them
            // (sender side): s' = ((s - r) mod n') + r, in interior coordinates
            s.dst_first[a] = o[a] < 0 ? -rad : (o[a] == 0 ? 0 : (int)n[a]);
            s.src_first[a] = o[a] < 0 ? (int)n[a] - rad : 0;
            s.extent[a] = o[a] == 0 ? (int)n[a] : rad;
            rc[a] = ((c[a] + o[a]) % P[a] + P[a]) % P[a];
            sc[a] = ((c[a] - o[a]) % P[a] + P[a]) % P[a];
          }
          s.recv_peer = rank_of_xyz(rc);
          s.send_peer = rank_of_xyz(sc);
          si.self = s.recv_peer == rank;  // then also send_peer == rank
          s.send_buf_cell = s.recv_buf_cell = -1;
          out.push_back(si);
        }
  }
  // buffer offsets: per peer, concatenation in canonical order
  std::vector<int64_t> sc(info->nranks, 0), rcnt(info->nranks, 0);
  for (auto& si : out) {
    if (si.self) continue;
    const int64_t cells = (int64_t)si.s.extent[0] * si.s.extent[1] * si.s.extent[2];
    si.s.send_buf_cell = sc[si.s.send_peer];
    sc[si.s.send_peer] += cells;
    si.s.recv_buf_cell = rcnt[si.s.recv_peer];
    rcnt[si.s.recv_peer] += cells;
  }
  return out;
}

template <typename T>
Coef<T> make_coef(const mhd_mesh_info& info, int k, double dt) {
  Coef<T> C;
  memset(&C, 0, sizeof(C));
  // central differences of order 2r, i = 1..r (readings R#1, R#2); e_i = d_i / 4
  static const double CW[5][4] = {{0}, {1.0 / 2.0}, {2.0 / 3.0, -1.0 / 12.0}, {3.0 / 4.0, -3.0 / 20.0, 1.0 / 60.0},
                                  {4.0 / 5.0, -1.0 / 5.0, 4.0 / 105.0, -1.0 / 280.0}};
  static const double DW[5][4] = {{0}, {1.0}, {4.0 / 3.0, -1.0 / 12.0}, {3.0 / 2.0, -3.0 / 20.0, 1.0 / 90.0},
                                  {8.0 / 5.0, -1.0 / 5.0, 8.0 / 315.0, -1.0 / 560.0}};
  static const double C0[5] = {0, -2.0, -5.0 / 2.0, -49.0 / 18.0, -205.0 / 72.0};
  const int rad = info.radius;
  const double* c = CW[rad];
  const double* d = DW[rad];
  const double c0 = C0[rad];
  const double* ds = info.ds;
  for (int a = 0; a < 3; ++a) {
    for (int i = 0; i < rad; ++i) {
      C.c1[a][i] = (T)(c[i] / ds[a]);
      C.d2[a][i] = (T)(d[i] / (ds[a] * ds[a]));
    }
    C.d0[a] = (T)(c0 / (ds[a] * ds[a]));
  }
  const int pa[3] = {0, 0, 1}, pb[3] = {1, 2, 2};
  for (int p = 0; p < 3; ++p)
    for (int i = 0; i < rad; ++i) C.xw[p][i] = (T)(d[i] / 4.0 / (ds[pa[p]] * ds[pb[p]]));
  const mhd_params& ph = info.phys;
  C.gamma_cp = (T)(ph.gamma / ph.cp);
  C.gm1 = (T)(ph.gamma - 1.0);
  C.inv_cp = (T)(1.0 / ph.cp);
  C.lnrho0 = (T)ph.lnrho0;
  C.cs0sq = (T)(ph.cs0 * ph.cs0);
  C.inv_T0 = (T)std::exp(-ph.lnT0);
  C.H_C = (T)(ph.H - ph.C);
  C.eta_inv_mu0 = (T)(ph.eta / ph.mu0);
  C.inv_mu0 = (T)(1.0 / ph.mu0);
  C.nu = (T)ph.nu;
  C.nu3 = (T)(ph.nu / 3.0);
  C.two_nu = (T)(2.0 * ph.nu);
  C.zeta = (T)ph.zeta;
  C.eta = (T)ph.eta;
  C.K = (T)ph.K;
  for (int i = 0; i < RMAX; ++i)
    for (int a = 0; a < 2; ++a) {
      C.xy_c1[i][a] = C.c1[a][i];
      C.xy_d2[i][a] = C.d2[a][i];
    }
  C.xy_d0[0] = C.d0[0];
  C.xy_d0[1] = C.d0[1];
  // Williamson (1980) 2N RK3 (R#3)
  const double alpha[3] = {0.0, -5.0 / 9.0, -153.0 / 128.0};
  const double beta[3] = {1.0 / 3.0, 15.0 / 16.0, 8.0 / 15.0};
  for (int j = 0; j < 3; ++j) {
    C.rkB[j] = (T)(beta[j] * dt);
    C.rkA[j] = j == 0 ? (T)0 : (T)(beta[j] * alpha[j] / beta[j - 1]);
  }
  (void)k;
  return C;
}

size_t align_up(size_t v, size_t a) { return (v + a - 1) / a * a; }

struct Layout {
  int64_t n[3];
  int64_t xo;    // elements of left pad: interior x = 0 sits at row offset xo (128-byte aligned)
  int64_t sy, sz, field_elems, origin;
  size_t field_bytes, state_off[2], send_off, recv_off, red_off, flags_off, total;
  int64_t send_cells, recv_cells;
};

Layout make_layout(const mhd_mesh_info* info, const std::vector<SegInfo>& segs) {
  Layout L;
  int P[3];
  partition_xyz(info->nranks, P);
  const size_t es = (size_t)info->dtype;
  const int64_t al = 128 / (int64_t)es;
  for (int a = 0; a < 3; ++a) L.n[a] = info->n[a] / P[a];
  L.xo = al;
  const int rad = info->radius;
  L.sy = (int64_t)align_up((size_t)(L.xo + L.n[0] + rad + 1), (size_t)al);
  L.sz = L.sy * (L.n[1] + 2 * rad);
  // + one row and a chunk of slack: tiled kernels may over-read (never use) past the last halo row
  L.field_elems = (int64_t)align_up((size_t)(L.sz * (L.n[2] + 2 * rad) + L.sy + 4 * al), (size_t)(256 / es));
  L.origin = rad * L.sz + rad * L.sy + L.xo;
  L.field_bytes = (size_t)L.field_elems * es;
  size_t off = 0;
  for (int s = 0; s < 2; ++s) {
    L.state_off[s] = off;
    off += NF * L.field_bytes;
  }
  L.send_cells = L.recv_cells = 0;
  for (auto& si : segs)
    if (!si.self) {
      const int64_t cells = (int64_t)si.s.extent[0] * si.s.extent[1] * si.s.extent[2];
      L.send_cells += cells;
      L.recv_cells += cells;
    }
  L.send_off = off;
  off = align_up(off + (size_t)L.send_cells * NF * es, 256);
  L.recv_off = off;
  off = align_up(off + (size_t)L.recv_cells * NF * es, 256);
  L.red_off = off;
  off = align_up(off + kReduceBlocks * kReduceVals * sizeof(double), 256);
  // peer-memory exchange flags: arrive[nranks] then done[nranks] (slot p written by rank p), then
  // the spin-timeout word
  L.flags_off = off;
  off = align_up(off + (2 * (size_t)info->nranks + 1) * sizeof(unsigned long long), 256);
  L.total = off;
  return L;
}

}  // namespace

struct PeerXfer {
  int peer;
  int64_t send_cell0, send_cells, recv_cell0, recv_cells;
};

// Several ranks driven by one process (mhd_group_create): the meshes in rank order.
struct mhd_group {
  std::vector<mhd_mesh*> m;
  int exchange = 0;
};

constexpr int kRing = 4;  // group mode: per-operation events, indexed by sequence number mod kRing

struct mhd_mesh {
  mhd_mesh_info info;
  int P[3], coord[3];
  Layout L;
  Geom g;
  char* ws;
  int device = 0;
  cudaStream_t stream;
  cudaStream_t comm_stream = nullptr;
  cudaEvent_t ev_ready = nullptr, ev_halo = nullptr;
  std::vector<SegInfo> segs;
  std::vector<PeerXfer> peers;
  SegList self_list, pack_list, unpack_list;
  SegList self_list_xy;  // self segments without a z component (z halo fetched by TMA wrap)
  SegList self_list_y;   // ... and with a y component (x faces written by the update epilogue)
  SegList remote_list;   // remote segments, buf_off = peer slot (peer-memory exchange)
  // Periodic x faces written by the update kernels' epilogue (Geom::xwrap: predicated stores of
  // the cells within one sector of an x face; B2MHD_XWRAP=0 disables).  One rank: the y rows are
  // then copied (0.014 ms instead of 0.06 ms for x and y) and the z planes are wrapped by TMA:
  // 12.87 -> 13.1 Gcell/s FP64, 21.0 -> 22.2 FP32 (profiles/r01/bench_xw2_*).
  bool xwrap = true;
  bool x_valid = false;  // the x faces of the current state were written by the last update
  bool x_fits() const {
    const int64_t W = 32 / (int64_t)info.dtype;
    return xwrap && L.sy - L.xo - g.nx >= W && g.nx >= 2 * W;
  }
  // persistent z-march schedule (one CTA per SM slot, equal plane ranges; B2MHD_PERSIST=1, one
  // rank only): measured 8 % slower than the chunked grid (11.70 vs 12.66 Gcell/s,
  // profiles/r01/bench_pers*.json): CTAs that run together no longer work on neighbouring tiles
  // at the same z, so the halo rows they share stop hitting in L2.  Off by default.
  bool persist = false;
  int persist_env = -1;
  // z chunk of the boundary-slab launches on the side stream: 16 planes for FP32 (more, shorter
  // CTAs shorten the slab chain, which is the critical path next to the fast FP32 inner segment:
  // 65.3 -> 82.7 Gcell/s at 4 GPUs), the default 64 for FP64 (16: -2 %; profiles/r01/bench_szc*).
  // B2MHD_SLAB_ZCHUNK=n overrides (0: 64).
  int slab_zchunk = -1;
  int zchunk_env = -1;  // z chunk of main-stream update launches (-1: wave-balanced, zmarch.cuh)
  int slab_env[3] = {0, 0, 0};
  ncclComm_t comm = nullptr;
  int cur = 0;
  int next_k = 0;
  int variant = 0;
  int split_env = -1;  // variant 0: warp-specialised z-march (B2MHD_ZSPLIT=0/1; -1: per-radius default)
  // peer-memory substeps: each boundary slab waits only for the neighbours whose halo it reads
  // (B2MHD_FINE_ARRIVAL=0: one wait for every neighbour before the first slab, the round-1
  // schedule).  Default: FP64 only.  The per-slab wait kernels co-reside with FP64 inner CTAs
  // (240 registers x 256 threads leave room for a small block), but an FP32 inner CTA takes the
  // whole register file (127 x 512), so each wait kernel then queues for a free SM: 4 GPUs FP32
  // 83.1 (per-slab) vs 86.9 Gcell/s (one wait); FP64 50.3 vs 50.2 (profiles/r02/mgpu/)
  int fine_env = -1;
  bool fine_arrival = true;
  int64_t launches = 0;
  double* h_red = nullptr;  // pinned
  TmapSet tmaps[2];          // [state read with the stencil]
  bool tmaps_ok = false;
  // exchange of the remote halo: 0 = packed segments (NCCL send/recv between processes; a
  // copy-engine pull from the neighbour's send buffer inside a group), 1 = peer memory (the new
  // boundary cells stored straight into the neighbours' halos)
  int exchange = 0;
  mhd_group* group = nullptr;       // set: this rank is driven by mhd_group_* in this process
  std::vector<char*> peer_ws;       // workspace of every rank as mapped here (nullptr: not a neighbour)
  std::vector<void*> ipc_bases;     // opened IPC allocations (closed at destroy)
  unsigned long long seq = 0;       // cross-rank operations so far (the same on every rank)
  unsigned long long op_seq = 0;    // sequence number of the operation in progress
  bool halo_valid = false;          // halos of the current state already delivered by the last update
  bool self_valid = false;          // periodic self-wrap halo of the current state is up to date
  FlagSet peer_arrive, peer_done, my_arrive, my_done;
  unsigned long long spin_timeout_ns = 60ull * 1000000000ull;  // B2MHD_SPIN_TIMEOUT_S
  cudaEvent_t ev_arrive[kRing] = {}, ev_done[kRing] = {};     // group mode
  int debug = 0;                    // MHD_DEBUG_* flags
  // asynchronous host I/O (mhd_store_async / mhd_load_async): per direction a device staging
  // buffer (8 interior fields), a copy stream and per-field events: ev_dev = the device side of
  // the slot is done (gathered for a store, scattered into the state for a load), ev_host = the
  // PCIe copy of the slot is done
  struct AsyncLane {
    char* stage = nullptr;
    int es = 0;
    cudaStream_t st = nullptr;
    cudaEvent_t ev_dev[NF] = {}, ev_host[NF] = {};
  } aio[2];  // [0] store (device -> host), [1] load (host -> device)
  template <typename T>
  RemoteMap<T> remote_map(int dest_state) const {
    RemoteMap<T> rm;
    memset(&rm, 0, sizeof(rm));
    for (size_t i = 0; i < peers.size() && i < (size_t)kMaxPeers; ++i)
      for (int q = 0; q < NF; ++q)
        rm.f[i][q] = reinterpret_cast<T*>(peer_ws[peers[i].peer] + L.state_off[dest_state] +
                                          (size_t)q * L.field_bytes) + L.origin;
    return rm;
  }
  // profiling: (start, stop) event pairs per phase, with the algorithmic bytes of the launch
  struct Rec {
    cudaEvent_t a, b;
    double bytes;
  };
  bool prof = false;
  std::vector<Rec> recs[MHD_NPHASES];
  std::vector<cudaEvent_t> pool;
  cudaEvent_t take_event() {
    if (pool.empty()) {
      cudaEvent_t e;
      cudaEventCreate(&e);
      return e;
    }
    cudaEvent_t e = pool.back();
    pool.pop_back();
    return e;
  }

  template <typename T>
  Fields<T> fields(int s) const {
    Fields<T> F;
    for (int q = 0; q < NF; ++q)
      F.f[q] = reinterpret_cast<T*>(ws + L.state_off[s] + (size_t)q * L.field_bytes) + L.origin;
    return F;
  }
  template <typename T>
  T* send_buf() const { return reinterpret_cast<T*>(ws + L.send_off); }
  template <typename T>
  T* recv_buf() const { return reinterpret_cast<T*>(ws + L.recv_off); }
  double* red_scratch() const { return reinterpret_cast<double*>(ws + L.red_off); }
  unsigned long long* flags() const { return reinterpret_cast<unsigned long long*>(ws + L.flags_off); }
  unsigned long long* err_word() const { return flags() + 2 * info.nranks; }
  bool distributed() const { return info.nranks > 1; }
};

namespace {

SegList make_list(const mhd_mesh& m, bool self, bool send, bool no_z = false, bool need_y = false) {
  SegList Ls;
  memset(&Ls, 0, sizeof(Ls));
  int nb = 0;
  for (auto& si : m.segs) {
    if (si.self != self) continue;
    if (no_z && si.s.offset[2] != 0) continue;
    if (need_y && si.s.offset[1] == 0) continue;
    SegDesc& d = Ls.s[Ls.n++];
    for (int a = 0; a < 3; ++a) {
      d.src[a] = si.s.src_first[a];
      d.dst[a] = si.s.dst_first[a];
      d.ext[a] = si.s.extent[a];
    }
    if (self && d.ext[0] == m.info.radius && m.g.nx >= 32 / (int)m.info.dtype) {
      // x-face self copies: widen the r-cell rows to one whole 32-byte sector (4 doubles, 8
      // floats) so that every load and store is a full sector; the extra cells land in the
      // unused row padding (left pad = 128 B, right pad checked) and are never read.
      const int W = 32 / (int)m.info.dtype, extra = W - m.info.radius;
      const bool fits = d.dst[0] < 0 || m.L.sy - m.L.xo - m.g.nx >= W;
      if (extra > 0 && fits) {
        if (d.dst[0] < 0) {
          d.dst[0] -= extra;
          d.src[0] -= extra;
        }
        d.ext[0] = W;
      }
    }
    d.count = (long long)d.ext[0] * d.ext[1] * d.ext[2];
    d.buf_off = 0;
    if (!self) {
      // global buffer offset = peer base + cell offset inside the peer's buffer, in values
      for (auto& p : m.peers) {
        if (send && p.peer == si.s.send_peer) d.buf_off = (p.send_cell0 + si.s.send_buf_cell) * NF;
        if (!send && p.peer == si.s.recv_peer) d.buf_off = (p.recv_cell0 + si.s.recv_buf_cell) * NF;
      }
    }
    d.block0 = nb;
    nb += (int)((d.count + 255) / 256);
  }
  Ls.nblocks = nb;
  return Ls;
}

// Remote segments for the peer-memory exchange: the P:705 send region of each segment, stored at
// the receiver's halo position; buf_off = the peer's slot in the mesh's peer list.
SegList make_remote_list(const mhd_mesh& m) {
  SegList Ls;
  memset(&Ls, 0, sizeof(Ls));
  int nb = 0;
  for (auto& si : m.segs) {
    if (si.self) continue;
    SegDesc& d = Ls.s[Ls.n++];
    for (int a = 0; a < 3; ++a) {
      d.src[a] = si.s.src_first[a];
      d.dst[a] = si.s.dst_first[a];
      d.ext[a] = si.s.extent[a];
    }
    d.count = (long long)d.ext[0] * d.ext[1] * d.ext[2];
    d.buf_off = 0;
    for (size_t i = 0; i < m.peers.size(); ++i)
      if (m.peers[i].peer == si.s.send_peer) d.buf_off = (long long)i;
    d.block0 = nb;
    nb += (int)((d.count + 255) / 256);
  }
  Ls.nblocks = nb;
  return Ls;
}

// TMA descriptors of the z-marching kernel: per state and field, a 3-D view
// (x: row pitch sy, y: ny + 2r rows, z: nz + 2r planes) of the pitched field, with the halo box
// and the f_{k-1} box of the kernel's tile.
mhd_status encode_tmaps(mhd_mesh* m) {
  static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
  if (!encode) {
    cudaDriverEntryPointQueryResult q;
    void* fn = nullptr;
    CU(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
    if (q != cudaDriverEntryPointSuccess || !fn) return fail(MHD_ECUDA, "cuTensorMapEncodeTiled unavailable");
    encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  }
  const bool f64 = m->info.dtype == MHD_F64;
  const size_t es = (size_t)m->info.dtype;
  const int rad = m->info.radius;
  const cuuint64_t dims[3] = {(cuuint64_t)m->L.sy, (cuuint64_t)(m->g.ny + 2 * rad), (cuuint64_t)(m->g.nz + 2 * rad)};
  const cuuint64_t strides[2] = {(cuuint64_t)(m->L.sy * es), (cuuint64_t)(m->L.sz * es)};
  int cols = 0, rows = 0, pty = 0;
  switch (rad) {
#define B2_BOX(RR)                                                             \
  case RR:                                                                     \
    cols = f64 ? zm_cols<double, RR>() : zm_cols<float, RR>();                 \
    rows = f64 ? zm_rows<double, RR>() : zm_rows<float, RR>();                 \
    pty = f64 ? zm_ty<double, RR>() : zm_ty<float, RR>();                      \
    break;
    B2_BOX(1) B2_BOX(2) B2_BOX(3) B2_BOX(4)
#undef B2_BOX
  }
  const cuuint32_t halo_box[3] = {(cuuint32_t)cols, (cuuint32_t)rows, 1};
  const cuuint32_t prev_box[3] = {(cuuint32_t)(f64 ? zm_pcols<double>() : zm_pcols<float>()), (cuuint32_t)pty, 1};
  const cuuint32_t estr[3] = {1, 1, 1};
  for (int s = 0; s < 2; ++s)
    for (int q = 0; q < NF; ++q) {
      for (int which = 0; which < 2; ++which) {
        const int state = which == 0 ? s : 1 - s;
        void* base = m->ws + m->L.state_off[state] + (size_t)q * m->L.field_bytes;
        CUtensorMap* map = which == 0 ? &m->tmaps[s].halo[q] : &m->tmaps[s].prev[q];
        CUresult r = encode(map, f64 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, base, dims,
                            strides, which == 0 ? halo_box : prev_box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                            CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) return fail(MHD_ECUDA, "cuTensorMapEncodeTiled failed: " + std::to_string((int)r));
      }
    }
  m->tmaps_ok = true;
  return MHD_OK;
}

// Phase timer: records a start event now and the stop event when it goes out of scope.
struct PhaseTimer {
  mhd_mesh* m;
  cudaStream_t st;
  int phase;
  double bytes;
  cudaEvent_t a = nullptr;
  PhaseTimer(mhd_mesh* m_, cudaStream_t s_, int ph, double by) : m(m_), st(s_), phase(ph), bytes(by) {
    if (m->prof) {
      a = m->take_event();
      cudaEventRecord(a, st);
    }
  }
  ~PhaseTimer() {
    if (!a) return;
    cudaEvent_t b = m->take_event();
    cudaEventRecord(b, st);
    m->recs[phase].push_back({a, b, bytes});
  }
};

double seg_bytes(const SegList& L, size_t es) {
  double c = 0;
  for (int i = 0; i < L.n; ++i) c += (double)L.s[i].count;
  return c * NF * (double)es * 2.0;
}

// ---- cross-rank ordering ---------------------------------------------------------------------------
// Every operation that touches halos across ranks has a sequence number s (the same on every rank)
// and two parts: a local part closed by xr_arrive(s), and a remote part opened by xr_wait(s).
//  * Process mode (one process per GPU): xr_arrive is the flag kernel that publishes arrive = s to
//    every neighbour and waits for each neighbour's arrive >= s and done >= s - 1 (kernels.cu);
//    xr_wait is empty; xr_done publishes done = s.
//  * Group mode (one process drives every rank, mhd_group_*): xr_arrive records an event; xr_wait
//    makes the stream wait for every neighbour's arrive(s) and done(s - 1) events; xr_done records
//    done(s).  The group driver runs a phase on every rank before the next phase on any, so each
//    event is recorded before anyone waits on it, and no kernel ever waits for another (running
//    waiting kernels of several ranks on one GPU can deadlock: B200_PROFILING.md).
void xr_arrive(mhd_mesh* m, cudaStream_t st, unsigned long long s) {
  if (m->group) {
    cudaEventRecord(m->ev_arrive[s % kRing], st);
  } else {
    launch_p2p_sync(st, m->peer_arrive, m->my_arrive, m->my_done, s, m->err_word(), m->spin_timeout_ns);
    m->launches++;
  }
}
void xr_wait(mhd_mesh* m, cudaStream_t st, unsigned long long s) {
  if (!m->group) return;  // the flag kernel of xr_arrive waited
  for (auto& p : m->peers) {
    mhd_mesh* n = m->group->m[p.peer];
    cudaStreamWaitEvent(st, n->ev_arrive[s % kRing], 0);
    if (s > 1) cudaStreamWaitEvent(st, n->ev_done[(s - 1) % kRing], 0);
  }
}
void xr_done(mhd_mesh* m, cudaStream_t st, unsigned long long s) {
  if (m->group) {
    cudaEventRecord(m->ev_done[s % kRing], st);
  } else {
    launch_p2p_signal(st, m->peer_done, s);
    m->launches++;
  }
}
// Fine-grained arrival (mhd_mesh::fine_arrival): the three parts of xr_arrive + xr_wait separately.
// xr_signal_arrive(s): publish arrive = s (all earlier work of this rank is complete: it is done
// reading the halo the neighbours are about to overwrite), without waiting.
void xr_signal_arrive(mhd_mesh* m, cudaStream_t st, unsigned long long s) {
  if (m->group) {
    cudaEventRecord(m->ev_arrive[s % kRing], st);
  } else {
    launch_p2p_signal(st, m->peer_arrive, s);
    m->launches++;
  }
}
// wait for done >= s of the neighbours `which` (indices into m->peers)
void xr_wait_done_of(mhd_mesh* m, cudaStream_t st, unsigned long long s, const std::vector<int>& which) {
  if (s == 0 || which.empty()) return;
  if (m->group) {
    for (int i : which) cudaStreamWaitEvent(st, m->group->m[m->peers[i].peer]->ev_done[s % kRing], 0);
  } else {
    FlagSet fs;
    memset(&fs, 0, sizeof(fs));
    for (int i : which) fs.ptr[fs.n++] = m->my_done.ptr[i];
    launch_p2p_wait(st, fs, s, m->err_word(), m->spin_timeout_ns);
    m->launches++;
  }
}
// wait for arrive >= s of every neighbour
void xr_wait_arrive(mhd_mesh* m, cudaStream_t st, unsigned long long s) {
  if (m->peers.empty()) return;
  if (m->group) {
    for (auto& p : m->peers) cudaStreamWaitEvent(st, m->group->m[p.peer]->ev_arrive[s % kRing], 0);
  } else {
    launch_p2p_wait(st, m->my_arrive, s, m->err_word(), m->spin_timeout_ns);
    m->launches++;
  }
}

// wait until every neighbour finished operation s (its stores into this rank's halo have landed)
void xr_wait_done(mhd_mesh* m, cudaStream_t st, unsigned long long s) {
  if (s == 0 || m->peers.empty()) return;
  if (m->group) {
    for (auto& p : m->peers) cudaStreamWaitEvent(st, m->group->m[p.peer]->ev_done[s % kRing], 0);
  } else {
    launch_p2p_wait(st, m->my_done, s, m->err_word(), m->spin_timeout_ns);
    m->launches++;
  }
}

// The update of one region of the subdomain, with the kernels of the mesh's stencil radius.
template <typename T, int RAD>
void update_region_r(mhd_mesh* m, cudaStream_t st, const Region& r, int k, double dt, T* rhs_out) {
  const Fields<T> in = m->fields<T>(m->cur), out = m->fields<T>(1 - m->cur);
  const Coef<T> C = make_coef<T>(m->info, k, dt);
  const bool zm = m->variant != 1 && m->tmaps_ok && zmarch_supported<T, RAD>(m->g, r);
  const double cells = (double)r.ext[0] * r.ext[1] * r.ext[2];
  PhaseTimer t(m, st, st == m->stream ? MHD_PHASE_UPDATE : MHD_PHASE_OUTER,
               cells * NF * sizeof(T) * (rhs_out ? 2.0 : (k == 0 ? 2.0 : 3.0)));
  // main stream: wave-balanced z chunks (B2MHD_ZCHUNK overrides); boundary slabs: 16 (FP32) / 32
  // (FP64: 50.6 vs 49.2 Gcell/s with 64 at 4 GPUs weak, profiles/r02/mgpu/slabc_*)
  const int zchunk = st == m->stream ? m->zchunk_env
                                     : (m->slab_zchunk >= 0 ? m->slab_zchunk : (sizeof(T) == 4 ? 16 : 32));
  bool done = false;
  if constexpr (std::is_same<T, double>::value && (RAD == 3 || RAD == 4)) {
    // warp-specialised variant (zsplit.cuh): variant 3, or variant 0 when enabled for the mesh
    // (B2MHD_ZSPLIT; default on for radius 4, where it doubles the warps per SM)
    const bool want = m->variant == 3 || (m->variant == 0 && (m->split_env >= 0 ? m->split_env != 0 : RAD == 4));
    if (zm && want && zsplit_supported<T, RAD>(m->g, r)) {
      launch_zsplit<T, RAD>(st, m->tmaps[m->cur], out, m->g, r, C, k, rhs_out, (int)m->L.xo, zchunk);
      done = true;
    }
  }
  if (done) {
  } else if (zm)
    launch_zmarch<T, RAD>(st, m->tmaps[m->cur], out, m->g, r, C, k, rhs_out, (int)m->L.xo, m->persist, zchunk);
  else
    launch_direct<T, RAD>(st, in, out, m->g, r, C, k, rhs_out);
  m->launches++;
}

template <typename T>
void update_region(mhd_mesh* m, const Region& r, int k, double dt, T* rhs_out, cudaStream_t st = nullptr) {
  if (r.ext[0] <= 0 || r.ext[1] <= 0 || r.ext[2] <= 0) return;
  if (!st) st = m->stream;
  switch (m->info.radius) {
    case 1: update_region_r<T, 1>(m, st, r, k, dt, rhs_out); break;
    case 2: update_region_r<T, 2>(m, st, r, k, dt, rhs_out); break;
    case 3: update_region_r<T, 3>(m, st, r, k, dt, rhs_out); break;
    case 4: update_region_r<T, 4>(m, st, r, k, dt, rhs_out); break;
  }
}

template <typename T>
bool zmarch_ok(const mhd_mesh* m, const Region& r) {
  switch (m->info.radius) {
    case 1: return zmarch_supported<T, 1>(m->g, r);
    case 2: return zmarch_supported<T, 2>(m->g, r);
    case 3: return zmarch_supported<T, 3>(m->g, r);
    case 4: return zmarch_supported<T, 4>(m->g, r);
  }
  return false;
}

// MHD_DEBUG_POISON_HALO: before an update, NaN into every halo cell of the state it writes (its
// interior holds f_{k-1}, read pointwise; its halo is refilled by this and the next substep's
// exchange).  A cell the schedule fails to refresh before a stencil reads it poisons the result.
template <typename T>
void poison_out(mhd_mesh* m, T* rhs_out) {
  if (!(m->debug & MHD_DEBUG_POISON_HALO) || rhs_out) return;
  launch_poison_halo<T>(m->stream, m->fields<T>(1 - m->cur), m->g, m->info.radius);
  m->launches++;
}

// Periodic self-copy of the halo, only when the last update did not already write it.
template <typename T>
void ensure_self(mhd_mesh* m) {
  // several ranks (z split, so every self segment lies in the xy plane): the x faces may already
  // be written by the last update's epilogue (x_valid), then only the segments with a y
  // component remain.  One rank: the whole list (its z halo is not kept by the substeps).
  const SegList& L = m->x_valid && m->distributed() ? m->self_list_y : m->self_list;
  if (L.n && !m->self_valid) {
    PhaseTimer t(m, m->stream, MHD_PHASE_SELF, seg_bytes(L, sizeof(T)));
    launch_segments<T>(m->stream, m->fields<T>(m->cur), m->g, L, SEG_SELF, nullptr);
    m->launches++;
  }
  m->self_valid = true;
}

// Inner region and outer slabs: only axes split across ranks need the remote halo;
// along unsplit axes the whole extent is inner (its halo is a self copy).  `thick` is the slab
// width per axis (at least the radius; one tile wide so that the slabs run on the tiled kernel).
void split_regions(const mhd_mesh* m, Region& inner, std::vector<Region>& outer, const int thick_in[3]) {
  const int n[3] = {m->g.nx, m->g.ny, m->g.nz};
  bool split[3];
  int thick[3];
  for (int a = 0; a < 3; ++a) {
    split[a] = m->P[a] > 1;
    thick[a] = std::max(m->info.radius, std::min(thick_in[a], n[a] / 2));
    inner.lo[a] = split[a] ? thick[a] : 0;
    inner.ext[a] = split[a] ? n[a] - 2 * thick[a] : n[a];
  }
  outer.clear();
  // slabs: z first (full x, y), then y (full x, inner z), then x (inner y, z)
  int lo[3] = {0, 0, 0}, hi[3] = {n[0], n[1], n[2]};
  for (int a = 2; a >= 0; --a) {
    if (!split[a]) continue;
    for (int side = 0; side < 2; ++side) {
      Region r;
      for (int b = 0; b < 3; ++b) {
        r.lo[b] = lo[b];
        r.ext[b] = hi[b] - lo[b];
      }
      r.lo[a] = side == 0 ? 0 : n[a] - thick[a];
      r.ext[a] = thick[a];
      if (r.ext[0] > 0 && r.ext[1] > 0 && r.ext[2] > 0) outer.push_back(r);
    }
    lo[a] = thick[a];
    hi[a] = n[a] - thick[a];
  }
  if (inner.ext[0] <= 0 || inner.ext[1] <= 0 || inner.ext[2] <= 0) inner.ext[0] = inner.ext[1] = inner.ext[2] = 0;
}

// The neighbours (indices into m->peers) whose halo cells the stencil of region r reads: every
// remote P:705 segment whose halo box meets r grown by the radius; 3-D corner segments are never
// read (Eq. 14 has no 3-D corner points).
std::vector<int> region_peers(const mhd_mesh* m, const Region& r) {
  std::vector<int> out;
  const int rad = m->info.radius;
  for (auto& si : m->segs) {
    if (si.self || si.s.kind == 3) continue;
    bool meets = true;
    for (int a = 0; a < 3; ++a) {
      const int h0 = si.s.dst_first[a], h1 = h0 + si.s.extent[a];
      const int b0 = r.lo[a] - rad, b1 = r.lo[a] + r.ext[a] + rad;
      meets = meets && h0 < b1 && b0 < h1;
    }
    if (!meets) continue;
    for (size_t i = 0; i < m->peers.size(); ++i)
      if (m->peers[i].peer == si.s.recv_peer && std::find(out.begin(), out.end(), (int)i) == out.end())
        out.push_back((int)i);
  }
  return out;
}

// Boundary-slab widths (x, y, z): one tile wide in x and y so that the slabs run on the tiled
// kernel; in z 8 planes for the packed exchange (the slabs wait for it: keep them small) and 16
// for the peer-memory exchange (the slabs run first, beside the inner segment: fewer planes lost
// to the 2r-plane prologue).  Measured at 256^3 per GPU (profiles/r01/bench_slab*.json): p2p 4
// GPUs 44.6 -> 45.9, 2 GPUs 22.7 -> 23.1 Gcell/s; NCCL best at 8.  B2MHD_SLAB="x,y,z" overrides.
template <typename T>
void slab_thickness(const mhd_mesh* m, int thick[3]) {
  thick[0] = zm_tx<T>();
  // 8 rows (for the 16-row FP32 order-6 tile a 16-row slab measured the same: 65.0 vs 65.8
  // Gcell/s at 4 GPUs, profiles/r01/bench_f32s_*.json)
  thick[1] = 8;
  thick[2] = m->exchange == 1 ? 16 : 8;
  if (m->slab_env[0] > 0)
    for (int a = 0; a < 3; ++a) thick[a] = m->slab_env[a];
}

// ---- the operations of the schedules, phase by phase ----------------------------------------------
// Each returns MHD_OK; phase 0 is the local part (ends with xr_arrive where there is a cross-rank
// step), phase 1 the remote part.  Process mode runs both phases of one mesh back to back; a
// group runs phase 0 of every rank, then phase 1 of every rank (run_phases).

// Peer-memory halo copy of the current state (after a load, or for mhd_halo_exchange): the P:705
// send regions straight into the neighbours' halos.
template <typename T>
mhd_status op_p2p_halo_copy(mhd_mesh* m, int ph) {
  if (ph == 0) {
    ensure_self<T>(m);
    m->op_seq = ++m->seq;
    xr_arrive(m, m->stream, m->op_seq);
  } else {
    const unsigned long long s = m->op_seq;
    xr_wait(m, m->stream, s);
    {
      PhaseTimer t(m, m->stream, MHD_PHASE_PACK, seg_bytes(m->remote_list, sizeof(T)));
      launch_remote_copy<T>(m->stream, m->fields<T>(m->cur), m->g, m->remote_list, m->remote_map<T>(m->cur));
      m->launches++;
    }
    xr_done(m, m->stream, s);
    m->halo_valid = true;
  }
  CU(cudaGetLastError());
  return MHD_OK;
}

// Peer-memory substep.  Side stream (high priority): wait until every
// neighbour is done with its previous operation, update the boundary slabs (one tile thick), then
// one copy kernel stores the new boundary cells (the send regions of P:705, all inside the slabs
// just written, L2-hot) into the neighbours' halos of the new state, and publishes done.  Compute
// stream, concurrently: the inner segment (needs no remote halo).  The x faces of an unsplit x
// axis are written by every update's epilogue; the y halo of an unsplit y axis is copied at the
// next substep's start.
template <typename T>
mhd_status op_p2p_substep(mhd_mesh* m, int ph, int k, double dt, T* rhs_out) {
  const bool xw = m->P[0] == 1 && m->x_fits();
  if (ph == 0) {
    poison_out<T>(m, rhs_out);
    ensure_self<T>(m);
    m->op_seq = ++m->seq;
    CU(cudaEventRecord(m->ev_ready, m->stream));
    CU(cudaStreamWaitEvent(m->comm_stream, m->ev_ready, 0));
    PhaseTimer t(m, m->comm_stream, MHD_PHASE_EXCHANGE, 0.0);
    if (m->fine_arrival)
      xr_signal_arrive(m, m->comm_stream, m->op_seq);
    else
      xr_arrive(m, m->comm_stream, m->op_seq);
    CU(cudaGetLastError());
    return MHD_OK;
  }
  const unsigned long long s = m->op_seq;
  Region inner;
  std::vector<Region> outer;
  int thick[3];
  slab_thickness<T>(m, thick);
  split_regions(m, inner, outer, thick);
  if (!m->fine_arrival) xr_wait(m, m->comm_stream, s);
  m->g.xwrap = !rhs_out && xw ? 1 : 0;
  for (auto& r : outer) {
    // per-slab arrival (the fine-grained start of P:1013): this slab waits only
    // until the neighbours whose halo it reads have landed their stores of operation s - 1
    if (m->fine_arrival) xr_wait_done_of(m, m->comm_stream, s - 1, region_peers(m, r));
    update_region<T>(m, r, k, dt, rhs_out, m->comm_stream);
  }
  // the copy into the neighbours' halos of the new state waits until each is done reading it
  if (m->fine_arrival) xr_wait_arrive(m, m->comm_stream, s);
  if (!rhs_out) {
    PhaseTimer t(m, m->comm_stream, MHD_PHASE_PACK, seg_bytes(m->remote_list, sizeof(T)));
    launch_remote_copy<T>(m->comm_stream, m->fields<T>(1 - m->cur), m->g, m->remote_list, m->remote_map<T>(1 - m->cur));
    m->launches++;
  }
  xr_done(m, m->comm_stream, s);
  CU(cudaEventRecord(m->ev_halo, m->comm_stream));
  update_region<T>(m, inner, k, dt, rhs_out);
  m->g.xwrap = 0;
  CU(cudaStreamWaitEvent(m->stream, m->ev_halo, 0));
  if (!rhs_out) {
    m->halo_valid = true;
    m->self_valid = !m->self_list.n || (xw && !m->self_list_y.n);
    m->x_valid = xw;
  }
  CU(cudaGetLastError());
  return MHD_OK;
}

// Packed exchange of the current state's remote halo on the side stream: pack ->
// transfer -> unpack.  Transfer: NCCL grouped send/recv per distinct peer between processes; in a
// group, each rank pulls its neighbours' send-buffer slices into its receive buffer with the copy
// engines (cudaMemcpyAsync over NVLink or within a device), ordered by events.
// Phase 0 ends after the pack (group) or the unpack (NCCL); phase 1 completes the transfer.
template <typename T>
mhd_status xchg_packed(mhd_mesh* m, int ph) {
  const Fields<T> F = m->fields<T>(m->cur);
  if (ph == 0) {
    ensure_self<T>(m);
    CU(cudaEventRecord(m->ev_ready, m->stream));
    CU(cudaStreamWaitEvent(m->comm_stream, m->ev_ready, 0));
    if (m->group) {
      m->op_seq = ++m->seq;
      xr_wait_done(m, m->comm_stream, m->op_seq - 1);  // neighbours finished pulling the last pack
    } else if (!m->comm) {
      return fail(MHD_ENCCL, "mhd_comm_init was not called");
    }
    {
      PhaseTimer t(m, m->comm_stream, MHD_PHASE_PACK, seg_bytes(m->pack_list, sizeof(T)));
      launch_segments<T>(m->comm_stream, F, m->g, m->pack_list, SEG_PACK, m->send_buf<T>());
      m->launches++;
    }
    if (m->group) {
      xr_arrive(m, m->comm_stream, m->op_seq);
      CU(cudaGetLastError());
      return MHD_OK;
    }
    {
      const ncclDataType_t dt = sizeof(T) == 8 ? ncclFloat64 : ncclFloat32;
      PhaseTimer t(m, m->comm_stream, MHD_PHASE_EXCHANGE, seg_bytes(m->pack_list, sizeof(T)));
      NC(ncclGroupStart());
      for (auto& p : m->peers) {
        NC(ncclSend(m->send_buf<T>() + p.send_cell0 * NF, (size_t)p.send_cells * NF, dt, p.peer, m->comm, m->comm_stream));
        NC(ncclRecv(m->recv_buf<T>() + p.recv_cell0 * NF, (size_t)p.recv_cells * NF, dt, p.peer, m->comm, m->comm_stream));
      }
      NC(ncclGroupEnd());
    }
  } else {
    if (!m->group) return MHD_OK;
    const unsigned long long s = m->op_seq;
    xr_wait(m, m->comm_stream, s);
    {
      PhaseTimer t(m, m->comm_stream, MHD_PHASE_EXCHANGE, seg_bytes(m->pack_list, sizeof(T)));
      for (auto& p : m->peers) {
        const mhd_mesh* n = m->group->m[p.peer];
        for (auto& q : n->peers)
          if (q.peer == m->info.rank) {
            if (q.send_cells != p.recv_cells) return fail(MHD_EINVAL, "group: peer buffer sizes disagree");
            CU(cudaMemcpyAsync(m->recv_buf<T>() + p.recv_cell0 * NF, n->send_buf<T>() + q.send_cell0 * NF,
                               (size_t)p.recv_cells * NF * sizeof(T), cudaMemcpyDefault, m->comm_stream));
          }
      }
    }
    xr_done(m, m->comm_stream, s);
  }
  if (ph == (m->group ? 1 : 0)) {
    PhaseTimer t(m, m->comm_stream, MHD_PHASE_UNPACK, seg_bytes(m->unpack_list, sizeof(T)));
    launch_segments<T>(m->comm_stream, F, m->g, m->unpack_list, SEG_UNPACK, m->recv_buf<T>());
    m->launches++;
  }
  CU(cudaGetLastError());
  return MHD_OK;
}

// Substep with the packed exchange (the paper's scheme): the exchange on the side
// stream, then the boundary slabs there; the inner segment concurrently on the compute stream.
template <typename T>
mhd_status op_packed_substep(mhd_mesh* m, int ph, int k, double dt, T* rhs_out) {
  if (m->peers.empty()) return fail(MHD_EINVAL, "distributed mesh without peers");
  if (ph == 0) {
    poison_out<T>(m, rhs_out);
    return xchg_packed<T>(m, 0);
  }
  mhd_status st = xchg_packed<T>(m, 1);
  if (st != MHD_OK) return st;
  const bool xw = m->P[0] == 1 && m->x_fits();
  Region inner;
  std::vector<Region> outer;
  int thick[3];
  slab_thickness<T>(m, thick);
  split_regions(m, inner, outer, thick);
  m->g.xwrap = !rhs_out && xw ? 1 : 0;
  for (auto& r : outer) update_region<T>(m, r, k, dt, rhs_out, m->comm_stream);
  CU(cudaEventRecord(m->ev_halo, m->comm_stream));
  update_region<T>(m, inner, k, dt, rhs_out);
  CU(cudaStreamWaitEvent(m->stream, m->ev_halo, 0));
  m->g.xwrap = 0;
  if (!rhs_out) {
    m->self_valid = !m->self_list.n || (xw && !m->self_list_y.n);
    m->x_valid = xw;
  }
  CU(cudaGetLastError());
  return MHD_OK;
}

// One rank: one update launch over the whole grid (z halo by the TMA plane wrap, x faces of the
// new state by its epilogue, y rows copied before it).  (Overlapping a self-copy with an inner
// segment and updating the boundary slabs on the side stream was measured slower, 11.4 vs 12.4
// Gcell/s at 256^3.)
template <typename T>
mhd_status substep_local(mhd_mesh* m, int k, double dt, T* rhs_out) {
  const Region full = {{0, 0, 0}, {m->g.nx, m->g.ny, m->g.nz}};
  // z unsplit and the z-marching kernel on the whole grid: planes beyond the z faces are fetched
  // from their periodic image by the TMA coordinates (the z halo is never materialised); the x
  // faces are written by the previous update's epilogue, so only the y rows are copied
  const bool zm = m->variant != 1 && m->tmaps_ok && zmarch_ok<T>(m, full);
  const bool zw = !m->self_valid && zm;
  const bool xw = zw && m->x_valid;
  poison_out<T>(m, rhs_out);
  if (!m->self_valid && m->self_list.n) {
    const SegList& L = xw ? m->self_list_y : (zw ? m->self_list_xy : m->self_list);
    PhaseTimer t(m, m->stream, MHD_PHASE_SELF, seg_bytes(L, sizeof(T)));
    launch_segments<T>(m->stream, m->fields<T>(m->cur), m->g, L, SEG_SELF, nullptr);
    m->launches++;
  }
  m->self_valid = !zw;  // the z halo of the current state stays stale with the TMA wrap
  const bool use_x = !rhs_out && zw && m->x_fits();
  m->g.zwrap = zw ? 1 : 0;
  m->g.xwrap = use_x ? 1 : 0;
  m->persist = m->persist_env == 1;
  update_region<T>(m, full, k, dt, rhs_out);
  m->persist = false;
  m->g.zwrap = 0;
  m->g.xwrap = 0;
  if (!rhs_out) {
    m->self_valid = false;
    m->x_valid = use_x;
  }
  CU(cudaGetLastError());
  return MHD_OK;
}

// Runs an operation of `nph` phases over the meshes of one process: phase p of every mesh before
// phase p + 1 of any (a single mesh: its phases back to back).  Each mesh's device is made current
// while its work is enqueued; the caller's current device is restored.
template <class F>
mhd_status run_phases(mhd_mesh* const* ms, int n, int nph, F&& f) {
  int dev0 = -1;
  if (n > 1) CU(cudaGetDevice(&dev0));
  mhd_status st = MHD_OK;
  for (int ph = 0; ph < nph && st == MHD_OK; ++ph)
    for (int i = 0; i < n && st == MHD_OK; ++i) {
      if (n > 1) CU(cudaSetDevice(ms[i]->device));
      st = f(ms[i], i, ph);
    }
  if (dev0 >= 0) CU(cudaSetDevice(dev0));
  return st;
}

// One substep of every mesh of `ms` (one process-mode mesh, or every rank of a group).
template <typename T>
mhd_status substep_all(mhd_mesh* const* ms, int n, int k, double dt, T* const* rhs) {
  mhd_mesh* m0 = ms[0];
  if (!m0->distributed()) return substep_local<T>(m0, k, dt, rhs ? rhs[0] : nullptr);
  auto R = [&](int i) { return rhs ? rhs[i] : nullptr; };
  if (m0->exchange == 1) {
    if (!m0->halo_valid) {
      mhd_status st = run_phases(ms, n, 2, [&](mhd_mesh* m, int, int ph) { return op_p2p_halo_copy<T>(m, ph); });
      if (st != MHD_OK) return st;
    }
    return run_phases(ms, n, 2, [&](mhd_mesh* m, int i, int ph) { return op_p2p_substep<T>(m, ph, k, dt, R(i)); });
  }
  return run_phases(ms, n, 2, [&](mhd_mesh* m, int i, int ph) { return op_packed_substep<T>(m, ph, k, dt, R(i)); });
}

// Fill the halo of the current state of every mesh of `ms`.
template <typename T>
mhd_status halo_exchange_all(mhd_mesh* const* ms, int n) {
  mhd_mesh* m0 = ms[0];
  if (!m0->distributed()) {
    ensure_self<T>(m0);
    CU(cudaGetLastError());
    return MHD_OK;
  }
  if (m0->exchange == 1)
    return run_phases(ms, n, 3, [&](mhd_mesh* m, int, int ph) -> mhd_status {
      if (ph < 2) return op_p2p_halo_copy<T>(m, ph);
      xr_wait_done(m, m->stream, m->seq);  // the neighbours' copies into this halo have landed
      CU(cudaGetLastError());
      return MHD_OK;
    });
  return run_phases(ms, n, 2, [&](mhd_mesh* m, int, int ph) -> mhd_status {
    if (m->peers.empty()) return ph == 0 ? (ensure_self<T>(m), MHD_OK) : MHD_OK;
    mhd_status st = xchg_packed<T>(m, ph);
    if (st != MHD_OK || ph == 0) return st;
    CU(cudaEventRecord(m->ev_halo, m->comm_stream));
    CU(cudaStreamWaitEvent(m->stream, m->ev_halo, 0));
    return MHD_OK;
  });
}

// Peer-memory exchange, process mode: before the host reuses or releases memory that neighbours
// may still be storing into, wait for their last operation to land.
void settle_remote(mhd_mesh* m) {
  if (m->exchange == 1 && m->distributed() && m->seq > 0) xr_wait_done(m, m->stream, m->seq);
}

// Spin waits that timed out (process-mode peer-memory exchange) leave the sequence number in the
// error word; a blocking call reports it.
mhd_status check_spin(mhd_mesh* m) {
  if (!(m->exchange == 1 && m->distributed() && !m->group)) return MHD_OK;
  unsigned long long e = 0;
  CU(cudaMemcpy(&e, m->err_word(), sizeof(e), cudaMemcpyDeviceToHost));
  if (e) return fail(MHD_ECUDA, "peer-memory exchange: a neighbour did not arrive at operation " + std::to_string(e) +
                                    " within B2MHD_SPIN_TIMEOUT_S (ranks must run the same substeps in lockstep)");
  return MHD_OK;
}

}  // namespace

namespace {
template <typename TM>
mhd_status load_impl(mhd_mesh* m, int field, const void* src, int src_dtype, int on_device) {
  TM* origin = m->fields<TM>(m->cur).f[field];
  const size_t es = (size_t)src_dtype;
  const size_t ncell = (size_t)m->g.nx * m->g.ny * m->g.nz;
  settle_remote(m);
  if (m->debug & MHD_DEBUG_POISON_HALO) {
    Fields<TM> one = m->fields<TM>(m->cur);
    for (int q = 0; q < NF; ++q) one.f[q] = one.f[field];
    launch_poison_halo<TM>(m->stream, one, m->g, m->info.radius);
    m->launches++;
  }
  if (src_dtype == (int)sizeof(TM)) {
    cudaMemcpy3DParms p;
    memset(&p, 0, sizeof(p));
    p.srcPtr = make_cudaPitchedPtr(const_cast<void*>(src), (size_t)m->g.nx * es, (size_t)m->g.nx, (size_t)m->g.ny);
    p.dstPtr = make_cudaPitchedPtr(origin, (size_t)m->g.sy * es, (size_t)m->g.sy, (size_t)(m->g.ny + 2 * m->info.radius));
    p.extent = make_cudaExtent((size_t)m->g.nx * es, (size_t)m->g.ny, (size_t)m->g.nz);
    p.kind = on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
    CU(cudaMemcpy3DAsync(&p, m->stream));
    return MHD_OK;
  }
  const void* dsrc = src;
  void* tmp = nullptr;
  if (!on_device) {
    CU(cudaMallocAsync(&tmp, ncell * es, m->stream));
    CU(cudaMemcpyAsync(tmp, src, ncell * es, cudaMemcpyHostToDevice, m->stream));
    dsrc = tmp;
  }
  if (src_dtype == MHD_F32)
    launch_copy_in<float, TM>(m->stream, static_cast<const float*>(dsrc), origin, m->g);
  else
    launch_copy_in<double, TM>(m->stream, static_cast<const double*>(dsrc), origin, m->g);
  m->launches++;
  if (tmp) CU(cudaFreeAsync(tmp, m->stream));
  return MHD_OK;
}

template <typename TM>
mhd_status store_impl(mhd_mesh* m, int field, void* dst, int dst_dtype, int on_device) {
  const TM* origin = m->fields<TM>(m->cur).f[field];
  const size_t es = (size_t)dst_dtype;
  const size_t ncell = (size_t)m->g.nx * m->g.ny * m->g.nz;
  if (dst_dtype == (int)sizeof(TM)) {
    cudaMemcpy3DParms p;
    memset(&p, 0, sizeof(p));
    p.srcPtr = make_cudaPitchedPtr(const_cast<TM*>(origin), (size_t)m->g.sy * es, (size_t)m->g.sy,
                                   (size_t)(m->g.ny + 2 * m->info.radius));
    p.dstPtr = make_cudaPitchedPtr(dst, (size_t)m->g.nx * es, (size_t)m->g.nx, (size_t)m->g.ny);
    p.extent = make_cudaExtent((size_t)m->g.nx * es, (size_t)m->g.ny, (size_t)m->g.nz);
    p.kind = on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost;
    CU(cudaMemcpy3DAsync(&p, m->stream));
  } else {
    void* tmp = nullptr;
    void* ddst = dst;
    if (!on_device) {
      CU(cudaMallocAsync(&tmp, ncell * es, m->stream));
      ddst = tmp;
    }
    if (dst_dtype == MHD_F32)
      launch_copy_out<TM, float>(m->stream, origin, static_cast<float*>(ddst), m->g);
    else
      launch_copy_out<TM, double>(m->stream, origin, static_cast<double*>(ddst), m->g);
    m->launches++;
    if (tmp) {
      CU(cudaMemcpyAsync(dst, tmp, ncell * es, cudaMemcpyDeviceToHost, m->stream));
      CU(cudaFreeAsync(tmp, m->stream));
    }
  }
  if (!on_device) {
    CU(cudaStreamSynchronize(m->stream));
    return check_spin(m);
  }
  return MHD_OK;
}

// Local partial reduction of one field of the current state into v[kReduceVals] on the host
// (min, max, sum, sum of squares, sum of exp; slots 3/4 only when asked).
mhd_status reduce_local(mhd_mesh* m, int field, int op, bool finish_on_host) {
  double* sc = m->red_scratch();
  const int want = op == MHD_RMS ? 3 : (op == MHD_SUM_EXP ? 4 : 0);
  if (m->info.dtype == MHD_F64)
    launch_reduce<double>(m->stream, m->fields<double>(m->cur).f[field], m->g, sc, kReduceBlocks, want);
  else
    launch_reduce<float>(m->stream, m->fields<float>(m->cur).f[field], m->g, sc, kReduceBlocks, want);
  m->launches += 2;
  if (finish_on_host) CU(cudaMemcpyAsync(m->h_red, sc, kReduceVals * sizeof(double), cudaMemcpyDeviceToHost, m->stream));
  CU(cudaGetLastError());
  return MHD_OK;
}

mhd_status reduce_finish(const double* v, const mhd_mesh_info& info, int op, double* out) {
  const double ncell = (double)info.n[0] * (double)info.n[1] * (double)info.n[2];
  double r = 0;
  switch (op) {
    case MHD_MIN: r = v[0]; break;
    case MHD_MAX: r = v[1]; break;
    case MHD_SUM: r = v[2]; break;
    case MHD_RMS: r = std::sqrt(v[3] / ncell); break;
    case MHD_SUM_EXP: r = v[4]; break;
  }
  *out = r;
  if (!std::isfinite(v[0]) || !std::isfinite(v[1]) || !std::isfinite(v[2]) || !std::isfinite(r))
    return fail(MHD_ENONFINITE, "field holds a NaN or Inf (or the statistic overflows)");
  return MHD_OK;
}

mhd_status open_peers(mhd_mesh* m) {
  m->remote_list = make_remote_list(*m);
  memset(&m->peer_arrive, 0, sizeof(FlagSet));
  memset(&m->peer_done, 0, sizeof(FlagSet));
  memset(&m->my_arrive, 0, sizeof(FlagSet));
  memset(&m->my_done, 0, sizeof(FlagSet));
  const int nr = m->info.nranks;
  for (auto& p : m->peers) {
    if (!m->peer_ws[p.peer]) return fail(MHD_EINVAL, "neighbour workspace not mapped");
    unsigned long long* peer_flags = reinterpret_cast<unsigned long long*>(m->peer_ws[p.peer] + m->L.flags_off);
    unsigned long long* my_flags = m->flags();
    m->peer_arrive.ptr[m->peer_arrive.n++] = peer_flags + m->info.rank;
    m->peer_done.ptr[m->peer_done.n++] = peer_flags + nr + m->info.rank;
    m->my_arrive.ptr[m->my_arrive.n++] = my_flags + p.peer;
    m->my_done.ptr[m->my_done.n++] = my_flags + nr + p.peer;
  }
  m->halo_valid = false;
  m->self_valid = false;
  m->x_valid = false;
  return MHD_OK;
}

bool in_group(const mhd_mesh* m) { return m->group != nullptr; }
}  // namespace

// =================================================================================================
extern "C" {

const char* mhd_status_str(mhd_status s) {
  switch (s) {
    case MHD_OK: return "ok";
    case MHD_EINVAL: return "invalid argument";
    case MHD_EDECOMP: return "invalid decomposition";
    case MHD_ESMALL: return "subdomain too small";
    case MHD_EUNSUPPORTED: return "unsupported";
    case MHD_ECUDA: return "CUDA error";
    case MHD_ENCCL: return "NCCL error";
    case MHD_ENOMEM: return "workspace too small";
    case MHD_ENONFINITE: return "non-finite value";
    case MHD_ESTATE: return "substep out of order";
  }
  return "unknown status";
}

const char* mhd_last_error(void) { return g_err.c_str(); }
int32_t mhd_abi_version(void) { return MHD_ABI_VERSION; }

mhd_status mhd_decompose(const mhd_mesh_info* info, int32_t rank, int32_t P[3], int32_t coord[3],
                         int64_t local_n[3]) {
  mhd_mesh_info tmp;
  if (!info) return fail(MHD_EINVAL, "info is null");
  tmp = *info;
  tmp.rank = rank;
  mhd_status st = check_info(&tmp);
  if (st != MHD_OK) return st;
  int p[3], c[3];
  partition_xyz(info->nranks, p);
  coord_xyz(rank, c);
  for (int a = 0; a < 3; ++a) {
    if (P) P[a] = p[a];
    if (coord) coord[a] = c[a];
    if (local_n) local_n[a] = info->n[a] / p[a];
  }
  return MHD_OK;
}

mhd_status mhd_segment_table(const mhd_mesh_info* info, int32_t rank, mhd_segment* out, int32_t max_segments,
                             int32_t* count) {
  mhd_mesh_info tmp;
  if (!info || !count) return fail(MHD_EINVAL, "null argument");
  tmp = *info;
  tmp.rank = rank;
  mhd_status st = check_info(&tmp);
  if (st != MHD_OK) return st;
  auto segs = build_segments(&tmp, rank);
  *count = (int32_t)segs.size();
  for (int i = 0; i < (int)segs.size() && i < max_segments; ++i) out[i] = segs[i].s;
  return MHD_OK;
}

mhd_status mhd_workspace_bytes(const mhd_mesh_info* info, size_t* bytes) {
  mhd_status st = check_info(info);
  if (st != MHD_OK) return st;
  if (!bytes) return fail(MHD_EINVAL, "bytes is null");
  auto segs = build_segments(info, info->rank);
  *bytes = make_layout(info, segs).total;
  return MHD_OK;
}

mhd_status mhd_mesh_create(const mhd_mesh_info* info, void* dev_workspace, size_t bytes, void* cuda_stream,
                           mhd_mesh** out) {
  mhd_status st = check_info(info);
  if (st != MHD_OK) return st;
  if (!dev_workspace || !out) return fail(MHD_EINVAL, "null workspace or out");
  mhd_mesh* m = new mhd_mesh();
  m->info = *info;
  if (const char* w = getenv("B2MHD_XWRAP")) m->xwrap = atoi(w) != 0;
  if (const char* w = getenv("B2MHD_PERSIST")) m->persist_env = atoi(w) != 0;
  if (const char* w = getenv("B2MHD_ZSPLIT")) m->split_env = atoi(w) != 0;
  if (const char* w = getenv("B2MHD_FINE_ARRIVAL")) m->fine_env = atoi(w) != 0;
  m->fine_arrival = m->fine_env >= 0 ? m->fine_env != 0 : info->dtype == MHD_F64;
  if (const char* w = getenv("B2MHD_SLAB_ZCHUNK")) m->slab_zchunk = atoi(w);
  if (const char* w = getenv("B2MHD_ZCHUNK")) m->zchunk_env = atoi(w);
  if (const char* w = getenv("B2MHD_SLAB")) sscanf(w, "%d,%d,%d", &m->slab_env[0], &m->slab_env[1], &m->slab_env[2]);
  if (const char* w = getenv("B2MHD_POISON")) m->debug |= atoi(w) ? MHD_DEBUG_POISON_HALO : 0;
  if (const char* w = getenv("B2MHD_SPIN_TIMEOUT_S")) m->spin_timeout_ns = (unsigned long long)(atof(w) * 1e9);
  partition_xyz(info->nranks, m->P);
  coord_xyz(info->rank, m->coord);
  m->segs = build_segments(info, info->rank);
  m->L = make_layout(info, m->segs);
  if (bytes < m->L.total) {
    delete m;
    return fail(MHD_ENOMEM, "workspace smaller than mhd_workspace_bytes");
  }
  m->g.nx = (int)m->L.n[0];
  m->g.ny = (int)m->L.n[1];
  m->g.nz = (int)m->L.n[2];
  m->g.sy = m->L.sy;
  m->g.sz = m->L.sz;
  m->g.zwrap = 0;
  m->g.xwrap = 0;
  m->ws = static_cast<char*>(dev_workspace);
  m->stream = static_cast<cudaStream_t>(cuda_stream);
  cudaGetDevice(&m->device);
  // peers in rank order, each with a contiguous slice of the send and recv buffers
  std::vector<int64_t> scount(info->nranks, 0), rcount(info->nranks, 0);
  for (auto& si : m->segs)
    if (!si.self) {
      const int64_t cells = (int64_t)si.s.extent[0] * si.s.extent[1] * si.s.extent[2];
      scount[si.s.send_peer] += cells;
      rcount[si.s.recv_peer] += cells;
    }
  int64_t s0 = 0, r0 = 0;
  for (int p = 0; p < info->nranks; ++p) {
    if (scount[p] == 0 && rcount[p] == 0) continue;
    m->peers.push_back(PeerXfer{p, s0, scount[p], r0, rcount[p]});
    s0 += scount[p];
    r0 += rcount[p];
  }
  m->self_list = make_list(*m, true, false);
  m->self_list_xy = make_list(*m, true, false, true);
  m->self_list_y = make_list(*m, true, false, true, true);
  m->pack_list = make_list(*m, false, true);
  m->unpack_list = make_list(*m, false, false);
  cudaError_t e = cudaMemsetAsync(m->ws, 0, m->L.total, m->stream);
  if (e == cudaSuccess) {  // side stream: halo exchange and the boundary slabs (N > 1)
    int lo, hi;
    cudaDeviceGetStreamPriorityRange(&lo, &hi);
    e = cudaStreamCreateWithPriority(&m->comm_stream, cudaStreamNonBlocking, hi);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&m->ev_ready, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&m->ev_halo, cudaEventDisableTiming);
  }
  if (e == cudaSuccess) e = cudaMallocHost(&m->h_red, kReduceVals * sizeof(double));
  if (e != cudaSuccess) {
    delete m;
    return fail(MHD_ECUDA, std::string("mesh create: ") + cudaGetErrorString(e));
  }
  st = encode_tmaps(m);
  if (st != MHD_OK) {
    delete m;
    return st;
  }
  *out = m;
  return MHD_OK;
}

mhd_status mhd_nccl_unique_id(void* out128) {
  if (!out128) return fail(MHD_EINVAL, "null out");
  ncclUniqueId id;
  NC(ncclGetUniqueId(&id));
  memcpy(out128, &id, sizeof(id));
  return MHD_OK;
}

mhd_status mhd_comm_init(mhd_mesh* m, const void* nccl_unique_id) {
  if (!m || !nccl_unique_id) return fail(MHD_EINVAL, "null argument");
  if (m->info.nranks == 1) return MHD_OK;
  if (in_group(m)) return fail(MHD_EINVAL, "mesh belongs to a group (no NCCL communicator)");
  ncclUniqueId id;
  memcpy(&id, nccl_unique_id, sizeof(id));
  NC(ncclCommInitRank(&m->comm, m->info.nranks, id, m->info.rank));
  return MHD_OK;
}

mhd_status mhd_mesh_destroy(mhd_mesh* m) {
  if (!m) return MHD_OK;
  if (m->group) return fail(MHD_EINVAL, "destroy the group (mhd_group_destroy) first");
  // peer memory: the neighbours' stores of their last operation into this workspace have landed
  // before the caller may release it (the caller also barriers across ranks: mesh.py)
  settle_remote(m);
  cudaStreamSynchronize(m->stream);
  if (m->comm) ncclCommDestroy(m->comm);
  for (void* b : m->ipc_bases) cudaIpcCloseMemHandle(b);
  if (m->comm_stream) cudaStreamDestroy(m->comm_stream);
  if (m->ev_ready) cudaEventDestroy(m->ev_ready);
  if (m->ev_halo) cudaEventDestroy(m->ev_halo);
  for (int i = 0; i < kRing; ++i) {
    if (m->ev_arrive[i]) cudaEventDestroy(m->ev_arrive[i]);
    if (m->ev_done[i]) cudaEventDestroy(m->ev_done[i]);
  }
  if (m->h_red) cudaFreeHost(m->h_red);
  for (auto& a : m->aio) {
    if (a.st) {
      cudaStreamSynchronize(a.st);
      cudaStreamDestroy(a.st);
    }
    for (int q = 0; q < NF; ++q) {
      if (a.ev_dev[q]) cudaEventDestroy(a.ev_dev[q]);
      if (a.ev_host[q]) cudaEventDestroy(a.ev_host[q]);
    }
    if (a.stage) cudaFree(a.stage);
  }
  for (auto& v : m->recs)
    for (auto& r : v) {
      cudaEventDestroy(r.a);
      cudaEventDestroy(r.b);
    }
  for (auto e : m->pool) cudaEventDestroy(e);
  delete m;
  return MHD_OK;
}

mhd_status mhd_load(mhd_mesh* m, int32_t field, const void* src, int32_t src_dtype, int32_t on_device) {
  if (!m || !src || field < 0 || field >= NF) return fail(MHD_EINVAL, "bad load argument");
  if (src_dtype != MHD_F32 && src_dtype != MHD_F64) return fail(MHD_EUNSUPPORTED, "src dtype");
  m->next_k = 0;
  m->halo_valid = false;
  m->self_valid = false;
  m->x_valid = false;
  return m->info.dtype == MHD_F64 ? load_impl<double>(m, field, src, src_dtype, on_device)
                                  : load_impl<float>(m, field, src, src_dtype, on_device);
}

mhd_status mhd_store(mhd_mesh* m, int32_t field, void* dst, int32_t dst_dtype, int32_t on_device) {
  if (!m || !dst || field < 0 || field >= NF) return fail(MHD_EINVAL, "bad store argument");
  if (dst_dtype != MHD_F32 && dst_dtype != MHD_F64) return fail(MHD_EUNSUPPORTED, "dst dtype");
  return m->info.dtype == MHD_F64 ? store_impl<double>(m, field, dst, dst_dtype, on_device)
                                  : store_impl<float>(m, field, dst, dst_dtype, on_device);
}

// Lazily creates the lane's stream and events and (re)allocates its staging for dtype `es`.
static mhd_status lane_ready(mhd_mesh* m, mhd_mesh::AsyncLane& a, int es) {
  if (!a.st) {
    CU(cudaStreamCreateWithFlags(&a.st, cudaStreamNonBlocking));
    for (int q = 0; q < NF; ++q) {
      CU(cudaEventCreateWithFlags(&a.ev_dev[q], cudaEventDisableTiming));
      CU(cudaEventCreateWithFlags(&a.ev_host[q], cudaEventDisableTiming));
    }
  }
  if (a.es != es) {
    CU(cudaStreamSynchronize(a.st));
    CU(cudaStreamSynchronize(m->stream));
    if (a.stage) CU(cudaFree(a.stage));
    a.stage = nullptr;
    CU(cudaMalloc(&a.stage, (size_t)m->g.nx * m->g.ny * m->g.nz * (size_t)es * NF));
    a.es = es;
    for (int q = 0; q < NF; ++q) {
      CU(cudaEventRecord(a.ev_dev[q], m->stream));
      CU(cudaEventRecord(a.ev_host[q], a.st));
    }
  }
  return MHD_OK;
}

mhd_status mhd_store_async(mhd_mesh* m, int32_t field, void* dst, int32_t dst_dtype) {
  if (!m || !dst || field < 0 || field >= NF) return fail(MHD_EINVAL, "bad store argument");
  if (dst_dtype != MHD_F32 && dst_dtype != MHD_F64) return fail(MHD_EUNSUPPORTED, "dst dtype");
  auto& a = m->aio[0];
  mhd_status s = lane_ready(m, a, dst_dtype);
  if (s != MHD_OK) return s;
  const size_t bytes = (size_t)m->g.nx * m->g.ny * m->g.nz * (size_t)dst_dtype;
  char* st = a.stage + bytes * (size_t)field;
  CU(cudaStreamWaitEvent(m->stream, a.ev_host[field], 0));  // the previous transfer of this slot is done
  s = m->info.dtype == MHD_F64 ? store_impl<double>(m, field, st, dst_dtype, 1)
                               : store_impl<float>(m, field, st, dst_dtype, 1);
  if (s != MHD_OK) return s;
  CU(cudaEventRecord(a.ev_dev[field], m->stream));
  CU(cudaStreamWaitEvent(a.st, a.ev_dev[field], 0));
  CU(cudaMemcpyAsync(dst, st, bytes, cudaMemcpyDeviceToHost, a.st));
  CU(cudaEventRecord(a.ev_host[field], a.st));
  return MHD_OK;
}

mhd_status mhd_load_async(mhd_mesh* m, int32_t field, const void* src, int32_t src_dtype) {
  if (!m || !src || field < 0 || field >= NF) return fail(MHD_EINVAL, "bad load argument");
  if (src_dtype != MHD_F32 && src_dtype != MHD_F64) return fail(MHD_EUNSUPPORTED, "src dtype");
  auto& a = m->aio[1];
  mhd_status s = lane_ready(m, a, src_dtype);
  if (s != MHD_OK) return s;
  const size_t bytes = (size_t)m->g.nx * m->g.ny * m->g.nz * (size_t)src_dtype;
  char* st = a.stage + bytes * (size_t)field;
  CU(cudaStreamWaitEvent(a.st, a.ev_dev[field], 0));  // the previous scatter out of this slot is done
  CU(cudaMemcpyAsync(st, src, bytes, cudaMemcpyHostToDevice, a.st));
  CU(cudaEventRecord(a.ev_host[field], a.st));
  CU(cudaStreamWaitEvent(m->stream, a.ev_host[field], 0));
  m->next_k = 0;
  m->halo_valid = false;
  m->self_valid = false;
  m->x_valid = false;
  s = m->info.dtype == MHD_F64 ? load_impl<double>(m, field, st, src_dtype, 1)
                               : load_impl<float>(m, field, st, src_dtype, 1);
  if (s != MHD_OK) return s;
  CU(cudaEventRecord(a.ev_dev[field], m->stream));
  return MHD_OK;
}

mhd_status mhd_store_grid(mhd_mesh* m, int32_t field, void* dst, int32_t on_device) {
  if (!m || !dst || field < 0 || field >= NF) return fail(MHD_EINVAL, "bad store_grid argument");
  const size_t es = (size_t)m->info.dtype;
  const char* base = m->ws + m->L.state_off[m->cur] + (size_t)field * m->L.field_bytes;
  const int rad = m->info.radius;
  const char* first = base + (size_t)(m->L.xo - rad) * es;  // (x, y, z) = (-r, -r, -r)
  const size_t mx = (size_t)m->g.nx + 2 * rad, my = (size_t)m->g.ny + 2 * rad;
  const size_t mz = (size_t)m->g.nz + 2 * rad;
  settle_remote(m);  // the neighbours' stores into this halo have landed (peer-memory exchange)
  CU(cudaMemcpy2DAsync(dst, mx * es, first, (size_t)m->g.sy * es, mx * es, my * mz,
                       on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, m->stream));
  if (!on_device) {
    CU(cudaStreamSynchronize(m->stream));
    return check_spin(m);
  }
  return MHD_OK;
}

mhd_status mhd_halo_exchange(mhd_mesh* m) {
  if (!m) return fail(MHD_EINVAL, "null mesh");
  if (in_group(m)) return fail(MHD_EINVAL, "mesh belongs to a group: use mhd_group_halo_exchange");
  return m->info.dtype == MHD_F64 ? halo_exchange_all<double>(&m, 1) : halo_exchange_all<float>(&m, 1);
}

mhd_status mhd_integrate_substep(mhd_mesh* m, int32_t k, double dt) {
  if (!m) return fail(MHD_EINVAL, "null mesh");
  if (in_group(m)) return fail(MHD_EINVAL, "mesh belongs to a group: use mhd_group_integrate_substep");
  if (k < 0 || k > 2) return fail(MHD_EINVAL, "k must be 0, 1 or 2");
  if (k != m->next_k) return fail(MHD_ESTATE, "substeps must run in the order 0, 1, 2");
  mhd_status st = m->info.dtype == MHD_F64 ? substep_all<double>(&m, 1, k, dt, nullptr)
                                           : substep_all<float>(&m, 1, k, dt, nullptr);
  if (st != MHD_OK) return st;
  m->cur = 1 - m->cur;
  m->next_k = (k + 1) % 3;
  return MHD_OK;
}

mhd_status mhd_integrate_step(mhd_mesh* m, double dt) {
  for (int k = 0; k < 3; ++k) {
    mhd_status st = mhd_integrate_substep(m, k, dt);
    if (st != MHD_OK) return st;
  }
  return MHD_OK;
}

mhd_status mhd_debug_rhs(mhd_mesh* m, void* dev_dst) {
  if (!m || !dev_dst) return fail(MHD_EINVAL, "null argument");
  if (in_group(m)) return fail(MHD_EINVAL, "mesh belongs to a group: use mhd_group_debug_rhs");
  if (m->info.dtype == MHD_F64) {
    double* d = static_cast<double*>(dev_dst);
    return substep_all<double>(&m, 1, 0, 0.0, &d);
  }
  float* d = static_cast<float*>(dev_dst);
  return substep_all<float>(&m, 1, 0, 0.0, &d);
}

mhd_status mhd_reduce(mhd_mesh* m, int32_t field, int32_t op, double* out) {
  if (!m || !out || field < 0 || field >= NF || op < 0 || op > MHD_SUM_EXP) return fail(MHD_EINVAL, "bad reduce argument");
  if (in_group(m)) return fail(MHD_EINVAL, "mesh belongs to a group: use mhd_group_reduce");
  mhd_status st = reduce_local(m, field, op, false);
  if (st != MHD_OK) return st;
  double* sc = m->red_scratch();
  if (m->distributed()) {
    if (!m->comm) return fail(MHD_ENCCL, "mhd_comm_init was not called");
    NC(ncclGroupStart());
    NC(ncclAllReduce(sc + 0, sc + 0, 1, ncclFloat64, ncclMin, m->comm, m->stream));
    NC(ncclAllReduce(sc + 1, sc + 1, 1, ncclFloat64, ncclMax, m->comm, m->stream));
    NC(ncclAllReduce(sc + 2, sc + 2, 3, ncclFloat64, ncclSum, m->comm, m->stream));
    NC(ncclGroupEnd());
  }
  CU(cudaMemcpyAsync(m->h_red, sc, kReduceVals * sizeof(double), cudaMemcpyDeviceToHost, m->stream));
  CU(cudaStreamSynchronize(m->stream));
  st = check_spin(m);
  if (st != MHD_OK) return st;
  return reduce_finish(m->h_red, m->info, op, out);
}

mhd_status mhd_synchronize(mhd_mesh* m) {
  if (!m) return fail(MHD_EINVAL, "null mesh");
  CU(cudaStreamSynchronize(m->stream));
  if (m->comm_stream) CU(cudaStreamSynchronize(m->comm_stream));
  for (auto& a : m->aio)
    if (a.st) CU(cudaStreamSynchronize(a.st));
  CU(cudaGetLastError());
  return check_spin(m);
}

mhd_status mhd_set_kernel(mhd_mesh* m, int32_t variant) {
  if (!m || variant < 0 || variant > 3) return fail(MHD_EINVAL, "variant must be 0, 1, 2 or 3");
  if (variant >= 2) {
    Region full = {{0, 0, 0}, {m->g.nx, m->g.ny, m->g.nz}};
    const bool ok = m->tmaps_ok && (m->info.dtype == MHD_F64 ? zmarch_ok<double>(m, full) : zmarch_ok<float>(m, full));
    if (!ok) return fail(MHD_EUNSUPPORTED, "z-marching kernel does not support this geometry");
    if (variant == 3 && !(m->info.dtype == MHD_F64 &&
                          ((m->info.radius == 3 && zsplit_supported<double, 3>(m->g, full)) ||
                           (m->info.radius == 4 && zsplit_supported<double, 4>(m->g, full)))))
      return fail(MHD_EUNSUPPORTED, "the warp-specialised kernel is FP64, radius 3 or 4 only");
  }
  m->variant = variant;
  return MHD_OK;
}

mhd_status mhd_set_debug(mhd_mesh* m, int32_t flags) {
  if (!m || (flags & ~MHD_DEBUG_POISON_HALO)) return fail(MHD_EINVAL, "unknown debug flag");
  m->debug = flags;
  return MHD_OK;
}

mhd_status mhd_mesh_query(const mhd_mesh* m, int32_t P[3], int32_t coord[3], int64_t local_n[3], int32_t* next_k) {
  if (!m) return fail(MHD_EINVAL, "null mesh");
  for (int a = 0; a < 3; ++a) {
    if (P) P[a] = m->P[a];
    if (coord) coord[a] = m->coord[a];
    if (local_n) local_n[a] = m->L.n[a];
  }
  if (next_k) *next_k = m->next_k;
  return MHD_OK;
}

mhd_status mhd_p2p_export(mhd_mesh* m, void* out_blob) {
  if (!m || !out_blob) return fail(MHD_EINVAL, "null argument");
  static PFN_cuMemGetAddressRange_v3020 range = nullptr;
  if (!range) {
    cudaDriverEntryPointQueryResult q;
    void* fn = nullptr;
    CU(cudaGetDriverEntryPoint("cuMemGetAddressRange", &fn, cudaEnableDefault, &q));
    if (q != cudaDriverEntryPointSuccess || !fn) return fail(MHD_ECUDA, "cuMemGetAddressRange unavailable");
    range = reinterpret_cast<PFN_cuMemGetAddressRange_v3020>(fn);
  }
  CUdeviceptr base = 0;
  size_t size = 0;
  if (range(&base, &size, (CUdeviceptr)m->ws) != CUDA_SUCCESS) return fail(MHD_ECUDA, "cuMemGetAddressRange failed");
  cudaIpcMemHandle_t h;
  CU(cudaIpcGetMemHandle(&h, (void*)base));
  unsigned char* b = static_cast<unsigned char*>(out_blob);
  memset(b, 0, MHD_P2P_HANDLE_BYTES);
  memcpy(b, &h, sizeof(h));
  const uint64_t off = (uint64_t)((char*)m->ws - (char*)base);
  memcpy(b + 64, &off, 8);
  const int32_t rank = m->info.rank;
  memcpy(b + 72, &rank, 4);
  return MHD_OK;
}

mhd_status mhd_p2p_open(mhd_mesh* m, const void* blobs) {
  if (!m || !blobs) return fail(MHD_EINVAL, "null argument");
  if (m->info.nranks == 1) return MHD_OK;
  if (in_group(m)) return fail(MHD_EINVAL, "mesh belongs to a group");
  if (m->peers.size() > (size_t)kMaxPeers) return fail(MHD_EUNSUPPORTED, "more than 7 neighbours");
  CU(cudaStreamSynchronize(m->stream));  // the zeroed flags are in place before anyone signals
  m->peer_ws.assign(m->info.nranks, nullptr);
  const unsigned char* b = static_cast<const unsigned char*>(blobs);
  for (auto& p : m->peers) {
    const unsigned char* blob = b + (size_t)p.peer * MHD_P2P_HANDLE_BYTES;
    int32_t r;
    memcpy(&r, blob + 72, 4);
    if (r != p.peer) return fail(MHD_EINVAL, "handle blobs are not in rank order");
    cudaIpcMemHandle_t h;
    memcpy(&h, blob, sizeof(h));
    uint64_t off;
    memcpy(&off, blob + 64, 8);
    void* base = nullptr;
    CU(cudaIpcOpenMemHandle(&base, h, cudaIpcMemLazyEnablePeerAccess));
    m->ipc_bases.push_back(base);
    m->peer_ws[p.peer] = static_cast<char*>(base) + off;
  }
  mhd_status st = open_peers(m);
  if (st != MHD_OK) return st;
  m->exchange = 1;
  return MHD_OK;
}

mhd_status mhd_set_exchange(mhd_mesh* m, int32_t mode) {
  if (!m || mode < 0 || mode > 1) return fail(MHD_EINVAL, "mode must be 0 (packed / NCCL) or 1 (peer memory)");
  if (in_group(m)) return fail(MHD_EINVAL, "mesh belongs to a group: the group fixes the exchange");
  if (mode == 1 && m->info.nranks > 1 && m->peer_ws.empty()) return fail(MHD_EINVAL, "mhd_p2p_open first");
  if (mode == 0 && m->info.nranks > 1 && !m->comm) return fail(MHD_ENCCL, "mhd_comm_init first");
  settle_remote(m);
  m->exchange = m->info.nranks > 1 ? mode : 0;
  m->halo_valid = false;
  m->self_valid = false;
  m->x_valid = false;
  return MHD_OK;
}

// ---- several ranks in one process ------------------------------------------------------------------

mhd_status mhd_group_create(mhd_mesh* const* meshes, int32_t n, int32_t exchange, mhd_group** out) {
  if (!meshes || !out || n < 1 || exchange < 0 || exchange > 1) return fail(MHD_EINVAL, "bad group argument");
  for (int i = 0; i < n; ++i) {
    const mhd_mesh* m = meshes[i];
    if (!m) return fail(MHD_EINVAL, "null mesh");
    if (m->info.nranks != n || m->info.rank != i) return fail(MHD_EINVAL, "meshes must be ranks 0..n-1 of an n-rank mesh, in order");
    if (m->group || m->comm || !m->peer_ws.empty()) return fail(MHD_EINVAL, "mesh already has a communicator or group");
    for (int a = 0; a < 3; ++a)
      if (m->info.n[a] != meshes[0]->info.n[a]) return fail(MHD_EINVAL, "meshes of different grids");
    if (m->info.dtype != meshes[0]->info.dtype || m->info.radius != meshes[0]->info.radius ||
        m->info.exchange_corners != meshes[0]->info.exchange_corners)
      return fail(MHD_EINVAL, "meshes of different dtype, radius or corner setting");
    if (exchange == 1 && m->peers.size() > (size_t)kMaxPeers) return fail(MHD_EUNSUPPORTED, "more than 7 neighbours");
  }
  int dev0 = 0;
  CU(cudaGetDevice(&dev0));
  // peer access between the devices of neighbouring ranks (ranks on one device need none)
  for (int i = 0; i < n; ++i)
    for (auto& p : meshes[i]->peers) {
      const int a = meshes[i]->device, b = meshes[p.peer]->device;
      if (a == b) continue;
      int can = 0;
      CU(cudaDeviceCanAccessPeer(&can, a, b));
      if (!can) return fail(MHD_EUNSUPPORTED, "group: devices without peer access");
      CU(cudaSetDevice(a));
      cudaError_t e = cudaDeviceEnablePeerAccess(b, 0);
      if (e == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
      else if (e != cudaSuccess) return fail(MHD_ECUDA, std::string("cudaDeviceEnablePeerAccess: ") + cudaGetErrorString(e));
    }
  mhd_group* g = new mhd_group();
  g->exchange = exchange;
  for (int i = 0; i < n; ++i) {
    mhd_mesh* m = meshes[i];
    CU(cudaSetDevice(m->device));
    CU(cudaStreamSynchronize(m->stream));
    for (int j = 0; j < kRing; ++j) {
      if (!m->ev_arrive[j]) CU(cudaEventCreateWithFlags(&m->ev_arrive[j], cudaEventDisableTiming));
      if (!m->ev_done[j]) CU(cudaEventCreateWithFlags(&m->ev_done[j], cudaEventDisableTiming));
    }
    m->peer_ws.assign(n, nullptr);
    for (auto& p : m->peers) m->peer_ws[p.peer] = meshes[p.peer]->ws;
    g->m.push_back(m);
  }
  for (auto* m : g->m) {
    mhd_status st = open_peers(m);
    if (st != MHD_OK) {
      delete g;
      return st;
    }
    m->group = g;
    m->exchange = exchange;
    m->seq = 0;
  }
  CU(cudaSetDevice(dev0));
  *out = g;
  return MHD_OK;
}

mhd_status mhd_group_destroy(mhd_group* g) {
  if (!g) return MHD_OK;
  for (auto* m : g->m) {
    cudaSetDevice(m->device);
    cudaStreamSynchronize(m->stream);
    if (m->comm_stream) cudaStreamSynchronize(m->comm_stream);
  }
  for (auto* m : g->m) {
    m->group = nullptr;
    m->peer_ws.clear();
    m->exchange = 0;
  }
  delete g;
  return MHD_OK;
}

mhd_status mhd_group_halo_exchange(mhd_group* g) {
  if (!g) return fail(MHD_EINVAL, "null group");
  mhd_mesh* const* ms = g->m.data();
  const int n = (int)g->m.size();
  return ms[0]->info.dtype == MHD_F64 ? halo_exchange_all<double>(ms, n) : halo_exchange_all<float>(ms, n);
}

mhd_status mhd_group_integrate_substep(mhd_group* g, int32_t k, double dt) {
  if (!g) return fail(MHD_EINVAL, "null group");
  if (k < 0 || k > 2) return fail(MHD_EINVAL, "k must be 0, 1 or 2");
  for (auto* m : g->m)
    if (k != m->next_k) return fail(MHD_ESTATE, "substeps must run in the order 0, 1, 2 on every rank");
  mhd_mesh* const* ms = g->m.data();
  const int n = (int)g->m.size();
  mhd_status st = ms[0]->info.dtype == MHD_F64 ? substep_all<double>(ms, n, k, dt, nullptr)
                                               : substep_all<float>(ms, n, k, dt, nullptr);
  if (st != MHD_OK) return st;
  for (auto* m : g->m) {
    m->cur = 1 - m->cur;
    m->next_k = (k + 1) % 3;
  }
  return MHD_OK;
}

mhd_status mhd_group_integrate_step(mhd_group* g, double dt) {
  for (int k = 0; k < 3; ++k) {
    mhd_status st = mhd_group_integrate_substep(g, k, dt);
    if (st != MHD_OK) return st;
  }
  return MHD_OK;
}

mhd_status mhd_group_debug_rhs(mhd_group* g, void* const* dev_dst) {
  if (!g || !dev_dst) return fail(MHD_EINVAL, "null argument");
  mhd_mesh* const* ms = g->m.data();
  const int n = (int)g->m.size();
  if (ms[0]->info.dtype == MHD_F64)
    return substep_all<double>(ms, n, 0, 0.0, reinterpret_cast<double* const*>(dev_dst));
  return substep_all<float>(ms, n, 0, 0.0, reinterpret_cast<float* const*>(dev_dst));
}

mhd_status mhd_group_reduce(mhd_group* g, int32_t field, int32_t op, double* out) {
  if (!g || !out || field < 0 || field >= NF || op < 0 || op > MHD_SUM_EXP) return fail(MHD_EINVAL, "bad reduce argument");
  int dev0 = 0;
  CU(cudaGetDevice(&dev0));
  for (auto* m : g->m) {
    CU(cudaSetDevice(m->device));
    mhd_status st = reduce_local(m, field, op, true);
    if (st != MHD_OK) return st;
  }
  double v[kReduceVals] = {INFINITY, -INFINITY, 0.0, 0.0, 0.0};
  for (auto* m : g->m) {  // combined in rank order on the host
    CU(cudaSetDevice(m->device));
    CU(cudaStreamSynchronize(m->stream));
    const double* h = m->h_red;
    v[0] = std::fmin(v[0], h[0]);
    v[1] = std::fmax(v[1], h[1]);
    for (int j = 2; j < kReduceVals; ++j) v[j] += h[j];
    if (std::isnan(h[0]) || std::isnan(h[1])) v[2] = NAN;
  }
  CU(cudaSetDevice(dev0));
  return reduce_finish(v, g->m[0]->info, op, out);
}

mhd_status mhd_group_synchronize(mhd_group* g) {
  if (!g) return fail(MHD_EINVAL, "null group");
  int dev0 = 0;
  CU(cudaGetDevice(&dev0));
  for (auto* m : g->m) {
    CU(cudaSetDevice(m->device));
    mhd_status st = mhd_synchronize(m);
    if (st != MHD_OK) return st;
  }
  CU(cudaSetDevice(dev0));
  return MHD_OK;
}

mhd_status mhd_profile_enable(mhd_mesh* m, int32_t enable) {
  if (!m) return fail(MHD_EINVAL, "null mesh");
  CU(cudaStreamSynchronize(m->stream));
  if (m->comm_stream) CU(cudaStreamSynchronize(m->comm_stream));
  for (auto& v : m->recs) {
    for (auto& r : v) {
      m->pool.push_back(r.a);
      m->pool.push_back(r.b);
    }
    v.clear();
  }
  m->prof = enable != 0;
  return MHD_OK;
}

mhd_status mhd_profile_read(mhd_mesh* m, int32_t phase, int64_t* launches, double* ms, double* bytes) {
  if (!m || phase < 0 || phase >= MHD_NPHASES) return fail(MHD_EINVAL, "bad profile_read argument");
  CU(cudaStreamSynchronize(m->stream));
  if (m->comm_stream) CU(cudaStreamSynchronize(m->comm_stream));
  double tot = 0, by = 0;
  for (auto& r : m->recs[phase]) {
    float t = 0;
    CU(cudaEventElapsedTime(&t, r.a, r.b));
    tot += t;
    by += r.bytes;
  }
  if (launches) *launches = (int64_t)m->recs[phase].size();
  if (ms) *ms = tot;
  if (bytes) *bytes = by;
  return MHD_OK;
}

mhd_status mhd_launch_count(const mhd_mesh* m, int64_t* count) {
  if (!m || !count) return fail(MHD_EINVAL, "null argument");
  *count = m->launches;
  return MHD_OK;
}

}  // extern "C"
