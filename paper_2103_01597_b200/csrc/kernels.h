// Internal (non-ABI) declarations shared by the runtime (mesh.cpp) and the kernels.
#pragma once
#include <cuda.h>  // CUtensorMap (TMA descriptors; encoded through the runtime driver entry point)
#include <cuda_runtime.h>
#include <stdint.h>

#include <type_traits>

#include "mhd_math.cuh"
#include "remote.cuh"

namespace b2 {

// Origin pointers of the 8 fields of one state: &f[q](x=0, y=0, z=0) of the interior.
template <typename T>
struct Fields {
  T* f[NF];
};

// Local pitched geometry shared by both states: element (x, y, z), x,y,z in [-3, n+3),
// lives at origin + z*sz + y*sy + x.
struct Geom {
  int nx, ny, nz;
  long long sy, sz;
  int zwrap;  // z-marching kernel: fetch planes outside [0, nz) from their periodic image
              // instead of the z halo (one rank, z unsplit); 0: read the halo planes
  int xwrap;  // update kernels: also store the periodic x faces of the output (x unsplit): the cells
              // in the first / last 32-byte sector of a row go to the row padding on the other side
};

// One copy region of the halo machinery: cells of extent ext starting at src
// (interior coordinates) go to dst, or to / from a staging buffer at buf_off values.
struct SegDesc {
  int src[3], dst[3], ext[3];
  long long count;        // ext[0]*ext[1]*ext[2]
  long long buf_off;      // value offset of field 0 of this segment in the staging buffer
  int block0;             // first block of this segment in the launch
};
constexpr int kMaxSeg = 26;
struct SegList {
  int n;
  int nblocks;
  SegDesc s[kMaxSeg];
};
enum SegKind { SEG_SELF = 0, SEG_PACK = 1, SEG_UNPACK = 2 };

struct Region {
  int lo[3];
  int ext[3];
};

// ---- launchers (kernels.cu) ----
template <typename T, int RAD>
void launch_direct(cudaStream_t st, const Fields<T>& in, const Fields<T>& out, const Geom& g,
                   const Region& r, const Coef<T>& C, int k, T* rhs_out);
// peer-memory exchange: copy the remote segments of a state into the peers' halos; flags
template <typename T>
void launch_remote_copy(cudaStream_t st, const Fields<T>& fl, const Geom& g, const SegList& L, const RemoteMap<T>& rm);
struct FlagSet {
  unsigned long long* ptr[kMaxPeers];
  int n;
};
// Spin waits on flags written by other GPUs give up after `timeout_ns` (B2MHD_SPIN_TIMEOUT_S) and
// record the sequence number they were waiting for in *err instead of trapping (a trap would
// leave a sticky, unrecoverable context error); the host reports it (mhd_synchronize).
void launch_p2p_signal(cudaStream_t st, const FlagSet& fs, unsigned long long seq);
void launch_p2p_sync(cudaStream_t st, const FlagSet& peer_arrive, const FlagSet& my_arrive, const FlagSet& my_done,
                     unsigned long long seq, unsigned long long* err, unsigned long long timeout_ns);
void launch_p2p_wait(cudaStream_t st, const FlagSet& fs, unsigned long long seq, unsigned long long* err,
                     unsigned long long timeout_ns);
// debug (MHD_DEBUG_POISON_HALO): every halo cell of the 8 fields of a state <- quiet NaN
template <typename T>
void launch_poison_halo(cudaStream_t st, const Fields<T>& fl, const Geom& g, int rad);
template <typename T>
void launch_segments(cudaStream_t st, const Fields<T>& fl, const Geom& g, const SegList& L, int kind, T* buf);
template <typename TS, typename TD>
void launch_copy_in(cudaStream_t st, const TS* src, TD* origin, const Geom& g);
template <typename TS, typename TD>
void launch_copy_out(cudaStream_t st, const TS* origin, TD* dst, const Geom& g);
template <typename T>
void launch_reduce(cudaStream_t st, const T* origin, const Geom& g, double* scratch, int nblocks, int want);

// ---- z-marching TMA kernel (zmarch.cuh, one instantiation per dtype and radius) ----
// TMA boxes per plane and field.  TMA requires the innermost start coordinate to be 16-byte
// aligned, so boxes start at x rounded down to 16 bytes and are widened accordingly: halo box
// COLS x ROWS x 1 from (floor16(x0 - r), y0 - r, z), f_{k-1} box PCOLS x TY x 1 from (floor16(x0), y0, z).
// Tile of a CTA: 32 x 8 cells (a 16 x 8 FP64 tile at two CTAs per SM measured slower); 32 x 4
// for FP64 at radius 4, whose (r + 2)-plane ring of 32 x 8 tiles would not fit in shared memory.
template <typename T>
constexpr int zm_tx() { return 32; }
// Tile height of the z-marching kernel.  FP64: 8 rows (4 at r = 4, where 8 does not fit in
// shared memory).  FP32 at r = 3: 16 rows (512 threads, 16 warps per SM at 122 registers),
// measured 21.4 vs 18.6 Gcell/s; at r = 1, 2 the 16-row tile was 10 % slower and at r = 4 it does
// not fit (profiles/r01/bench_f32ty*.json).
#ifndef B2_ZM_TY_F32
#define B2_ZM_TY_F32 16
#endif
#ifndef B2_ZM_TY_F64
#define B2_ZM_TY_F64 8
#endif
template <typename T, int RAD = 3>
constexpr int zm_ty() { return sizeof(T) == 8 ? (RAD >= 4 ? 4 : B2_ZM_TY_F64) : (RAD == 3 ? B2_ZM_TY_F32 : 8); }
template <typename T>
constexpr int zm_ch() { return 16 / (int)sizeof(T); }
template <typename T, int RAD>
constexpr int zm_cols() { return (zm_tx<T>() + 2 * RAD + zm_ch<T>() - 1 + zm_ch<T>() - 1) / zm_ch<T>() * zm_ch<T>(); }
template <typename T>
constexpr int zm_pcols() { return zm_tx<T>() + zm_ch<T>(); }
template <typename T, int RAD>
constexpr int zm_rows() { return zm_ty<T, RAD>() + 2 * RAD; }
struct TmapSet {
  CUtensorMap halo[NF];  // fields of the state read with the stencil
  CUtensorMap prev[NF];  // fields of the other state (f_{k-1}, read pointwise)
};
template <typename T, int RAD>
bool zmarch_supported(const Geom& g, const Region& r);
template <typename T, int RAD>
void launch_zmarch(cudaStream_t st, const TmapSet& tm, const Fields<T>& out, const Geom& g, const Region& r,
                   const Coef<T>& C, int k, T* rhs_out, int xo, bool persist = false, int zchunk = 0);

// ---- warp-specialised z-marching kernel (zsplit.cuh; FP64, radius 3) ----
template <typename T, int RAD>
bool zsplit_supported(const Geom& g, const Region& r);
template <typename T, int RAD>
void launch_zsplit(cudaStream_t st, const TmapSet& tm, const Fields<T>& out, const Geom& g, const Region& r,
                   const Coef<T>& C, int k, T* rhs_out, int xo, int zchunk = 0);

constexpr int kReduceBlocks = 592;  // 4 x 148 SMs
constexpr int kReduceVals = 5;      // min, max, sum, sum of squares, sum of exp

}  // namespace b2
