// Direct update kernel, halo segment copy/pack/unpack, load/store and reduction kernels.
//
// The direct kernel is one thread per cell, reading its 55-point neighbourhood
// (Eq. 14) through the read-only data path.  It is the general-region
// kernel (any box, used for the thin outer slabs of a decomposed subdomain)
// and the correctness baseline of the z-marching kernel; both run the canonical
// per-cell arithmetic of mhd_math.cuh.
#include <cfloat>

#include "kernels.h"

namespace b2 {

template <typename T>
struct GAcc {
  Fields<T> F;
  long long base, sy, sz;
  __device__ __forceinline__ T operator()(int q, int dx, int dy, int dz) const {
    return __ldg(F.f[q] + base + (long long)dz * sz + (long long)dy * sy + dx);
  }
};

// MODE 0: RK3 update into `out` (which holds f_{k-1} for k > 0); MODE 1: RHS to rhs_out.
template <typename T, int RAD, int MODE>
__global__ void __launch_bounds__(128) direct_kernel(Fields<T> in, Fields<T> out, Geom g, Region r, Coef<T> C,
                                                     int k, T* __restrict__ rhs_out) {
  const int x = r.lo[0] + blockIdx.x * blockDim.x + threadIdx.x;
  const int y = r.lo[1] + blockIdx.y * blockDim.y + threadIdx.y;
  const int z = r.lo[2] + blockIdx.z * blockDim.z + threadIdx.z;
  if (x >= r.lo[0] + r.ext[0] || y >= r.lo[1] + r.ext[1] || z >= r.lo[2] + r.ext[2]) return;
  const long long base = (long long)z * g.sz + (long long)y * g.sy + x;
  GAcc<T> V{in, base, g.sy, g.sz};
  Derivs<T> D;
  gather<T, RAD>(V, C, D);
  T rhs[NF];
  rhs_cell<T>(D, C, rhs);
  if (MODE == 0) {
    T fn[NF];
#pragma unroll
    for (int q = 0; q < NF; ++q) {
      const T fprev = k > 0 ? out.f[q][base] : (T)0;
      fn[q] = rk_update<T>(k, D.f[q], fprev, rhs[q], C);
      out.f[q][base] = fn[q];
    }
    if (g.xwrap) {
      // periodic x faces (x unsplit), as in the z-marching kernel's epilogue: the cells of
      // the first / last 32-byte sector of a row also go to the row padding on the other side
      constexpr int W = 32 / (int)sizeof(T);
      const long long sh = x < W ? (long long)g.nx : (x >= g.nx - W ? -(long long)g.nx : 0);
      if (sh != 0) {
#pragma unroll
        for (int q = 0; q < NF; ++q) out.f[q][base + sh] = fn[q];
      }
    }
  } else {
    const long long n = (long long)g.nx * g.ny * g.nz;
    const long long li = ((long long)z * g.ny + y) * g.nx + x;
#pragma unroll
    for (int q = 0; q < NF; ++q) rhs_out[q * n + li] = rhs[q];
  }
}

template <typename T, int RAD>
void launch_direct(cudaStream_t st, const Fields<T>& in, const Fields<T>& out, const Geom& g, const Region& r,
                   const Coef<T>& C, int k, T* rhs_out) {
  if (r.ext[0] <= 0 || r.ext[1] <= 0 || r.ext[2] <= 0) return;
  // thin x-slabs of the outer shell get a block shaped along y
  const dim3 blk = r.ext[0] >= 16 ? dim3(32, 4, 1) : dim3(r.ext[0], (128 / r.ext[0]) < 32 ? (128 / r.ext[0]) : 32, 1);
  dim3 grd((r.ext[0] + blk.x - 1) / blk.x, (r.ext[1] + blk.y - 1) / blk.y, (r.ext[2] + blk.z - 1) / blk.z);
  if (rhs_out)
    direct_kernel<T, RAD, 1><<<grd, blk, 0, st>>>(in, out, g, r, C, k, rhs_out);
  else
    direct_kernel<T, RAD, 0><<<grd, blk, 0, st>>>(in, out, g, r, C, k, nullptr);
}

// ---- peer-memory exchange helpers -------------------------------------------------------------------
// Copy of the remote segments of a state (SegDesc::buf_off = peer slot) straight into the peers'
// halos of the same state: the halo exchange of a freshly loaded state.
template <typename T>
__global__ void __launch_bounds__(256) remote_copy_kernel(Fields<T> F, Geom g, SegList L, RemoteMap<T> rm) {
  int s = 0;
  while (s + 1 < L.n && (int)blockIdx.x >= L.s[s + 1].block0) ++s;
  const SegDesc& d = L.s[s];
  const unsigned c = (blockIdx.x - (unsigned)d.block0) * blockDim.x + threadIdx.x;
  if (c < (unsigned)d.count) {
    const unsigned ex = (unsigned)d.ext[0], ey = (unsigned)d.ext[1];
    const unsigned rr = c / ex;
    const int cx = (int)(c - rr * ex);
    const unsigned czu = rr / ey;
    const int cy = (int)(rr - czu * ey);
    const int cz = (int)czu;
    const long long so = (long long)(d.src[2] + cz) * g.sz + (long long)(d.src[1] + cy) * g.sy + (d.src[0] + cx);
    const long long dof = (long long)(d.dst[2] + cz) * g.sz + (long long)(d.dst[1] + cy) * g.sy + (d.dst[0] + cx);
    const int p = (int)d.buf_off;
#pragma unroll
    for (int q = 0; q < NF; ++q) rm.f[p][q][dof] = F.f[q][so];
  }
  __threadfence_system();
}

template <typename T>
void launch_remote_copy(cudaStream_t st, const Fields<T>& fl, const Geom& g, const SegList& L, const RemoteMap<T>& rm) {
  if (L.n == 0 || L.nblocks == 0) return;
  remote_copy_kernel<T><<<L.nblocks, 256, 0, st>>>(fl, g, L, rm);
}

// Cross-GPU ordering with system-scope flags (process mode: one process per GPU).  Every operation
// that touches halos across ranks (a boundary update whose results are copied into the neighbours'
// halos, or a halo copy) has a sequence number s and is bracketed by
//   sync(s):  publish arrive = s to every neighbour (all earlier work of this rank on the stream,
//             reads of its own halo included, is complete), then wait until every neighbour has
//             arrive >= s (it is done reading what we are about to overwrite) and done >= s - 1
//             (its writes into our halo from the previous operation have landed);
//   done(s):  after the remote stores, fence and publish done = s.
// Ranks must enqueue their operations in lockstep (the same sequence on every rank).  A wait that
// outlasts timeout_ns gives up and records s in *err (reported by the host) instead of trapping.
__device__ __forceinline__ unsigned long long now_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];\n" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__global__ void p2p_sync_kernel(FlagSet peer_arrive, FlagSet my_arrive, FlagSet my_done, unsigned long long seq,
                                unsigned long long* err, unsigned long long timeout_ns) {
  for (int i = 0; i < peer_arrive.n; ++i)
    asm volatile("st.release.sys.global.u64 [%0], %1;\n" ::"l"(peer_arrive.ptr[i]), "l"(seq) : "memory");
  const unsigned long long t0 = now_ns();
  for (int i = 0; i < my_arrive.n; ++i) {
    while (!(ld_acquire_sys(my_arrive.ptr[i]) >= seq && ld_acquire_sys(my_done.ptr[i]) + 1 >= seq)) {
      __nanosleep(128);
      if (now_ns() - t0 > timeout_ns) {
        atomicMax(err, seq);
        return;
      }
    }
  }
}

__global__ void p2p_signal_kernel(FlagSet fs, unsigned long long seq) {
  __threadfence_system();
  for (int i = 0; i < fs.n; ++i)
    asm volatile("st.release.sys.global.u64 [%0], %1;\n" ::"l"(fs.ptr[i]), "l"(seq) : "memory");
}

__global__ void p2p_wait_kernel(FlagSet fs, unsigned long long seq, unsigned long long* err,
                                unsigned long long timeout_ns) {
  const unsigned long long t0 = now_ns();
  for (int i = 0; i < fs.n; ++i) {
    while (ld_acquire_sys(fs.ptr[i]) < seq) {
      __nanosleep(128);
      if (now_ns() - t0 > timeout_ns) {
        atomicMax(err, seq);
        return;
      }
    }
  }
}

void launch_p2p_sync(cudaStream_t st, const FlagSet& peer_arrive, const FlagSet& my_arrive, const FlagSet& my_done,
                     unsigned long long seq, unsigned long long* err, unsigned long long timeout_ns) {
  p2p_sync_kernel<<<1, 1, 0, st>>>(peer_arrive, my_arrive, my_done, seq, err, timeout_ns);
}
void launch_p2p_signal(cudaStream_t st, const FlagSet& fs, unsigned long long seq) {
  p2p_signal_kernel<<<1, 1, 0, st>>>(fs, seq);
}
void launch_p2p_wait(cudaStream_t st, const FlagSet& fs, unsigned long long seq, unsigned long long* err,
                     unsigned long long timeout_ns) {
  p2p_wait_kernel<<<1, 1, 0, st>>>(fs, seq, err, timeout_ns);
}

// ---- debug: NaN poison of a state's halo ----------------------------------------------------------
// Every cell of the halo-inclusive box [-r, n + r)^3 outside the interior, all 8 fields, gets a quiet
// NaN: a stencil that reads a halo cell the schedule did not refresh (a corner that is not
// exchanged; a z plane behind the TMA wrap; a stale face) turns the result into NaN.
template <typename T>
__global__ void __launch_bounds__(256) poison_kernel(Fields<T> F, Geom g, int rad) {
  const int mx = g.nx + 2 * rad, my = g.ny + 2 * rad, mz = g.nz + 2 * rad;
  const long long n = (long long)mx * my * mz;
  const T nan = (T)__longlong_as_double(0x7ff8000000000000LL);
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const int x = (int)(i % mx) - rad;
    const long long rr = i / mx;
    const int y = (int)(rr % my) - rad, z = (int)(rr / my) - rad;
    if (x >= 0 && x < g.nx && y >= 0 && y < g.ny && z >= 0 && z < g.nz) continue;
    const long long o = (long long)z * g.sz + (long long)y * g.sy + x;
#pragma unroll
    for (int q = 0; q < NF; ++q) F.f[q][o] = nan;
  }
}
template <typename T>
void launch_poison_halo(cudaStream_t st, const Fields<T>& fl, const Geom& g, int rad) {
  poison_kernel<T><<<148 * 4, 256, 0, st>>>(fl, g, rad);
}

// ---- halo segments ---------------------------------------------------------
// One launch covers every segment of a list; each block belongs to exactly one segment.
template <typename T, int KIND>
__global__ void __launch_bounds__(256) seg_kernel(Fields<T> F, Geom g, SegList L, T* __restrict__ buf) {
  int s = 0;
  while (s + 1 < L.n && (int)blockIdx.x >= L.s[s + 1].block0) ++s;
  const SegDesc& d = L.s[s];
  // 32-bit index math (a segment holds < 2^31 cells): 64-bit div/mod per cell dominated this kernel
  const unsigned c = (blockIdx.x - (unsigned)d.block0) * blockDim.x + threadIdx.x;
  if (c >= (unsigned)d.count) return;
  const unsigned ex = (unsigned)d.ext[0], ey = (unsigned)d.ext[1];
  const unsigned rr = c / ex;
  const int cx = (int)(c - rr * ex);
  const unsigned cz = rr / ey;
  const int cy = (int)(rr - cz * ey);
  const long long so = (long long)(d.src[2] + (int)cz) * g.sz + (long long)(d.src[1] + cy) * g.sy + (d.src[0] + cx);
  const long long dof = (long long)(d.dst[2] + (int)cz) * g.sz + (long long)(d.dst[1] + cy) * g.sy + (d.dst[0] + cx);
  T v[NF];
#pragma unroll
  for (int q = 0; q < NF; ++q) v[q] = KIND == SEG_UNPACK ? buf[d.buf_off + (long long)q * d.count + c] : F.f[q][so];
#pragma unroll
  for (int q = 0; q < NF; ++q) {
    if (KIND == SEG_SELF || KIND == SEG_UNPACK) F.f[q][dof] = v[q];
    if (KIND == SEG_PACK) buf[d.buf_off + (long long)q * d.count + c] = v[q];
  }
}

template <typename T>
void launch_segments(cudaStream_t st, const Fields<T>& fl, const Geom& g, const SegList& L, int kind, T* buf) {
  if (L.n == 0 || L.nblocks == 0) return;
  if (kind == SEG_SELF) seg_kernel<T, SEG_SELF><<<L.nblocks, 256, 0, st>>>(fl, g, L, buf);
  if (kind == SEG_PACK) seg_kernel<T, SEG_PACK><<<L.nblocks, 256, 0, st>>>(fl, g, L, buf);
  if (kind == SEG_UNPACK) seg_kernel<T, SEG_UNPACK><<<L.nblocks, 256, 0, st>>>(fl, g, L, buf);
}

// ---- load / store: contiguous local interior <-> pitched field ----------------------------------
template <typename TS, typename TD>
__global__ void copy_in_kernel(const TS* __restrict__ src, TD* origin, Geom g) {
  const long long n = (long long)g.nx * g.ny * g.nz;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const int x = (int)(i % g.nx);
    const long long r = i / g.nx;
    const int y = (int)(r % g.ny);
    const int z = (int)(r / g.ny);
    origin[(long long)z * g.sz + (long long)y * g.sy + x] = (TD)src[i];
  }
}
template <typename TS, typename TD>
__global__ void copy_out_kernel(const TS* origin, TD* __restrict__ dst, Geom g) {
  const long long n = (long long)g.nx * g.ny * g.nz;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const int x = (int)(i % g.nx);
    const long long r = i / g.nx;
    const int y = (int)(r % g.ny);
    const int z = (int)(r / g.ny);
    dst[i] = (TD)origin[(long long)z * g.sz + (long long)y * g.sy + x];
  }
}
template <typename TS, typename TD>
void launch_copy_in(cudaStream_t st, const TS* src, TD* origin, const Geom& g) {
  copy_in_kernel<TS, TD><<<148 * 8, 256, 0, st>>>(src, origin, g);
}
template <typename TS, typename TD>
void launch_copy_out(cudaStream_t st, const TS* origin, TD* dst, const Geom& g) {
  copy_out_kernel<TS, TD><<<148 * 8, 256, 0, st>>>(origin, dst, g);
}

// ---- reductions (min, max, sum, and the sum of squares or of exp when asked), two stages --------------
// min, max and sum are always formed (a NaN or Inf anywhere shows in the sum, so every reduction
// checks finiteness); slot 3 holds the sum of squares (want == 3) or of exp (want == 4), else 0.
__device__ __forceinline__ void red_combine(double* a, const double* b) {
  a[0] = fmin(a[0], b[0]);
  a[1] = fmax(a[1], b[1]);
  a[2] += b[2];
  a[3] += b[3];
  a[4] += b[4];
}

template <typename T>
__global__ void __launch_bounds__(256) reduce_stage1(const T* origin, Geom g, double* partial, int want) {
  double v[kReduceVals] = {DBL_MAX, -DBL_MAX, 0.0, 0.0, 0.0};
  const long long n = (long long)g.nx * g.ny * g.nz;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const int x = (int)(i % g.nx);
    const long long r = i / g.nx;
    const int y = (int)(r % g.ny);
    const int z = (int)(r / g.ny);
    const double f = (double)origin[(long long)z * g.sz + (long long)y * g.sy + x];
    // NaN propagates through fmin/fmax only if both are NaN: track it in the sum instead
    v[0] = fmin(v[0], f);
    v[1] = fmax(v[1], f);
    v[2] += f;
    if (want == 3) v[3] += f * f;
    if (want == 4) v[4] += exp(f);
  }
  __shared__ double sh[256][kReduceVals];
  for (int j = 0; j < kReduceVals; ++j) sh[threadIdx.x][j] = v[j];
  __syncthreads();
  for (int w = blockDim.x / 2; w > 0; w >>= 1) {
    if ((int)threadIdx.x < w) red_combine(sh[threadIdx.x], sh[threadIdx.x + w]);
    __syncthreads();
  }
  if (threadIdx.x == 0)
    for (int j = 0; j < kReduceVals; ++j) partial[blockIdx.x * kReduceVals + j] = sh[0][j];
}

__global__ void reduce_stage2(double* partial, int nblocks) {
  __shared__ double sh[256][kReduceVals];
  double v[kReduceVals] = {DBL_MAX, -DBL_MAX, 0.0, 0.0, 0.0};
  for (int b = threadIdx.x; b < nblocks; b += blockDim.x) red_combine(v, partial + b * kReduceVals);
  for (int j = 0; j < kReduceVals; ++j) sh[threadIdx.x][j] = v[j];
  __syncthreads();
  for (int w = blockDim.x / 2; w > 0; w >>= 1) {
    if ((int)threadIdx.x < w) red_combine(sh[threadIdx.x], sh[threadIdx.x + w]);
    __syncthreads();
  }
  if (threadIdx.x == 0)
    for (int j = 0; j < kReduceVals; ++j) partial[j] = sh[0][j];
}

template <typename T>
void launch_reduce(cudaStream_t st, const T* origin, const Geom& g, double* scratch, int nblocks, int want) {
  reduce_stage1<T><<<nblocks, 256, 0, st>>>(origin, g, scratch, want);
  reduce_stage2<<<1, 256, 0, st>>>(scratch, nblocks);
}

// ---- explicit instantiations ----------------------------------------------------------------------
#define B2_DIRECT(T, RAD)                                                                               \
  template void launch_direct<T, RAD>(cudaStream_t, const Fields<T>&, const Fields<T>&, const Geom&,      \
                                      const Region&, const Coef<T>&, int, T*);
B2_DIRECT(float, 1)
B2_DIRECT(float, 2)
B2_DIRECT(float, 3)
B2_DIRECT(float, 4)
B2_DIRECT(double, 1)
B2_DIRECT(double, 2)
B2_DIRECT(double, 3)
B2_DIRECT(double, 4)
#undef B2_DIRECT
#define B2_INST(T)                                                                                       \
  template void launch_remote_copy<T>(cudaStream_t, const Fields<T>&, const Geom&, const SegList&,        \
                                      const RemoteMap<T>&);                                              \
  template void launch_segments<T>(cudaStream_t, const Fields<T>&, const Geom&, const SegList&, int, T*); \
  template void launch_reduce<T>(cudaStream_t, const T*, const Geom&, double*, int, int);              \
  template void launch_poison_halo<T>(cudaStream_t, const Fields<T>&, const Geom&, int);
B2_INST(float)
B2_INST(double)
#undef B2_INST
template void launch_copy_in<float, float>(cudaStream_t, const float*, float*, const Geom&);
template void launch_copy_in<double, double>(cudaStream_t, const double*, double*, const Geom&);
template void launch_copy_in<float, double>(cudaStream_t, const float*, double*, const Geom&);
template void launch_copy_in<double, float>(cudaStream_t, const double*, float*, const Geom&);
template void launch_copy_out<float, float>(cudaStream_t, const float*, float*, const Geom&);
template void launch_copy_out<double, double>(cudaStream_t, const double*, double*, const Geom&);
template void launch_copy_out<float, double>(cudaStream_t, const float*, double*, const Geom&);
template void launch_copy_out<double, float>(cudaStream_t, const double*, float*, const Geom&);

}  // namespace b2
