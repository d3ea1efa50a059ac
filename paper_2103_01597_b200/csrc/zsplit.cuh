// Warp-specialised z-marching update (FP64; the default for order 8, an option for order 6).
//
// Same staging as zmarch.cuh (TMA ring of r + 2 planes of the tile with its radius-r halo,
// f_{k-1} of the output plane in the same transaction, z column in registers, push/pull z-cross
// terms), but each cell is served by TWO threads in two warp groups: for the 32 x 8 tile of order
// 6, 2 x 8 warps (512 threads, 16 warps per SM instead of 8, registers rebalanced by setmaxnreg);
// for the 32 x 4 tile of order 8, 2 x 4 warps (8 warps per SM instead of 4, up to 255 registers
// each).  Measured: order 8 9.46 vs 6.59 Gcell/s (default); order 6 12.3 vs 13.3.
//   group 0 ("magnetic"):  A -> B, mu0 j, lap A (the magnetic contraction of Eq. B.2-B.4),
//                          grad lnrho and lap lnrho; then dA/dt (B.4) and the A update;
//   group 1 ("flow"):      u and s derivatives; then B.1-B.3 and the lnrho, u, s update.
// Group 0 hands grad lnrho, lap lnrho and the pointwise factors of mhd_math.cuh::thermo (Lorentz
// acceleration, ohmic heating, 1/rho, c_s^2, 1/T: 11 values per cell) to group 1 through tensor
// memory (tcgen05.st / tcgen05.ld, 32x32b: the two threads of a cell sit in the same lane of warps
// w and w + NWARP/2, which share a TMEM lane quadrant), double-buffered by plane parity and ordered by
// named barriers.  Each thread carries half the register state of the single-group kernel (the z
// history and cross accumulators of its own fields), so twice the warps fit; ring slots are
// released per plane through "empty" mbarriers (one arrival per warp) instead of a CTA barrier,
// so the magnetic group runs up to a plane ahead and its load-heavy derivative phase overlaps the
// flow group's load-free RHS phase.
//
// The march is not unrolled by phase (the z history and the cross accumulators shift by register
// moves): two groups of r-fold unrolled code did not fit the instruction cache.
// Every value is produced by the same expressions in the same order as mhd_math.cuh (rhs_rest =
// visc_parts + thermo + rhs_flow + rhs_induction), so the result is bit-identical to the direct and
// single-group kernels (tests/test_gpu_parity.py::test_kernel_variants_bit_identical,
// test_orders_rhs_steps_and_kernels).
#pragma once
#include "zmarch.cuh"

namespace b2 {
namespace zs {
using zm::mbar_expect_tx;
using zm::mbar_init;
using zm::mbar_wait;
using zm::smem_u32;
using zm::tma_load_3d;
using zm::ZCfg;

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void nbar_sync(int id, int count) {
  asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(count) : "memory");
}
__device__ __forceinline__ void nbar_arrive(int id, int count) {
  asm volatile("bar.arrive %0, %1;\n" ::"r"(id), "r"(count) : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory"); }

// The 11 handed-over values of one cell as 22 32-bit TMEM columns of this thread's lane.
constexpr int kXV = 11;
__device__ __forceinline__ void xchg_store(unsigned addr, const double (&v)[kXV]) {
  unsigned r[2 * kXV];
#pragma unroll
  for (int i = 0; i < kXV; ++i) {
    r[2 * i] = (unsigned)__double2loint(v[i]);
    r[2 * i + 1] = (unsigned)__double2hiint(v[i]);
  }
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
      "%15, %16};\n" ::"r"(addr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
      "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
      : "memory");
  asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1, %2, %3, %4};\n" ::"r"(addr + 16), "r"(r[16]),
               "r"(r[17]), "r"(r[18]), "r"(r[19])
               : "memory");
  asm volatile("tcgen05.st.sync.aligned.32x32b.x2.b32 [%0], {%1, %2};\n" ::"r"(addr + 20), "r"(r[20]), "r"(r[21])
               : "memory");
  asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
}
__device__ __forceinline__ void xchg_load(unsigned addr, double (&v)[kXV]) {
  unsigned r[2 * kXV];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
      "%15}, [%16];\n"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(addr)
      : "memory");
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0, %1, %2, %3}, [%4];\n"
               : "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19])
               : "r"(addr + 16)
               : "memory");
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x2.b32 {%0, %1}, [%2];\n"
               : "=r"(r[20]), "=r"(r[21])
               : "r"(addr + 20)
               : "memory");
  asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
  for (int i = 0; i < kXV; ++i) v[i] = __hiloint2double((int)r[2 * i + 1], (int)r[2 * i]);
}

// Register state one thread carries along z: its group's vector field (A or u) and scalar field
// (lnrho or s).
template <typename T, int RAD>
struct GState {
  T hv[3][RAD];   // f(o-r) .. f(o-1) of the vector components (f(o-i) at [RAD - i])
  T hs[RAD];      // same for the scalar field
  T acc[RAD][3];  // [output o + j][z-part of x_0, x_1, x_2]

  // after plane o: append its values to the history
  __device__ __forceinline__ void append(const T (&v)[3], T sc) {
#pragma unroll
    for (int j = 0; j + 1 < RAD; ++j) {
#pragma unroll
      for (int c = 0; c < 3; ++c) hv[c][j] = hv[c][j + 1];
      hs[j] = hs[j + 1];
    }
#pragma unroll
    for (int c = 0; c < 3; ++c) hv[c][RAD - 1] = v[c];
    hs[RAD - 1] = sc;
  }
};

template <typename T, int RAD>
struct SCfg {
  using Z = ZCfg<T, RAD>;
  static constexpr int NT = 2 * Z::NT;  // two threads per cell
  static constexpr int NWARP = NT / 32;
  // r + 2 ring slots and f_{k-1} staged by TMA as in zmarch.cuh.  (Measured alternative: r + 3
  // slots with f_{k-1} read straight from global memory to make room: k = 0 7 % slower, k > 0 45 %
  // slower, the pointwise global loads exposed; profiles/r02/split3_*.)
  static constexpr int NSLOT = RAD + 2;
  static constexpr size_t SMEM = (size_t)(NSLOT * Z::SLOT + 2 * NF * Z::PSZ) * Z::ES + 128;
  // 32 x 8 tiles (512 threads, registers rebalanced by setmaxnreg) and the 32 x 4 tiles of radius 4
  // (256 threads: every thread may use 255 registers, 8 warps per SM instead of 4)
  static constexpr bool OK = sizeof(T) == 8 && (Z::NT == 256 || Z::NT == 128) && SMEM <= 227 * 1024;
};

template <typename T, int RAD, int MODE>
struct SStep {
  using Z = ZCfg<T, RAD>;
  const T* ring;
  const T* prevbuf;
  const Coef<T>& C;
  int cell;
  int pcell;
  int slot0;

  __device__ __forceinline__ const T* slot_of(int plane) const {
    return ring + ((plane - slot0) % SCfg<T, RAD>::NSLOT) * Z::SLOT + cell;
  }
  static __device__ __forceinline__ T at(const T* sp, int q, int dx, int dy) {
    return sp[q * Z::FSZ + dy * Z::COLS + dx];
  }
  __device__ __forceinline__ void axis_xy(const T* sp, int q, T f0, T (&d1)[2], T (&d2)[2], T (&dlx)[RAD],
                                          T (&dly)[RAD]) const {
    T sgx[RAD], sgy[RAD];
#pragma unroll
    for (int i = 1; i <= RAD; ++i) {
      const T px = at(sp, q, i, 0), mx = at(sp, q, -i, 0);
      const T py = at(sp, q, 0, i), my = at(sp, q, 0, -i);
      dlx[i - 1] = px - mx;
      sgx[i - 1] = px + mx;
      dly[i - 1] = py - my;
      sgy[i - 1] = py + my;
    }
    d1[0] = d1_of<T, RAD>(dlx, C.c1[0]);
    d2[0] = d2_of<T, RAD>(f0, sgx, C.d2[0], C.d0[0]);
    d1[1] = d1_of<T, RAD>(dly, C.c1[1]);
    d2[1] = d2_of<T, RAD>(f0, sgy, C.d2[1], C.d0[1]);
  }
  __device__ __forceinline__ void axis_z(const T (&h)[RAD], int q, T f0, const T* const (&sk)[RAD + 1], T& d1,
                                         T& d2) const {
    T dl[RAD], sg[RAD];
#pragma unroll
    for (int i = 1; i <= RAD; ++i) {
      const T p = at(sk[i], q, 0, 0), m = h[RAD - i];
      dl[i - 1] = p - m;
      sg[i - 1] = p + m;
    }
    d1 = d1_of<T, RAD>(dl, C.c1[2]);
    d2 = d2_of<T, RAD>(f0, sg, C.d2[2], C.d0[2]);
  }
  __device__ __forceinline__ T cross_xy_s(const T* sp, int q) const {
    const T* w = C.xw[0];
    T a = (-w[RAD - 1]) * (at(sp, q, RAD, -RAD) - at(sp, q, -RAD, -RAD));
#pragma unroll
    for (int k = -RAD + 1; k <= RAD; ++k) {
      if (k == 0) continue;
      const int i = k < 0 ? -k : k;
      a = fma_(k < 0 ? -w[i - 1] : w[i - 1], at(sp, q, i, k) - at(sp, q, -i, k), a);
    }
    return a;
  }
  // k < 0 half of the z-cross terms of plane o (the current output, whose accumulator acc[0] has
  // been consumed): outputs o + j, j < r, and a fresh accumulator for o + r; then shift by one plane
  __device__ __forceinline__ void push(GState<T, RAD>& st, const T (&dlx_x)[RAD], const T (&dly_y)[RAD],
                                       const T (&dlx_z)[RAD], const T (&dly_z)[RAD]) const {
    const T* wxz = C.xw[1];
    const T* wyz = C.xw[2];
#pragma unroll
    for (int j = 1; j < RAD; ++j) {
      T* a = st.acc[j];
      a[0] = fma_(-wxz[j - 1], dlx_z[j - 1], a[0]);
      a[1] = fma_(-wyz[j - 1], dly_z[j - 1], a[1]);
      a[2] = fma_(-wxz[j - 1], dlx_x[j - 1], a[2]);
      a[2] = fma_(-wyz[j - 1], dly_y[j - 1], a[2]);
    }
#pragma unroll
    for (int j = 0; j + 1 < RAD; ++j)
#pragma unroll
      for (int c = 0; c < 3; ++c) st.acc[j][c] = st.acc[j + 1][c];
    T* f = st.acc[RAD - 1];
    f[0] = (-wxz[RAD - 1]) * dlx_z[RAD - 1];
    f[1] = (-wyz[RAD - 1]) * dly_z[RAD - 1];
    f[2] = fma_(-wyz[RAD - 1], dly_y[RAD - 1], (-wxz[RAD - 1]) * dlx_x[RAD - 1]);
  }
  // push-only pass over a plane below the chunk (prologue)
  __device__ __forceinline__ void push_only(GState<T, RAD>& st, int p, int qx, int qs) const {
    const T* s0 = slot_of(p);
    T dlx_x[RAD], dly_y[RAD], dlx_z[RAD], dly_z[RAD];
#pragma unroll
    for (int i = 1; i <= RAD; ++i) {
      dlx_x[i - 1] = at(s0, qx, i, 0) - at(s0, qx, -i, 0);
      dly_y[i - 1] = at(s0, qx + 1, 0, i) - at(s0, qx + 1, 0, -i);
      dlx_z[i - 1] = at(s0, qx + 2, i, 0) - at(s0, qx + 2, -i, 0);
      dly_z[i - 1] = at(s0, qx + 2, 0, i) - at(s0, qx + 2, 0, -i);
    }
    push(st, dlx_x, dly_y, dlx_z, dly_z);
    const T v[3] = {at(s0, qx, 0, 0), at(s0, qx + 1, 0, 0), at(s0, qx + 2, 0, 0)};
    st.append(v, at(s0, qs, 0, 0));
  }
  // derivatives of the group's vector field at output plane o (as ZStep::vector_derivs)
  __device__ __forceinline__ void vec(GState<T, RAD>& st, int qx, const T* const (&sk)[RAD + 1], T (&f)[3],
                                      T (&g)[3][3], T (&d2)[3][3], T (&x)[3]) const {
    const T* s0 = sk[0];
    T dlx[3][RAD], dly[3][RAD];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const int q = qx + c;
      T d1a[2], d2a[2];
      f[c] = at(s0, q, 0, 0);
      axis_xy(s0, q, f[c], d1a, d2a, dlx[c], dly[c]);
      axis_z(st.hv[c], q, f[c], sk, g[c][2], d2[c][2]);
      g[c][0] = d1a[0];
      g[c][1] = d1a[1];
      d2[c][0] = d2a[0];
      d2[c][1] = d2a[1];
    }
    const T P0 = cross_xy_s(s0, qx + 1);  // d_x d_y v_y
    const T P1 = cross_xy_s(s0, qx);      // d_x d_y v_x
    const T* a = st.acc[0];
    x[0] = a[0] + P0;
    x[1] = a[1] + P1;
    x[2] = a[2];
    const T* wxz = C.xw[1];
    const T* wyz = C.xw[2];
#pragma unroll
    for (int kk = 1; kk <= RAD; ++kk) {
      const T* s = sk[kk];
      x[0] = fma_(wxz[kk - 1], at(s, qx + 2, kk, 0) - at(s, qx + 2, -kk, 0), x[0]);
      x[1] = fma_(wyz[kk - 1], at(s, qx + 2, 0, kk) - at(s, qx + 2, 0, -kk), x[1]);
      x[2] = fma_(wxz[kk - 1], at(s, qx, kk, 0) - at(s, qx, -kk, 0), x[2]);
      x[2] = fma_(wyz[kk - 1], at(s, qx + 1, 0, kk) - at(s, qx + 1, 0, -kk), x[2]);
    }
    push(st, dlx[0], dly[1], dlx[2], dly[2]);
  }
  // gradient and Laplacian of the group's scalar field
  __device__ __forceinline__ void scalar(const GState<T, RAD>& st, int q, const T* const (&sk)[RAD + 1], T& f,
                                         T (&g)[3], T& lap) const {
    T d1a[2], d2a[2], dlx[RAD], dly[RAD], d2z;
    f = at(sk[0], q, 0, 0);
    axis_xy(sk[0], q, f, d1a, d2a, dlx, dly);
    axis_z(st.hs, q, f, sk, g[2], d2z);
    g[0] = d1a[0];
    g[1] = d1a[1];
    lap = (d2a[0] + d2a[1]) + d2z;
  }
  // RK3 update (or RHS output) of fields q0 .. q0 + NQ - 1 of this cell; f_{k-1} from the staged tile
  template <int NQ>
  __device__ __forceinline__ void finish(int o, int q0, const T (&fk)[NQ], const T (&rhs)[NF], const Fields<T>& out,
                                         const Geom& g, int k, int x, int y, T* rhs_out) const {
    if (MODE == 0) {
      const long long gidx = (long long)o * g.sz + (long long)y * g.sy + x;
      const T* pv = prevbuf + ((o & 1) * NF) * Z::PSZ + pcell;
      T fn[NQ];
#pragma unroll
      for (int i = 0; i < NQ; ++i) {
        const int q = q0 + i;
        fn[i] = rk_update<T>(k, fk[i], k > 0 ? pv[q * Z::PSZ] : (T)0, rhs[q], C);
        out.f[q][gidx] = fn[i];
      }
      if (g.xwrap) {
        constexpr int W = 32 / (int)sizeof(T);
        const long long sh = x < W ? (long long)g.nx : (x >= g.nx - W ? -(long long)g.nx : 0);
        if (sh != 0) {
#pragma unroll
          for (int i = 0; i < NQ; ++i) out.f[q0 + i][gidx + sh] = fn[i];
        }
      }
    } else {
      const long long n = (long long)g.nx * g.ny * g.nz;
      const long long li = ((long long)o * g.ny + y) * g.nx + x;
#pragma unroll
      for (int i = 0; i < NQ; ++i) rhs_out[(q0 + i) * n + li] = rhs[q0 + i];
    }
  }
};

// named barrier ids: 1, 2 = "exchange of plane o written" (by o & 1); 3, 4 = "exchange of plane o read"
constexpr int kBarProd = 1, kBarCons = 3;


// Registers per thread of each group after setmaxnreg (the kernel starts at 65536 / 512 = 128):
// the flow group carries the RHS of B.1-B.3, the magnetic group only the contraction and B.4.
#ifndef B2_ZS_REG_MAG
#define B2_ZS_REG_MAG 128  // measured 112 / 120 / 128 / 136: 11.8 / 12.3 / 13.2 / (spills) Gcell/s
#endif
#define B2_ZS_REG_FLOW (256 - B2_ZS_REG_MAG)

// Shared per-CTA context of the split kernel (pointers to the grid-constant kernel parameters).
template <typename T, int RAD, int MODE>
struct SCtx {
  using Z = ZCfg<T, RAD>;
  static constexpr int NSLOT = SCfg<T, RAD>::NSLOT;
  T* ring;
  T* prevbuf;
  uint64_t* full;
  uint64_t* empty;
  const TmapSet* tm;
  const Fields<T>* out;
  const Geom* g;
  const Coef<T>* C;
  int k, xo;
  T* rhs_out;
  int zb, ze, first, last, xs, pxs, x0, y0;
  bool need_prev, active;

  // one TMA transaction per staged plane P: its halo tile, plus f_{k-1} of output plane P - r
  __device__ __forceinline__ void issue(int P) const {
    const int s = (P - first) % NSLOT;
    const int po = P - RAD;
    const bool pv = need_prev && po >= zb && po < ze;
    mbar_expect_tx(&full[s], Z::HALO_TX + (pv ? Z::PREV_TX : 0u));
    T* dst = ring + s * Z::SLOT;
    const int pz = !g->zwrap ? P : (P < 0 ? P + g->nz : (P >= g->nz ? P - g->nz : P));
#pragma unroll
    for (int q = 0; q < NF; ++q) tma_load_3d(dst + q * Z::FSZ, &tm->halo[q], &full[s], xs + xo, y0, pz + RAD);
    if (pv) {
      T* pd = prevbuf + (po & 1) * NF * Z::PSZ;
#pragma unroll
      for (int q = 0; q < NF; ++q) tma_load_3d(pd + q * Z::PSZ, &tm->prev[q], &full[s], pxs + xo, y0 + RAD, po + RAD);
    }
  }
  __device__ __forceinline__ void wait_full(int P) const {
    const int rel = P - first;
    mbar_wait(&full[rel % NSLOT], (unsigned)(rel / NSLOT) & 1u);
  }
};

// The march of one group over the CTA's column (GRP 0: magnetic, 1: flow).
template <typename T, int RAD, int MODE, int GRP>
__device__ __forceinline__ void group_march(const SCtx<T, RAD, MODE>& X, int ct, int lane, unsigned tq) {
  using Z = ZCfg<T, RAD>;
  using S = SCfg<T, RAD>;
  constexpr int TX = Z::TX, NSLOT = S::NSLOT;
  const int tx = ct % TX, ty = ct / TX;
  const int cx = X.x0 + tx, cy = X.y0 + ty;  // the cell
  const bool producer = GRP == 1 && ct == 0;
  const SStep<T, RAD, MODE> S2{X.ring, X.prevbuf, *X.C, (ty + RAD) * Z::COLS + (cx - X.xs), ty * Z::PCOLS + (cx - X.pxs),
                               X.first};
  const Coef<T>& C = *X.C;
  GState<T, RAD> st;
#pragma unroll
  for (int j = 0; j < RAD; ++j)
#pragma unroll
    for (int c = 0; c < 3; ++c) st.acc[j][c] = (T)0;
  const int zb = X.zb, ze = X.ze;

#pragma unroll
  for (int i = 0; i < RAD; ++i) X.wait_full(X.first + i);

#pragma unroll 1
  for (int p = X.first; p < ze; ++p) {
    X.wait_full(p + RAD);
    if (p < zb) {
      S2.push_only(st, p, GRP ? UX : AX, GRP ? SS : LNRHO);
    } else {
      const T* sk[RAD + 1];
#pragma unroll
      for (int i = 0; i <= RAD; ++i) sk[i] = S2.slot_of(p + i);
      const unsigned xb = (unsigned)((p & 1) * 2 * 2 * kXV);  // exchange buffer of this plane's parity
      T rhs[NF];
      if constexpr (GRP == 0) {
        T fA[3], gA[3][3], d2A[3][3], xA[3];
        S2.vec(st, AX, sk, fA, gA, d2A, xA);
        const MagPart<T> m = mag_part<T>(gA, d2A, xA);
        T lr, gl[3], lapl;
        S2.scalar(st, LNRHO, sk, lr, gl, lapl);
        {
          const Thermo<T> t = thermo<T>(lr, S2.at(sk[0], SS, 0, 0), m, C);
          if (p >= zb + 2) {
            nbar_sync(kBarCons + (p & 1), S::NT);  // the flow group has read plane p - 2's values
            tc_fence_after();
          }
          const double v[kXV] = {t.L[0], t.L[1], t.L[2], t.ohm, t.inv_rho, t.cs2, t.inv_T, gl[0], gl[1], gl[2], lapl};
          xchg_store(tq + xb, v);
          tc_fence_before();
          nbar_arrive(kBarProd + (p & 1), S::NT);
        }
        const T u[3] = {S2.at(sk[0], UX, 0, 0), S2.at(sk[0], UY, 0, 0), S2.at(sk[0], UZ, 0, 0)};
        rhs_induction<T>(u, m, C, rhs);
        if (X.active) S2.template finish<3>(p, AX, fA, rhs, *X.out, *X.g, X.k, cx, cy, X.rhs_out);
        st.append(fA, lr);
      } else {
        T u[3], gu[3][3], lapu[3], gdu[3];
        {
          T d2u[3][3], xu[3];
          S2.vec(st, UX, sk, u, gu, d2u, xu);
          visc_parts<T>(d2u, xu, lapu, gdu);
        }
        T sv, gs[3], laps;
        S2.scalar(st, SS, sk, sv, gs, laps);
        double v[kXV];
        nbar_sync(kBarProd + (p & 1), S::NT);
        tc_fence_after();
        xchg_load(tq + xb, v);
        tc_fence_before();
        nbar_arrive(kBarCons + (p & 1), S::NT);
        Thermo<T> t;
        t.L[0] = v[0];
        t.L[1] = v[1];
        t.L[2] = v[2];
        t.ohm = v[3];
        t.inv_rho = v[4];
        t.cs2 = v[5];
        t.inv_T = v[6];
        const T gl[3] = {v[7], v[8], v[9]};
        rhs_flow<T>(u, gl, gs, gu, v[10], laps, lapu, gdu, t, C, rhs);
        const T fk[5] = {S2.at(sk[0], LNRHO, 0, 0), u[0], u[1], u[2], sv};  // fields LNRHO .. SS are 0 .. 4
        if (X.active) S2.template finish<5>(p, LNRHO, fk, rhs, *X.out, *X.g, X.k, cx, cy, X.rhs_out);
        st.append(u, sv);
      }
    }
    // release plane p's slot (one arrival per warp); the producer refills it with plane p + NSLOT
    __syncwarp();
    if (lane == 0) mbar_arrive(&X.empty[(p - X.first) % NSLOT]);
    if (producer && p + NSLOT <= X.last) {
      mbar_wait(&X.empty[(p - X.first) % NSLOT], (unsigned)((p - X.first) / NSLOT) & 1u);
      asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
      X.issue(p + NSLOT);
    }
    __syncwarp();
  }

  // balance the "read" barrier: the flow group arrived for every output plane, the magnetic group
  // waited for all but the last two
  if constexpr (GRP == 0)
    for (int o = max(zb, ze - 2); o < ze; ++o) nbar_sync(kBarCons + (o & 1), S::NT);
}

template <typename T, int RAD, int MODE>
__global__ void __launch_bounds__(SCfg<T, RAD>::NT, 1)
    zsplit_kernel(const __grid_constant__ TmapSet tm, const __grid_constant__ Fields<T> out,
                  const __grid_constant__ Geom g, Region r, const __grid_constant__ Coef<T> C, int k,
                  T* __restrict__ rhs_out, int nzc, int xo) {
  using Z = ZCfg<T, RAD>;
  using S = SCfg<T, RAD>;
  constexpr int TX = Z::TX, NC = Z::NT, NSLOT = S::NSLOT;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  T* const ring = reinterpret_cast<T*>(smem_raw);
  T* const prevbuf = ring + NSLOT * Z::SLOT;
  uint64_t* const full = reinterpret_cast<uint64_t*>(prevbuf + 2 * NF * Z::PSZ);
  uint64_t* const empty = full + NSLOT;
  unsigned* const tslot = reinterpret_cast<unsigned*>(empty + NSLOT);

  const int tid = (int)threadIdx.x;
  const int grp = tid >= NC;  // 0: magnetic (A, lnrho), 1: flow (u, s)
  const int ct = tid - grp * NC;
  const int warp = tid >> 5, lane = tid & 31;
  const int gw = ct >> 5;  // warp within the group; warps gw and gw + 8 share a TMEM lane quadrant

  if (tid == 0) {
    if (smem_u32(smem_raw) & 127) __trap();
    for (int s = 0; s < NSLOT; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], S::NWARP);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;\n" ::"r"(smem_u32(tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  // exchange columns of this thread: lane quadrant gw % 4, column group gw / 4 (2 kXV columns),
  // plus 4 kXV columns for odd planes
  const unsigned tq = *tslot + ((unsigned)((gw & 3) * 32) << 16) + (unsigned)((gw >> 2) * 2 * kXV);

  SCtx<T, RAD, MODE> X;
  const int zs0 = (int)blockIdx.z * nzc;
  const int x0 = r.lo[0] + (int)blockIdx.x * TX;
  X.ring = ring;
  X.prevbuf = prevbuf;
  X.full = full;
  X.empty = empty;
  X.tm = &tm;
  X.out = &out;
  X.g = &g;
  X.C = &C;
  X.k = k;
  X.xo = xo;
  X.rhs_out = rhs_out;
  X.x0 = x0;
  X.y0 = r.lo[1] + (int)blockIdx.y * Z::TY;
  X.zb = r.lo[2] + zs0;
  X.ze = X.zb + min(nzc, r.ext[2] - zs0);
  X.first = X.zb - RAD;
  X.last = X.ze + RAD - 1;
  X.xs = (x0 - RAD) & ~(Z::CH - 1);
  X.pxs = x0 & ~(Z::CH - 1);
  X.need_prev = MODE == 0 && k > 0;
  {
    const int cx = x0 + ct % TX, cy = X.y0 + ct / TX;
    X.active = cx < r.lo[0] + r.ext[0] && cy < r.lo[1] + r.ext[1];
  }

  if (tid == NC)  // the producer: first thread of the flow group (the last group to release a plane)
    for (int P = X.first; P <= X.last && P < X.first + NSLOT; ++P) X.issue(P);

  // (setmaxnreg: the group giving registers away decreases first; 128 / 128 needs none)
  if (grp == 0) {
    if constexpr (S::NT == 512 && B2_ZS_REG_MAG < 128)
      asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" ::"n"(B2_ZS_REG_MAG));
    if constexpr (S::NT == 512 && B2_ZS_REG_MAG > 128)
      asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;\n" ::"n"(B2_ZS_REG_MAG));
    group_march<T, RAD, MODE, 0>(X, ct, lane, tq);
  } else {
    if constexpr (S::NT == 512 && B2_ZS_REG_FLOW > 128)
      asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;\n" ::"n"(B2_ZS_REG_FLOW));
    if constexpr (S::NT == 512 && B2_ZS_REG_FLOW < 128)
      asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" ::"n"(B2_ZS_REG_FLOW));
    group_march<T, RAD, MODE, 1>(X, ct, lane, tq);
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;\n" ::"r"(*tslot));
  }
}

template <typename T, int RAD, int MODE>
void launch_cfg(cudaStream_t st, const TmapSet& tm, const Fields<T>& out, const Geom& g, const Region& r,
                const Coef<T>& C, int k, T* rhs_out, int xo, int zchunk) {
  using Z = ZCfg<T, RAD>;
  using S = SCfg<T, RAD>;
  static bool attr[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (!attr[dev & 63]) {
    cudaFuncSetAttribute(zsplit_kernel<T, RAD, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)S::SMEM);
    attr[dev & 63] = true;
  }
  const int cz = zchunk > 0 ? zchunk : zm::kNZC;
  const int nzc = r.ext[2] < cz ? r.ext[2] : cz;
  dim3 grd((r.ext[0] + Z::TX - 1) / Z::TX, (r.ext[1] + Z::TY - 1) / Z::TY, (r.ext[2] + nzc - 1) / nzc);
  zsplit_kernel<T, RAD, MODE><<<grd, S::NT, S::SMEM, st>>>(tm, out, g, r, C, k, rhs_out, nzc, xo);
}

}  // namespace zs

template <typename T, int RAD>
bool zsplit_supported(const Geom& g, const Region& r) {
  return zs::SCfg<T, RAD>::OK && zmarch_supported<T, RAD>(g, r);
}

template <typename T, int RAD>
void launch_zsplit(cudaStream_t st, const TmapSet& tm, const Fields<T>& out, const Geom& g, const Region& r,
                   const Coef<T>& C, int k, T* rhs_out, int xo, int zchunk) {
  if constexpr (zs::SCfg<T, RAD>::OK) {
    if (rhs_out)
      zs::launch_cfg<T, RAD, 1>(st, tm, out, g, r, C, k, rhs_out, xo, zchunk);
    else
      zs::launch_cfg<T, RAD, 0>(st, tm, out, g, r, C, k, nullptr, xo, zchunk);
  }
}

#define B2_ZSPLIT_INSTANTIATE(T, RAD)                                                                     \
  template bool zsplit_supported<T, RAD>(const Geom&, const Region&);                                      \
  template void launch_zsplit<T, RAD>(cudaStream_t, const TmapSet&, const Fields<T>&, const Geom&, const Region&, \
                                      const Coef<T>&, int, T*, int, int);

}  // namespace b2
