// z-marching update kernel: the hot path on sm_100a (template; instantiated per dtype and
// stencil radius by zmarch_<dtype>_r<r>.cu).
//
// A CTA owns a TX x TY column of cells and marches it along z over a chunk of planes.
//  * Staging: each plane (8 fields, tile + radius-r halo in x and y) is fetched by TMA
//    (cp.async.bulk.tensor.3d, one elected thread, mbarrier completion) into an (r + 2)-slot
//    shared-memory ring, one plane ahead of the computation; f_{k-1} of the output plane
//    (read pointwise by the RK3 update) rides in the same transaction.  One CTA barrier per
//    plane protects slot reuse (a barrier-free variant with per-slot release counters measured
//    3 % slower: profiles/r01/).
//  * In-plane derivatives (x, y axes and the d_x d_y diagonals of Eq. 14) are read
//    from the slot of the output plane o; the z column of every field comes from registers
//    (planes o-r..o-1) and from the ring (o+1..o+r).
//  * The d_x d_z / d_y d_z cross terms are split: the k < 0 half is PUSHED from each plane into
//    register accumulators of the next three outputs, reusing that plane's own x/y differences;
//    the k > 0 half is PULLED from the ring.  This reproduces mhd_math.cuh::cross_parts term by
//    term, so the result is bit-identical to the direct kernel
//    (tests/test_gpu_parity.py::test_kernel_variants_bit_identical).
//  * Fields are processed one vector at a time (A, then u, then lnrho and s) and the magnetic
//    derivatives are contracted to B, mu0 j and lap A as soon as they exist, to keep the live
//    register set small.  The march is unrolled by r so the register history rotates by
//    renaming, not by moves.
#pragma once
#include <algorithm>

#include "kernels.h"

namespace b2 {
namespace zm {

__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];\n" ::"r"(
          smem_u32(dst)),
      "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
      : "memory");
}

// Warp-group skew (ZCfg::SKEW): the CTA's upper half of rows (the "leading" group) runs half an
// iteration ahead of the lower half, so that one group's load-heavy derivative phase overlaps the
// other's load-free RHS phase instead of both hitting the shared-memory pipe at once.  Two named
// barriers (alternating by plane parity) replace the per-plane CTA barrier; the lagging group
// refills the ring.  Measured (256^3, one B200): +15 % for the FP64 order-8 kernel (32x4 tile,
// 4 warps per SM); slower with 8 warps per SM (-12 % FP64 / -17 % FP32 at order 6, -15 % FP32 at
// order 8), so only the 4-row tiles use it.
__device__ __forceinline__ void bar_sync(int id, int count) {
  asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(count) : "memory");
}
__device__ __forceinline__ void bar_arrive(int id, int count) {
  asm volatile("bar.arrive %0, %1;\n" ::"r"(id), "r"(count) : "memory");
}

// B2_ZM_NEXT=1 (build option): the centres of plane o + 1, loaded from the ring as the first z taps
// of output o, are kept in registers and reused as the centres of output o + 1 (8 LDS per cell
// fewer, 252 instead of 240 registers).  One GPU: 13.36 vs 13.30 Gcell/s; 4 GPUs weak: 47.7-49.9
// vs 50.6 (the boundary slabs and the inner launch interleave worse), so it is off
// (profiles/r02/next_*, mgpu/next_*).
// FP32: the x and y axes of axis_xy evaluated as FP32x2 pairs (FFMA2 / FADD2)
#ifndef B2_ZM_F32_XY2
#define B2_ZM_F32_XY2 1
#endif
#ifndef B2_ZM_SKEW_ALL
#define B2_ZM_SKEW_ALL 0  // build option: the warp-group skew on every tile (measured slower at 8 warps)
#endif
#ifndef B2_ZM_NEXT
#define B2_ZM_NEXT 0
#endif
#ifndef B2_ZM_F32_CPT
#define B2_ZM_F32_CPT 1
#endif
template <int CPT, typename T>
struct ZVal {
  using type = T;
};
template <>
struct ZVal<2, float> {
  using type = F2;
};

template <typename T, int RAD>
struct ZCfg {
  static constexpr int TX = zm_tx<T>(), TY = zm_ty<T, RAD>();
  static constexpr int ES = (int)sizeof(T);
  static constexpr int COLS = zm_cols<T, RAD>();
  static constexpr int ROWS = zm_rows<T, RAD>();
  static constexpr int FSZ = (ROWS * COLS * ES + 127) / 128 * 128 / ES;  // 128-B aligned TMA destinations
  static constexpr int SLOT = NF * FSZ;
  // r + 2 slots: planes o..o+r in use while o+r+1 streams in.  One CTA per SM (a 16x8 FP64 tile at
  // two CTAs per SM and a 2-CTA FP32 variant both measured slower: profiles/r01/).
  static constexpr int NSLOT = RAD + 2;
  // cells per thread.  B2_ZM_F32_CPT=2 (build option): FP32 threads own two cells of a column
  // (rows y and y + RS of the tile) and evaluate both with FP32x2 instructions (FFMA2 / FADD2,
  // mhd_math.cuh::F2), bit-identical to the scalar kernels; -31 % instructions, but at 246
  // registers only 8 warps fit and the kernel is latency bound: 22.8 vs 24.6 Gcell/s at 256^3
  // (profiles/r02/f32_*), so the default is one cell per thread (16 warps)
  static constexpr int CPT = sizeof(T) == 4 && RAD <= 3 ? B2_ZM_F32_CPT : 1;
  static constexpr int RS = TY / CPT;
  static constexpr int NT = TX * TY / CPT;
  static constexpr int CH = zm_ch<T>();
  static constexpr int PCOLS = zm_pcols<T>();
  static constexpr int PSZ = (TY * PCOLS * ES + 127) / 128 * 128 / ES;  // f_{k-1} tile per field
  static constexpr unsigned HALO_TX = (unsigned)(NF * ROWS * COLS * ES);
  static constexpr unsigned PREV_TX = (unsigned)(NF * TY * PCOLS * ES);
  static constexpr size_t SMEM = (size_t)(NSLOT * SLOT + 2 * NF * PSZ) * ES + 128 + 16;
  static constexpr bool FITS = SMEM <= 227 * 1024;
  static constexpr bool SKEW = TY < 8 || B2_ZM_SKEW_ALL;  // the 4-row tiles (FP64, r = 4)
  using V = typename ZVal<CPT, T>::type;  // compute type: T, or two FP32 cells (F2)
};

// lane c of a compute value (the cell in row y + c RS of a two-cell FP32 thread)
template <typename V>
__device__ __forceinline__ auto lane_of(V v, int c) {
  if constexpr (std::is_same<V, F2>::value)
    return c == 0 ? v.v.x : v.v.y;
  else
    return v;
}

// Register state carried along z by one thread.
template <typename T, int RAD>
struct March {
#if B2_ZM_NEXT
  T nxt[NF];  // centres of plane o + 1, loaded as z taps of output o, reused as the centres of o + 1
#endif
  T hist[NF][RAD];   // f(o-r) .. f(o-1); logical index j at phase PH lives at (j + PH) % r
  T acc[2][RAD][3];  // [u|A][logical output o .. o+r-1 -> physical (j + PH) % r][z-part of x_0, x_1, x_2]
};

template <typename T, int RAD, int MODE>
struct ZStep {
  using Z = ZCfg<T, RAD>;
  using V = typename Z::V;  // compute type (storage type T)
  const T* ring;
  const T* prevbuf;
  const Coef<V>& C;
  int cell;   // offset of this thread's cell inside a field of a slot
  int pcell;  // offset inside a field of the f_{k-1} tile
  int slot0;  // plane zb - r (first staged plane) has slot 0
  bool lead;  // leading warp group (ZCfg::SKEW): signals "past the loads of plane o" mid-iteration

  __device__ __forceinline__ void signal_half(int o) const {
    if (Z::SKEW && lead) bar_arrive(1 + (o & 1), Z::NT);
  }

  __device__ __forceinline__ const T* slot_of(int plane) const {
    return ring + ((plane - slot0) % Z::NSLOT) * Z::SLOT + cell;
  }
  // field q at offset (dx, dy) in a staged plane: this thread's cell, or its two cells (rows y, y + RS)
  static __device__ __forceinline__ V at(const T* sp, int q, int dx, int dy) {
    const T* e = sp + q * Z::FSZ + dy * Z::COLS + dx;
    if constexpr (Z::CPT == 2)
      return V(e[0], e[Z::RS * Z::COLS]);
    else
      return e[0];
  }
  static __device__ __forceinline__ void nxt_store(March<V, RAD>& st, int q, V p) {
#if B2_ZM_NEXT
    st.nxt[q] = p;
#endif
  }
  static __device__ __forceinline__ V at_prev(const T* pv) {
    if constexpr (Z::CPT == 2)
      return V(pv[0], pv[Z::RS * Z::PCOLS]);
    else
      return pv[0];
  }

  // x/y first and second derivatives of field q in the slot, with the differences kept
  __device__ __forceinline__ void axis_xy(const T* sp, int q, V f0, V (&d1)[2], V (&d2)[2], V (&dlx)[RAD],
                                          V (&dly)[RAD]) const {
#if B2_ZM_F32_XY2
    if constexpr (std::is_same<V, float>::value) {
      // FP32: the x and y axes as the two lanes of FP32x2 instructions, each lane the same
      // operations in the same order as d1_of / d2_of (bit-identical to the scalar path)
      float2 dl[RAD], sg[RAD];
#pragma unroll
      for (int i = 1; i <= RAD; ++i) {
        const float2 pp = make_float2(at(sp, q, i, 0), at(sp, q, 0, i));
        const float2 mm = make_float2(at(sp, q, -i, 0), at(sp, q, 0, -i));
        dl[i - 1] = __fadd2_rn(pp, make_float2(-mm.x, -mm.y));
        sg[i - 1] = __fadd2_rn(pp, mm);
        dlx[i - 1] = dl[i - 1].x;
        dly[i - 1] = dl[i - 1].y;
      }
      const float2* c1 = reinterpret_cast<const float2*>(C.xy_c1);
      const float2* dd = reinterpret_cast<const float2*>(C.xy_d2);
      float2 a = __ffma2_rn(c1[0], dl[0], b2_f2_nz);  // the product, opaque to contraction
#pragma unroll
      for (int i = 1; i < RAD; ++i) a = __ffma2_rn(c1[i], dl[i], a);
      float2 b = __ffma2_rn(*reinterpret_cast<const float2*>(C.xy_d0), make_float2(f0, f0), b2_f2_nz);
#pragma unroll
      for (int i = 0; i < RAD; ++i) b = __ffma2_rn(dd[i], sg[i], b);
      d1[0] = a.x;
      d1[1] = a.y;
      d2[0] = b.x;
      d2[1] = b.y;
      return;
    }
#endif
    V sgx[RAD], sgy[RAD];
#pragma unroll
    for (int i = 1; i <= RAD; ++i) {
      const V px = at(sp, q, i, 0), mx = at(sp, q, -i, 0);
      const V py = at(sp, q, 0, i), my = at(sp, q, 0, -i);
      dlx[i - 1] = px - mx;
      sgx[i - 1] = px + mx;
      dly[i - 1] = py - my;
      sgy[i - 1] = py + my;
    }
    d1[0] = d1_of<V, RAD>(dlx, C.c1[0]);
    d2[0] = d2_of<V, RAD>(f0, sgx, C.d2[0], C.d0[0]);
    d1[1] = d1_of<V, RAD>(dly, C.c1[1]);
    d2[1] = d2_of<V, RAD>(f0, sgy, C.d2[1], C.d0[1]);
  }
  // z derivatives from the column: f(o+1..o+r) from the ring, f(o-r..o-1) from registers
  template <int PH>
  __device__ __forceinline__ void axis_z(March<V, RAD>& st, int q, V f0, const T* const (&sk)[RAD + 1], V& d1,
                                         V& d2) const {
    V dl[RAD], sg[RAD];
#pragma unroll
    for (int i = 1; i <= RAD; ++i) {
      const V p = at(sk[i], q, 0, 0), m = st.hist[q][(RAD - i + PH) % RAD];
#if B2_ZM_NEXT
      if (i == 1) nxt_store(st, q, p);
#endif
      dl[i - 1] = p - m;
      sg[i - 1] = p + m;
    }
    d1 = d1_of<V, RAD>(dl, C.c1[2]);
    d2 = d2_of<V, RAD>(f0, sg, C.d2[2], C.d0[2]);
  }
  __device__ __forceinline__ V cross_xy_s(const T* sp, int q) const {
    const V* w = C.xw[0];
    V a = (-w[RAD - 1]) * (at(sp, q, RAD, -RAD) - at(sp, q, -RAD, -RAD));
#pragma unroll
    for (int k = -RAD + 1; k <= RAD; ++k) {
      if (k == 0) continue;
      const int i = k < 0 ? -k : k;
      a = fma_(k < 0 ? -w[i - 1] : w[i - 1], at(sp, q, i, k) - at(sp, q, -i, k), a);
    }
    return a;
  }
  // k < 0 half of the z-cross terms of plane p for vector v: outputs p+j (k = -j, j < r) and a
  // fresh accumulator for p+r (k = -r), which lands in the physical slot of output p.
  template <int PH>
  __device__ __forceinline__ void push(March<V, RAD>& st, int v, const V (&dlx_x)[RAD], const V (&dly_y)[RAD],
                                       const V (&dlx_z)[RAD], const V (&dly_z)[RAD]) const {
    const V* wxz = C.xw[1];
    const V* wyz = C.xw[2];
#pragma unroll
    for (int j = 1; j < RAD; ++j) {
      V* a = st.acc[v][(j + PH) % RAD];
      a[0] = fma_(-wxz[j - 1], dlx_z[j - 1], a[0]);
      a[1] = fma_(-wyz[j - 1], dly_z[j - 1], a[1]);
      a[2] = fma_(-wxz[j - 1], dlx_x[j - 1], a[2]);
      a[2] = fma_(-wyz[j - 1], dly_y[j - 1], a[2]);
    }
    V* f = st.acc[v][(0 + PH) % RAD];
    f[0] = (-wxz[RAD - 1]) * dlx_z[RAD - 1];
    f[1] = (-wyz[RAD - 1]) * dly_z[RAD - 1];
    f[2] = fma_(-wyz[RAD - 1], dly_y[RAD - 1], (-wxz[RAD - 1]) * dlx_x[RAD - 1]);
  }

  // push-only pass over a plane below the chunk (prologue)
  template <int PH>
  __device__ __forceinline__ void push_only(March<V, RAD>& st, int p) const {
    const T* s0 = slot_of(p);
#pragma unroll
    for (int v = 0; v < 2; ++v) {
      const int qx = v == 0 ? UX : AX;
      V dlx_x[RAD], dly_y[RAD], dlx_z[RAD], dly_z[RAD];
#pragma unroll
      for (int i = 1; i <= RAD; ++i) {
        dlx_x[i - 1] = at(s0, qx, i, 0) - at(s0, qx, -i, 0);
        dly_y[i - 1] = at(s0, qx + 1, 0, i) - at(s0, qx + 1, 0, -i);
        dlx_z[i - 1] = at(s0, qx + 2, i, 0) - at(s0, qx + 2, -i, 0);
        dly_z[i - 1] = at(s0, qx + 2, 0, i) - at(s0, qx + 2, 0, -i);
      }
      push<PH>(st, v, dlx_x, dly_y, dlx_z, dly_z);
    }
#pragma unroll
    for (int q = 0; q < NF; ++q) st.hist[q][(0 + PH) % RAD] = at(s0, q, 0, 0);
#if B2_ZM_NEXT
#pragma unroll
    for (int q = 0; q < NF; ++q) st.nxt[q] = at(slot_of(p + 1), q, 0, 0);
#endif
    signal_half(p);
  }

  // Derivatives of one vector field (u or A) at output plane o: first and second derivatives
  // along every axis, the graddiv cross parts, and the push of plane o's differences.
  template <int PH>
  __device__ __forceinline__ void vector_derivs(March<V, RAD>& st, int v, const T* const (&sk)[RAD + 1], V (&f)[3],
                                                V (&g)[3][3], V (&d2)[3][3], V (&x)[3]) const {
    const int qx = v == 0 ? UX : AX;
    const T* s0 = sk[0];
    V dlx[3][RAD], dly[3][RAD];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const int q = qx + c;
      V d1a[2], d2a[2];
#if B2_ZM_NEXT
      f[c] = st.nxt[q];
#else
      f[c] = at(s0, q, 0, 0);
#endif
      axis_xy(s0, q, f[c], d1a, d2a, dlx[c], dly[c]);
      axis_z<PH>(st, q, f[c], sk, g[c][2], d2[c][2]);
      g[c][0] = d1a[0];
      g[c][1] = d1a[1];
      d2[c][0] = d2a[0];
      d2[c][1] = d2a[1];
    }
    // graddiv cross parts: k < 0 (accumulated), + in-plane part at k = 0, then k = 1..r
    const V P0 = cross_xy_s(s0, qx + 1);  // d_x d_y v_y
    const V P1 = cross_xy_s(s0, qx);      // d_x d_y v_x
    const V* a = st.acc[v][(0 + PH) % RAD];
    x[0] = a[0] + P0;
    x[1] = a[1] + P1;
    x[2] = a[2];
    const V* wxz = C.xw[1];
    const V* wyz = C.xw[2];
#pragma unroll
    for (int kk = 1; kk <= RAD; ++kk) {
      const T* s = sk[kk];
      x[0] = fma_(wxz[kk - 1], at(s, qx + 2, kk, 0) - at(s, qx + 2, -kk, 0), x[0]);
      x[1] = fma_(wyz[kk - 1], at(s, qx + 2, 0, kk) - at(s, qx + 2, 0, -kk), x[1]);
      x[2] = fma_(wxz[kk - 1], at(s, qx, kk, 0) - at(s, qx, -kk, 0), x[2]);
      x[2] = fma_(wyz[kk - 1], at(s, qx + 1, 0, kk) - at(s, qx + 1, 0, -kk), x[2]);
    }
    push<PH>(st, v, dlx[0], dly[1], dlx[2], dly[2]);
  }

  template <int PH>
  __device__ __forceinline__ void full(March<V, RAD>& st, int o, const Fields<T>& out, const Geom& g, int k,
                                       const bool (&active)[Z::CPT], int x, int y, T* rhs_out) const {
    const T* sk[RAD + 1];
#pragma unroll
    for (int i = 0; i <= RAD; ++i) sk[i] = slot_of(o + i);
    // magnetic potential: derivatives, then B, mu0 j, lap A right away
    V fA[3], gA[3][3], d2A[3][3], xA[3];
    vector_derivs<PH>(st, 1, sk, fA, gA, d2A, xA);
    const MagPart<V> m = mag_part<V>(gA, d2A, xA);
    // velocity
    V u[3], gu[3][3], d2u[3][3], xu[3];
    vector_derivs<PH>(st, 0, sk, u, gu, d2u, xu);
    signal_half(o);
    // log density and entropy
    V sc[2], gsc[2][3], lap[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int q = h == 0 ? LNRHO : SS;
      V d1a[2], d2a[2], dlx[RAD], dly[RAD], d2z;
#if B2_ZM_NEXT
      sc[h] = st.nxt[q];
#else
      sc[h] = at(sk[0], q, 0, 0);
#endif
      axis_xy(sk[0], q, sc[h], d1a, d2a, dlx, dly);
      axis_z<PH>(st, q, sc[h], sk, gsc[h][2], d2z);
      gsc[h][0] = d1a[0];
      gsc[h][1] = d1a[1];
      lap[h] = (d2a[0] + d2a[1]) + d2z;
    }
    V rhs[NF];
    rhs_rest<V>(sc[0], sc[1], u, gsc[0], gsc[1], gu, lap[0], lap[1], d2u, xu, m, C, rhs);
    const V fk[NF] = {sc[0], u[0], u[1], u[2], sc[1], fA[0], fA[1], fA[2]};
    if (active[0] || (Z::CPT == 2 && active[Z::CPT - 1])) {
      V fn[NF];
      if (MODE == 0) {
        const T* pv = prevbuf + ((o & 1) * NF) * Z::PSZ + pcell;
#pragma unroll
        for (int q = 0; q < NF; ++q) fn[q] = rk_update<V>(k, fk[q], k > 0 ? at_prev(pv + q * Z::PSZ) : (V)0, rhs[q], C);
      }
#pragma unroll
      for (int c = 0; c < Z::CPT; ++c) {
        if (!active[c]) continue;
        const int yc = y + c * Z::RS;
        const long long gidx = (long long)o * g.sz + (long long)yc * g.sy + x;
        if (MODE == 0) {
#pragma unroll
          for (int q = 0; q < NF; ++q) out.f[q][gidx] = lane_of(fn[q], c);
          if (g.xwrap) {
            // periodic x faces of this rank's own halo (x unsplit) written here: the cells
            // in the first / last 32-byte sector of a row also go to the row padding on the other
            // side (whole sectors: the extra cell lands in unused padding).  (Adding the y faces
            // here pushed the kernel to 255 registers with spills: the y rows are copied instead.)
            constexpr int W = 32 / (int)sizeof(T);
            const long long sh = x < W ? (long long)g.nx : (x >= g.nx - W ? -(long long)g.nx : 0);
            if (sh != 0) {
#pragma unroll
              for (int q = 0; q < NF; ++q) out.f[q][gidx + sh] = lane_of(fn[q], c);
            }
          }
        } else {
          const long long n = (long long)g.nx * g.ny * g.nz;
          const long long li = ((long long)o * g.ny + yc) * g.nx + x;
#pragma unroll
          for (int q = 0; q < NF; ++q) rhs_out[q * n + li] = lane_of(rhs[q], c);
        }
      }
    }
#pragma unroll
    for (int q = 0; q < NF; ++q) st.hist[q][(0 + PH) % RAD] = fk[q];
  }
};

template <int N, int PH = 0, class F>
__device__ __forceinline__ void unroll_phases(F&& f, int p, int ze) {
  if constexpr (PH < N) {
    if (p + PH < ze) f(std::integral_constant<int, PH>{}, p + PH);
    unroll_phases<N, PH + 1>(f, p, ze);
  }
}

template <typename T, int RAD, int MODE>
__global__ void __launch_bounds__(ZCfg<T, RAD>::NT, 1)
    zmarch_kernel(const __grid_constant__ TmapSet tm, Fields<T> out, Geom g, Region r,
                  const __grid_constant__ Coef<typename ZCfg<T, RAD>::V> C,
                  int k, T* __restrict__ rhs_out, int nzc, int xo, int persist) {
  using Z = ZCfg<T, RAD>;
  constexpr int TX = Z::TX, TY = Z::TY;
  // Dynamic shared memory starts at the (1024-B aligned) base of the CTA window (no static
  // shared memory in this kernel).  The pointer must stay visibly __shared__ so that the stencil
  // reads compile to LDS, not generic loads.
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  T* const ring = reinterpret_cast<T*>(smem_raw);
  T* const prevbuf = ring + Z::NSLOT * Z::SLOT;
  uint64_t* const mbar = reinterpret_cast<uint64_t*>(prevbuf + 2 * NF * Z::PSZ);

  const int tid = (int)threadIdx.x;
  const int tx = tid % TX, ty = tid / TX;
  const bool need_prev = MODE == 0 && k > 0;
  const bool lead = ty >= TY / 2;

  if (tid == 0) {
    if (smem_u32(smem_raw) & 127) __trap();  // TMA destinations need 128-B alignment
    for (int s = 0; s < Z::NSLOT; ++s) mbar_init(&mbar[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();

  // One segment: the tile column at (x0, y0), output planes [zb, ze).  `base` = planes this CTA
  // staged before the segment: ring slot and mbarrier phase of plane P are those of the running
  // count base + (P - first).
  auto segment = [&](const int x0, const int y0, const int zb, const int ze, const unsigned base) {
    const int x = x0 + tx, y = y0 + ty;
    bool active[Z::CPT];
#pragma unroll
    for (int c = 0; c < Z::CPT; ++c) active[c] = x < r.lo[0] + r.ext[0] && y + c * Z::RS < r.lo[1] + r.ext[1];
    const int first = zb - RAD;
    const int xs = (x0 - RAD) & ~(Z::CH - 1);  // 16-byte aligned box starts (interior origin is 128-B aligned)
    const int pxs = x0 & ~(Z::CH - 1);

    // one TMA transaction per staged plane P: its halo tile, plus f_{k-1} of output plane P - r.
    // Memory coordinates: the pitched field has a halo of r cells (element = interior + r in y, z).
    auto issue = [&](int P) {
      const int s = (int)((base + (unsigned)(P - first)) % Z::NSLOT);
      const int po = P - RAD;
      const bool pv = need_prev && po >= zb && po < ze;
      mbar_expect_tx(&mbar[s], Z::HALO_TX + (pv ? Z::PREV_TX : 0u));
      T* dst = ring + s * Z::SLOT;
      const int pz = !g.zwrap ? P : (P < 0 ? P + g.nz : (P >= g.nz ? P - g.nz : P));
#pragma unroll
      for (int q = 0; q < NF; ++q) tma_load_3d(dst + q * Z::FSZ, &tm.halo[q], &mbar[s], xs + xo, y0, pz + RAD);
      if (pv) {
        T* pd = prevbuf + (po & 1) * NF * Z::PSZ;
#pragma unroll
        for (int q = 0; q < NF; ++q) tma_load_3d(pd + q * Z::PSZ, &tm.prev[q], &mbar[s], pxs + xo, y0 + RAD, po + RAD);
      }
    };
    auto wait_plane = [&](int P) {
      const unsigned rel = base + (unsigned)(P - first);
      mbar_wait(&mbar[rel % Z::NSLOT], (rel / Z::NSLOT) & 1u);
    };

    const ZStep<T, RAD, MODE> S{ring, prevbuf, C, (ty + RAD) * Z::COLS + (x - xs), ty * Z::PCOLS + (x - pxs),
                                        first - (int)(base % Z::NSLOT), lead};
    March<typename Z::V, RAD> st;
#pragma unroll
    for (int v = 0; v < 2; ++v)
#pragma unroll
      for (int j = 0; j < RAD; ++j)
#pragma unroll
        for (int c = 0; c < 3; ++c) st.acc[v][j][c] = (typename Z::V)0;

    if (tid == 0)
      for (int P = first; P <= zb && P <= ze + RAD - 1; ++P) issue(P);
#pragma unroll
    for (int i = 0; i < RAD; ++i) wait_plane(first + i);

    auto iter = [&](auto ph, int p) {
      constexpr int PH = decltype(ph)::value;
      if constexpr (Z::SKEW) {
        // lagging group: wait until the leading group is past the loads of plane p (and so done
        // with plane p - 1), and every lagging thread is done with p - 1; then refill p - 1's slot
        if (!lead) bar_sync(1 + (p & 1), Z::NT);
      } else {
        __syncthreads();  // every thread is done with iteration p - 1: its slot is refilled now
      }
      if (tid == 0 && p + RAD + 1 <= ze + RAD - 1) {
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
        issue(p + RAD + 1);
      }
      wait_plane(p + RAD);  // plane p+r and f_{k-1}(p) have landed
      if (p < zb)
        S.template push_only<PH>(st, p);
      else
        S.template full<PH>(st, p, out, g, k, active, x, y, rhs_out);
    };
#pragma unroll 1
    for (int p = first; p < ze; p += RAD) unroll_phases<RAD>(iter, p, ze);
  };

  // The CTA's work is a range [u, u1) of "column planes": the gx * gy tile columns laid end to
  // end, ez planes each.  Chunked grid: one z chunk of one column per CTA.  Persistent schedule:
  // gridDim.x equal ranges, each spanning a few column segments.
  const int gx = (r.ext[0] + TX - 1) / TX, gy = (r.ext[1] + TY - 1) / TY, ez = r.ext[2];
  long long u, u1;
  if (!persist) {
    const int zs = (int)blockIdx.z * nzc;
    u = ((long long)blockIdx.y * gx + blockIdx.x) * ez + zs;
    u1 = u + min(nzc, ez - zs);
  } else {
    const long long total = (long long)gx * gy * ez;
    const long long len = (total + gridDim.x - 1) / gridDim.x;
    u = (long long)blockIdx.x * len;
    u1 = min(total, u + len);
  }
  unsigned base = 0;
#pragma unroll 1
  while (u < u1) {
    const int col = (int)(u / ez), zs = (int)(u % ez);
    const int zlen = (int)min((long long)(ez - zs), u1 - u);
    segment(r.lo[0] + (col % gx) * TX, r.lo[1] + (col / gx) * TY, r.lo[2] + zs, r.lo[2] + zs + zlen, base);
    base += (unsigned)(zlen + 2 * RAD);
    u += zlen;
    if (u < u1) __syncthreads();  // every thread is done with the ring before the next prologue
  }
}

constexpr int kNZC = 64;

// The coefficients in the kernel's compute type (two-cell FP32: every constant broadcast to both lanes).
template <typename V, typename T>
Coef<V> coef_as(const Coef<T>& c) {
  if constexpr (std::is_same<V, T>::value) {
    return c;
  } else {
    Coef<V> o;
    auto cv = [](T x) { return V((double)x); };
    for (int a = 0; a < 3; ++a) {
      for (int i = 0; i < RMAX; ++i) {
        o.c1[a][i] = cv(c.c1[a][i]);
        o.d2[a][i] = cv(c.d2[a][i]);
        o.xw[a][i] = cv(c.xw[a][i]);
      }
      o.d0[a] = cv(c.d0[a]);
      o.rkA[a] = cv(c.rkA[a]);
      o.rkB[a] = cv(c.rkB[a]);
    }
    for (int i = 0; i < RMAX; ++i)
      for (int a = 0; a < 2; ++a) {
        o.xy_c1[i][a] = cv(c.xy_c1[i][a]);
        o.xy_d2[i][a] = cv(c.xy_d2[i][a]);
      }
    o.xy_d0[0] = cv(c.xy_d0[0]);
    o.xy_d0[1] = cv(c.xy_d0[1]);
#define B2_CV(f) o.f = cv(c.f)
    B2_CV(gamma_cp); B2_CV(gm1); B2_CV(inv_cp); B2_CV(lnrho0); B2_CV(cs0sq); B2_CV(inv_T0); B2_CV(H_C);
    B2_CV(eta_inv_mu0); B2_CV(inv_mu0); B2_CV(nu); B2_CV(nu3); B2_CV(two_nu); B2_CV(zeta); B2_CV(eta); B2_CV(K);
#undef B2_CV
    return o;
  }
}

// z chunk of a whole-grid launch (zchunk < 0): the chunk count per tile column that minimises
// (waves of `resident` CTAs) x (planes per CTA, the 2r prologue planes counted at half cost), so
// that the last wave is not left mostly empty.  E.g. 256^3 FP64 (256 columns, 148 resident CTAs):
// 4 chunks of 64 (6.9 waves); FP32 (128 columns of the 32 x 16 tile): 8 chunks of 32 (6.9 waves)
// instead of 4 of 64 (3.5 waves: the fourth wave half empty; measured 24.6 vs 22.3 Gcell/s).
inline int balanced_zchunk(int columns, int nz, int rad, int resident) {
  double best = 1e300;
  int arg = std::min(nz, kNZC);
  for (int c = 1; c <= nz; ++c) {
    const int len = (nz + c - 1) / c;
    if (len < 2 * rad || len > 4 * kNZC) continue;
    const long long ctas = (long long)columns * ((nz + len - 1) / len);
    const long long waves = (ctas + resident - 1) / resident;
    const double t = (double)waves * (len + rad);
    if (t < best - 1e-9) {
      best = t;
      arg = len;
    }
  }
  return arg;
}

template <typename T, int RAD, int MODE>
void launch_cfg(cudaStream_t st, const TmapSet& tm, const Fields<T>& out, const Geom& g, const Region& r,
                const Coef<T>& C, int k, T* rhs_out, int xo, bool persist, int zchunk) {
  using Z = ZCfg<T, RAD>;
  // CTAs of this instantiation that fit on the GPU at once, per device (one process may drive several
  // devices: mhd_group_*); the >48 KB dynamic shared memory attribute is set on each device's first use
  static int resident_of[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  int& resident = resident_of[dev & 63];
  if (!resident) {
    if constexpr (sizeof(T) == 4) {
      const float2 nz = make_float2(-0.0f, -0.0f);  // the opaque addend of FP32x2 products (mhd_math.cuh)
      cudaMemcpyToSymbol(b2_f2_nz, &nz, sizeof(nz));
    }
    cudaFuncSetAttribute(zmarch_kernel<T, RAD, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)Z::SMEM);
    int sms = 0, per = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, zmarch_kernel<T, RAD, MODE>, Z::NT, Z::SMEM);
    resident = std::max(1, sms * std::max(1, per));
  }
  const int cz = zchunk > 0 ? zchunk : (zchunk < 0 ? balanced_zchunk((r.ext[0] + Z::TX - 1) / Z::TX *
                                                                      ((r.ext[1] + Z::TY - 1) / Z::TY),
                                                                  r.ext[2], RAD, resident)
                                                 : kNZC);
  const int nzc = r.ext[2] < cz ? r.ext[2] : cz;
  dim3 grd((r.ext[0] + Z::TX - 1) / Z::TX, (r.ext[1] + Z::TY - 1) / Z::TY, (r.ext[2] + nzc - 1) / nzc);
  // persistent schedule when the chunked grid would take more than one wave (and the warp-group
  // skew, whose barrier ids follow the plane parity, is off)
  const bool pers = persist && !Z::SKEW && (long long)grd.x * grd.y * grd.z > resident;
  if (pers) grd = dim3(resident, 1, 1);
  zmarch_kernel<T, RAD, MODE>
      <<<grd, Z::NT, Z::SMEM, st>>>(tm, out, g, r, coef_as<typename Z::V>(C), k, rhs_out, nzc, xo, pers ? 1 : 0);
}

}  // namespace zm

template <typename T, int RAD>
bool zmarch_supported(const Geom& g, const Region& r) {
  (void)g;
  return zm::ZCfg<T, RAD>::FITS && r.ext[0] >= 16 && r.ext[1] >= 4 && r.ext[2] >= 1;
}

template <typename T, int RAD>
void launch_zmarch(cudaStream_t st, const TmapSet& tm, const Fields<T>& out, const Geom& g, const Region& r,
                   const Coef<T>& C, int k, T* rhs_out, int xo, bool persist, int zchunk) {
  if constexpr (zm::ZCfg<T, RAD>::FITS) {
    if (rhs_out)
      zm::launch_cfg<T, RAD, 1>(st, tm, out, g, r, C, k, rhs_out, xo, persist, zchunk);
    else
      zm::launch_cfg<T, RAD, 0>(st, tm, out, g, r, C, k, nullptr, xo, persist, zchunk);
  }
}

#define B2_ZMARCH_INSTANTIATE(T, RAD)                                                                      \
  template bool zmarch_supported<T, RAD>(const Geom&, const Region&);                                       \
  template void launch_zmarch<T, RAD>(cudaStream_t, const TmapSet&, const Fields<T>&, const Geom&, const Region&, \
                                      const Coef<T>&, int, T*, int, bool, int);

}  // namespace b2
