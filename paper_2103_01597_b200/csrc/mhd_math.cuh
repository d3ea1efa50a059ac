// Per-cell arithmetic of the fused MHD substep: 6th-order derivatives in a fixed
// canonical order, the RHS of Eqs. B.1-B.4 and the
// Williamson 2N RK3 update.  Every update kernel (direct, z-marching,
// inner/outer) evaluates exactly these operations in exactly this order, so a
// cell's result is bit-identical whichever kernel or decomposition computed it.
//
// The library is compiled with -fmad=false: every fused multiply-add below is an
// explicit fma(), nothing is contracted behind our back.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace b2 {

constexpr int R = 3;     // default stencil radius (Eq. 1); 6th order, k = 2r
constexpr int RMAX = 4;  // orders 2, 4, 6, 8
constexpr int NF = 8;  // lnrho, ux, uy, uz, s, Ax, Ay, Az (Table B.1; order R#14)
enum { LNRHO = 0, UX = 1, UY = 2, UZ = 3, SS = 4, AX = 5, AY = 6, AZ = 7 };

// Coefficients of one mesh, passed by value as a kernel parameter.
// Stencil weights (readings R#1, R#2) of order 2r are pre-divided by the grid spacing; at r = 3:
// c = (3/4, -3/20, 1/60), d = (3/2, -3/20, 1/90), centre -49/18, e = d / 4 = (270, -27, 2)/720.
template <typename T>
struct Coef {
  T c1[3][RMAX];  // [axis][i-1]: first derivative  c_i / ds_a
  T d2[3][RMAX];  // [axis][i-1]: second derivative d_i / ds_a^2
  T d0[3];        // [axis]:      centre weight    c_0 / ds_a^2
  T xw[3][RMAX];  // [pair][i-1]: cross derivative e_i / (ds_a ds_b); pairs 0 = (x,y), 1 = (x,z), 2 = (y,z)
  // physics (Table B.2; EOS reading R#5, conduction R#6)
  T gamma_cp, gm1, inv_cp, lnrho0, cs0sq, inv_T0, H_C, eta_inv_mu0, inv_mu0, nu, nu3, two_nu, zeta, eta, K;
  // RK3 update: f_{k+1} = f_k + rkA[k] (f_k - f_{k-1}) + rkB[k] RHS  (R#3, R#4)
  T rkA[3], rkB[3];
  // (x, y) pairs of the in-plane weights, for paired FP32x2 evaluation of the x and y axes
  alignas(2 * sizeof(T)) T xy_c1[RMAX][2];
  alignas(2 * sizeof(T)) T xy_d2[RMAX][2];
  alignas(2 * sizeof(T)) T xy_d0[2];
};

// All derivative quantities one cell needs.
template <typename T>
struct Derivs {
  T f[NF];
  T gl[3], gs[3];      // grad lnrho, grad s
  T gu[3][3];          // gu[i][j] = d u_i / d x_j
  T gA[3][3];          // gA[i][j] = d A_i / d x_j (i != j used)
  T lapl, laps;        // Laplacians of lnrho and s
  T d2u[3][3];         // d2u[i][j] = d^2 u_i / d x_j^2
  T d2A[3][3];
  T xu[3], xA[3];      // (grad div v)_i - d^2 v_i / d x_i^2 : the cross-derivative part
};

template <typename T> __device__ __forceinline__ T fma_(T a, T b, T c);
template <> __device__ __forceinline__ double fma_<double>(double a, double b, double c) { return fma(a, b, c); }
template <> __device__ __forceinline__ float fma_<float>(float a, float b, float c) { return fmaf(a, b, c); }
template <typename T> __device__ __forceinline__ T exp_(T x);
template <> __device__ __forceinline__ double exp_<double>(double x) { return exp(x); }
template <> __device__ __forceinline__ float exp_<float>(float x) { return expf(x); }

#ifdef __CUDACC__
// Two FP32 cells evaluated together (the FP32 z-marching kernel gives each thread two cells of a
// column): every arithmetic operation is one sm_100a FP32x2 instruction (FFMA2 / FADD2 / FMUL2)
// whose lanes round exactly as the scalar FP32 instruction, so each lane's result is bit-identical
// to the scalar kernels' (R#19).
struct alignas(8) F2 {
  float2 v;
  F2() = default;
  __host__ __device__ explicit F2(double c) : v(make_float2((float)c, (float)c)) {}
  __host__ __device__ F2(float a, float b) : v(make_float2(a, b)) {}
};
__device__ __forceinline__ F2 mk2(float2 a) {
  F2 r;
  r.v = a;
  return r;
}
__device__ __forceinline__ F2 operator+(F2 a, F2 b) { return mk2(__fadd2_rn(a.v, b.v)); }
__device__ __forceinline__ F2 operator-(F2 a, F2 b) { return mk2(__fadd2_rn(a.v, make_float2(-b.v.x, -b.v.y))); }
// The product is an FFMA2 with an addend of -0 that the compiler cannot see (b2_f2_nz, set to
// (-0, -0) by the launcher; a*b + -0 == a*b exactly): the CUDA 12.9 compiler contracts an FP32x2
// multiply followed by an add into FFMA2 even with -fmad=false and explicit .rn (also at the PTX
// level), which would round differently from the scalar kernels.
static __constant__ float2 b2_f2_nz;
__device__ __forceinline__ F2 operator*(F2 a, F2 b) { return mk2(__ffma2_rn(a.v, b.v, b2_f2_nz)); }
__device__ __forceinline__ F2 operator/(F2 a, F2 b) { return F2(a.v.x / b.v.x, a.v.y / b.v.y); }
__device__ __forceinline__ F2 operator-(F2 a) { return F2(-a.v.x, -a.v.y); }
template <> __device__ __forceinline__ F2 fma_<F2>(F2 a, F2 b, F2 c) { return mk2(__ffma2_rn(a.v, b.v, c.v)); }
template <> __device__ __forceinline__ F2 exp_<F2>(F2 x) { return F2(expf(x.v.x), expf(x.v.y)); }
#endif

// ---- canonical operator forms -------------------------------------------------------------
// D1 along an axis from the differences  Dl_i = f(+i) - f(-i), i = 1..RAD
template <typename T, int RAD>
__device__ __forceinline__ T d1_of(const T (&dl)[RAD], const T* c) {
  T acc = c[0] * dl[0];
#pragma unroll
  for (int i = 1; i < RAD; ++i) acc = fma_(c[i], dl[i], acc);
  return acc;
}
// D2 along an axis from the sums  Sg_i = f(+i) + f(-i)  and the centre value
template <typename T, int RAD>
__device__ __forceinline__ T d2_of(T f0, const T (&sg)[RAD], const T* d, T d0) {
  T acc = d0 * f0;
#pragma unroll
  for (int i = 0; i < RAD; ++i) acc = fma_(d[i], sg[i], acc);
  return acc;
}

// Accessor-driven gather of every derivative, in the canonical order.
// V(q, dx, dy, dz) returns field q at the cell offset (dx, dy, dz).
//
// Cross derivatives (reading R#2; Eq. 14 point set):
//   d_a d_b f = sum_{k=-r..r, k!=0} sgn(k) e_|k| / (ds_a ds_b) * Dl^a_|k|(f at +k e_b),
// accumulated in increasing k (the z-marching kernel accumulates plane by plane in this
// same order).  The graddiv cross parts are
//   x_0 = d_x d_z v_z  (+ d_x d_y v_y inserted at k = 0)
//   x_1 = d_y d_z v_z  (+ d_x d_y v_x inserted at k = 0)
//   x_2 = d_x d_z v_x and d_y d_z v_y interleaved per k.
template <typename T, int RAD, class Acc>
__device__ __forceinline__ void axis_pair(const Acc& V, int q, int a, const Coef<T>& C, T f0, T& d1, T& d2) {
  const int ox = a == 0, oy = a == 1, oz = a == 2;
  T dl[RAD], sg[RAD];
#pragma unroll
  for (int i = 1; i <= RAD; ++i) {
    const T p = V(q, i * ox, i * oy, i * oz), m = V(q, -i * ox, -i * oy, -i * oz);
    dl[i - 1] = p - m;
    sg[i - 1] = p + m;
  }
  d1 = d1_of<T, RAD>(dl, C.c1[a]);
  d2 = d2_of<T, RAD>(f0, sg, C.d2[a], C.d0[a]);
}

// in-plane d_x d_y of field q (a = x, b = y), k = -r..r in increasing order
template <typename T, int RAD, class Acc>
__device__ __forceinline__ T cross_xy(const Acc& V, int q, const Coef<T>& C) {
  const T* w = C.xw[0];
  T acc = (-w[RAD - 1]) * (V(q, RAD, -RAD, 0) - V(q, -RAD, -RAD, 0));
#pragma unroll
  for (int k = -RAD + 1; k <= RAD; ++k) {
    if (k == 0) continue;
    const int i = k < 0 ? -k : k;
    acc = fma_(k < 0 ? -w[i - 1] : w[i - 1], V(q, i, k, 0) - V(q, -i, k, 0), acc);
  }
  return acc;
}

// Term of a z-cross at plane offset k (k != 0): Dl^a_|k|(f at +k e_z), a = 0 (x) or 1 (y)
template <typename T, class Acc>
__device__ __forceinline__ T zdelta(const Acc& V, int q, int a, int k) {
  const int i = k < 0 ? -k : k;
  return a == 0 ? V(q, i, 0, k) - V(q, -i, 0, k) : V(q, 0, i, k) - V(q, 0, -i, k);
}
template <typename T>
__device__ __forceinline__ T zweight(const Coef<T>& C, int pair, int k) {
  return k < 0 ? -C.xw[pair][-k - 1] : C.xw[pair][k - 1];
}

template <typename T, int RAD, class Acc>
__device__ __forceinline__ void cross_parts(const Acc& V, int qx, int qy, int qz, const Coef<T>& C, T x[3]) {
  const T P0 = cross_xy<T, RAD>(V, qy, C);  // d_x d_y v_y
  const T P1 = cross_xy<T, RAD>(V, qx, C);  // d_x d_y v_x
  T a0 = zweight(C, 1, -RAD) * zdelta<T>(V, qz, 0, -RAD);
  T a1 = zweight(C, 2, -RAD) * zdelta<T>(V, qz, 1, -RAD);
  T a2 = zweight(C, 1, -RAD) * zdelta<T>(V, qx, 0, -RAD);
  a2 = fma_(zweight(C, 2, -RAD), zdelta<T>(V, qy, 1, -RAD), a2);
#pragma unroll
  for (int k = -RAD + 1; k <= RAD; ++k) {
    if (k == 0) {
      a0 = a0 + P0;
      a1 = a1 + P1;
      continue;
    }
    a0 = fma_(zweight(C, 1, k), zdelta<T>(V, qz, 0, k), a0);
    a1 = fma_(zweight(C, 2, k), zdelta<T>(V, qz, 1, k), a1);
    a2 = fma_(zweight(C, 1, k), zdelta<T>(V, qx, 0, k), a2);
    a2 = fma_(zweight(C, 2, k), zdelta<T>(V, qy, 1, k), a2);
  }
  x[0] = a0;
  x[1] = a1;
  x[2] = a2;
}

template <typename T, int RAD, class Acc>
__device__ __forceinline__ void gather(const Acc& V, const Coef<T>& C, Derivs<T>& D) {
#pragma unroll
  for (int q = 0; q < NF; ++q) D.f[q] = V(q, 0, 0, 0);
  // lnrho and s: first derivatives and Laplacian (axis points only)
  {
    T d2x, d2y, d2z;
    axis_pair<T, RAD>(V, LNRHO, 0, C, D.f[LNRHO], D.gl[0], d2x);
    axis_pair<T, RAD>(V, LNRHO, 1, C, D.f[LNRHO], D.gl[1], d2y);
    axis_pair<T, RAD>(V, LNRHO, 2, C, D.f[LNRHO], D.gl[2], d2z);
    D.lapl = (d2x + d2y) + d2z;
    axis_pair<T, RAD>(V, SS, 0, C, D.f[SS], D.gs[0], d2x);
    axis_pair<T, RAD>(V, SS, 1, C, D.f[SS], D.gs[1], d2y);
    axis_pair<T, RAD>(V, SS, 2, C, D.f[SS], D.gs[2], d2z);
    D.laps = (d2x + d2y) + d2z;
  }
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      axis_pair<T, RAD>(V, UX + i, a, C, D.f[UX + i], D.gu[i][a], D.d2u[i][a]);
      axis_pair<T, RAD>(V, AX + i, a, C, D.f[AX + i], D.gA[i][a], D.d2A[i][a]);
    }
  cross_parts<T, RAD>(V, UX, UY, UZ, C, D.xu);
  cross_parts<T, RAD>(V, AX, AY, AZ, C, D.xA);
}

// ---- RHS of Eqs. B.1-B.4 -------------------------------------------------------
// j = mu0^-1 (grad div A - lap A) (R#7); S traceless rate of shear (R#9); the rho in
// 2 rho nu S:S and zeta rho (div u)^2 cancels against 1/(rho T).
// Split in stages so a kernel may contract the magnetic derivatives as soon as they exist;
// every kernel evaluates the same expressions, so values are identical wherever they run.
template <typename T>
struct MagPart {
  T B[3], J[3], lapA[3];  // B = curl A, J = mu0 j, lap A
};

template <typename T>
__device__ __forceinline__ MagPart<T> mag_part(const T (&gA)[3][3], const T (&d2A)[3][3], const T (&xA)[3]) {
  MagPart<T> m;
  m.B[0] = gA[2][1] - gA[1][2];
  m.B[1] = gA[0][2] - gA[2][0];
  m.B[2] = gA[1][0] - gA[0][1];
  // mu0 j = grad div A - lap A  (the d^2 A_i / dx_i^2 terms cancel exactly)
  m.J[0] = xA[0] - (d2A[0][1] + d2A[0][2]);
  m.J[1] = xA[1] - (d2A[1][0] + d2A[1][2]);
  m.J[2] = xA[2] - (d2A[2][0] + d2A[2][1]);
#pragma unroll
  for (int i = 0; i < 3; ++i) m.lapA[i] = (d2A[i][0] + d2A[i][1]) + d2A[i][2];
  return m;
}

// (B.4) dA/dt = u x B + eta lap A
template <typename T>
__device__ __forceinline__ void rhs_induction(const T (&u)[3], const MagPart<T>& m, const Coef<T>& C, T out[NF]) {
  const T u0 = u[0], u1 = u[1], u2 = u[2];
  const T B0 = m.B[0], B1 = m.B[1], B2 = m.B[2];
  out[AX] = fma_(C.eta, m.lapA[0], u1 * B2 - u2 * B1);
  out[AY] = fma_(C.eta, m.lapA[1], u2 * B0 - u0 * B2);
  out[AZ] = fma_(C.eta, m.lapA[2], u0 * B1 - u1 * B0);
}

// Pointwise thermodynamic and magnetic factors of the cell (no derivative of u or s): the
// equation of state (R#5), the Lorentz acceleration rho^-1 mu0^-1 (mu0 j) x B of B.2 and the ohmic
// heating of B.3 per unit rho T.  The warp-specialised kernel evaluates these in its magnetic
// warp group and hands them over; every kernel uses this same split, so results stay bit-identical.
template <typename T>
struct Thermo {
  T L[3];      // (j x B) / rho
  T ohm;       // (H - C + eta mu0 j^2) / rho
  T inv_rho;   // 1 / rho
  T cs2;       // c_s^2
  T inv_T;     // 1 / T
};

template <typename T>
__device__ __forceinline__ Thermo<T> thermo(T lnrho, T s, const MagPart<T>& m, const Coef<T>& C) {
  Thermo<T> t;
  const T B0 = m.B[0], B1 = m.B[1], B2 = m.B[2];
  const T J0 = m.J[0], J1 = m.J[1], J2 = m.J[2];
  // equation of state (R#5): theta = lnT - lnT0
  const T theta = fma_(C.gamma_cp, s, C.gm1 * (lnrho - C.lnrho0));
  t.inv_rho = exp_(-lnrho);
  const T eth = exp_(theta);
  t.cs2 = C.cs0sq * eth;
  t.inv_T = C.inv_T0 / eth;
  const T lor = t.inv_rho * C.inv_mu0;
  t.L[0] = lor * (J1 * B2 - J2 * B1);
  t.L[1] = lor * (J2 * B0 - J0 * B2);
  t.L[2] = lor * (J0 * B1 - J1 * B0);
  const T J2s = fma_(J2, J2, fma_(J1, J1, J0 * J0));
  t.ohm = fma_(C.eta_inv_mu0, J2s, C.H_C) * t.inv_rho;
  return t;
}

// (B.1)-(B.3): lnrho, u, s.  u is the cell value; lapu_i = lap u_i, gdu_i = (grad div u)_i.
template <typename T>
__device__ __forceinline__ void rhs_flow(const T (&u)[3], const T (&gl)[3], const T (&gs)[3], const T (&gu)[3][3],
                                         T lapl, T laps, const T (&lapu)[3], const T (&gdu)[3], const Thermo<T>& t,
                                         const Coef<T>& C, T out[NF]) {
  const T u0 = u[0], u1 = u[1], u2 = u[2];
  const T divu = (gu[0][0] + gu[1][1]) + gu[2][2];

  // (B.1) d lnrho/dt = -u.grad lnrho - div u
  out[LNRHO] = -fma_(u2, gl[2], fma_(u1, gl[1], u0 * gl[0])) - divu;

  // traceless rate of shear
  const T divu3 = divu * (T)(1.0 / 3.0);
  T S[3][3];
  S[0][0] = gu[0][0] - divu3;
  S[1][1] = gu[1][1] - divu3;
  S[2][2] = gu[2][2] - divu3;
  S[0][1] = S[1][0] = (T)0.5 * (gu[0][1] + gu[1][0]);
  S[0][2] = S[2][0] = (T)0.5 * (gu[0][2] + gu[2][0]);
  S[1][2] = S[2][1] = (T)0.5 * (gu[1][2] + gu[2][1]);

  // (B.2) momentum
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    const T adv = fma_(u2, gu[i][2], fma_(u1, gu[i][1], u0 * gu[i][0]));
    const T pg = fma_(gs[i], C.inv_cp, gl[i]);
    const T sgl = fma_(S[i][2], gl[2], fma_(S[i][1], gl[1], S[i][0] * gl[0]));
    // nu (lap u + 1/3 grad div u + 2 S.grad lnrho) + zeta grad div u
    const T visc = fma_(C.nu, lapu[i], fma_(C.two_nu, sgl, fma_(C.nu3, gdu[i], C.zeta * gdu[i])));
    out[UX + i] = t.L[i] + fma_(-t.cs2, pg, visc - adv);
  }

  // (B.3) entropy: -u.grad s + [H - C + eta mu0 j^2]/(rho T) + [2 nu S:S + zeta (div u)^2]/T
  //                + K/rho (lap theta + |grad theta|^2)
  T SS2 = S[0][0] * S[0][0];
  SS2 = fma_(S[1][1], S[1][1], SS2);
  SS2 = fma_(S[2][2], S[2][2], SS2);
  T off = S[0][1] * S[0][1];
  off = fma_(S[0][2], S[0][2], off);
  off = fma_(S[1][2], S[1][2], off);
  SS2 = fma_((T)2, off, SS2);
  const T gth0 = fma_(C.gamma_cp, gs[0], C.gm1 * gl[0]);
  const T gth1 = fma_(C.gamma_cp, gs[1], C.gm1 * gl[1]);
  const T gth2 = fma_(C.gamma_cp, gs[2], C.gm1 * gl[2]);
  const T lapth = fma_(C.gamma_cp, laps, C.gm1 * lapl);
  const T cond = C.K * t.inv_rho * fma_(gth2, gth2, fma_(gth1, gth1, fma_(gth0, gth0, lapth)));
  const T visch = fma_(C.two_nu, SS2, C.zeta * divu * divu);
  const T udgs = fma_(u2, gs[2], fma_(u1, gs[1], u0 * gs[0]));
  out[SS] = fma_(t.ohm + visch, t.inv_T, cond - udgs);
}

// The viscous contractions of the u derivatives: lap u_i and (grad div u)_i = d_ii u_i + x_i.
template <typename T>
__device__ __forceinline__ void visc_parts(const T (&d2u)[3][3], const T (&xu)[3], T (&lapu)[3], T (&gdu)[3]) {
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    lapu[i] = (d2u[i][0] + d2u[i][1]) + d2u[i][2];
    gdu[i] = d2u[i][i] + xu[i];
  }
}

// Everything but the magnetic contraction.  u, lnrho, s are the cell values.
template <typename T>
__device__ __forceinline__ void rhs_rest(T lnrho, T s, const T (&u)[3], const T (&gl)[3], const T (&gs)[3],
                                         const T (&gu)[3][3], T lapl, T laps, const T (&d2u)[3][3], const T (&xu)[3],
                                         const MagPart<T>& m, const Coef<T>& C, T out[NF]) {
  T lapu[3], gdu[3];
  visc_parts<T>(d2u, xu, lapu, gdu);
  const Thermo<T> t = thermo<T>(lnrho, s, m, C);
  rhs_flow<T>(u, gl, gs, gu, lapl, laps, lapu, gdu, t, C, out);
  rhs_induction<T>(u, m, C, out);
}

template <typename T>
__device__ __forceinline__ void rhs_cell(const Derivs<T>& D, const Coef<T>& C, T out[NF]) {
  const MagPart<T> m = mag_part<T>(D.gA, D.d2A, D.xA);
  const T u[3] = {D.f[UX], D.f[UY], D.f[UZ]};
  rhs_rest<T>(D.f[LNRHO], D.f[SS], u, D.gl, D.gs, D.gu, D.lapl, D.laps, D.d2u, D.xu, m, C, out);
}

// Williamson 2N RK3 with w reconstructed from two stored states (R#3, R#4):
//   k = 0:  f1 = f0 + beta_0 dt RHS
//   k > 0:  f_{k+1} = f_k + (beta_k alpha_k / beta_{k-1}) (f_k - f_{k-1}) + beta_k dt RHS
template <typename T>
__device__ __forceinline__ T rk_update(int k, T fk, T fprev, T rhs, const Coef<T>& C) {
  const T t = fma_(C.rkB[k], rhs, fk);
  return k == 0 ? t : fma_(C.rkA[k], fk - fprev, t);
}

}  // namespace b2
