/*
 * ORACLE — TEST INFRASTRUCTURE ONLY.
 *
 * A plain, slow, obviously-correct CPU implementation of one RK3 step of the
 * non-ideal compressible MHD system of arXiv 2103.01597 (Pekkilä et al.),
 * Appendix B, on a periodic 3-D grid with 6th-order central differences.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline leg and
 * --impl reference) may load this library.  It shares no code, header, table
 * or constant with the CUDA path under paper_2103_01597_b200/; neither side
 * includes or imports the other.
 *
 * Precision: `real` is double by default; compiled again with
 * -DORACLE_LONG_DOUBLE to bound the oracle's own rounding.
 *
 * Citations are PAPER.md line numbers (P:n) plus the section / equation;
 * readings of passages where the paper is silent are listed in DESIGN.md
 * ("Readings") and referenced here as R#n.
 *
 *   Grid, halo, radius r ............ P:108-112 (Eq. 1), P:194-211 (Eqs. 2-3)
 *   Periodic halo map s' = ((s-r) mod n') + r ... P:705 (§3.3)
 *   Stencil point set (axes + in-plane diagonals) P:832-836 (Eq. 14)
 *   central differences, order 2r ... P:829-830 (§4); weights R#1, R#2
 *   RK3, Williamson 2N storage ...... P:830 (§4); coefficients R#3
 *   MHD equations B.1-B.4 ........... P:1092-1111 (App. B); EOS R#5, R#6
 *
 * Layout: each field is an array of (nz+2r)(ny+2r)(nx+2r) values, x fastest,
 * with a halo of r cells on every side; "interior" arrays are nz*ny*nx,
 * x fastest.  Field order: lnrho, ux, uy, uz, s, Ax, Ay, Az (R#14).
 * The radius r = 1, 2, 3, 4 selects 2nd-, 4th-, 6th- or 8th-order central
 * differences ("2nd-, 4th-, 6th-, and 8th-order"; k = 2r).
 */
#include <math.h>
#include <stdlib.h>
#include <string.h>
#include <stddef.h>

#ifdef ORACLE_LONG_DOUBLE
typedef long double real;
#define EXP expl
#else
typedef double real;
#define EXP exp
#endif

#define RMAX 4       /* largest stencil radius: 8th order (k = 2r) */
#define NF 8         /* eight scalar fields, Table B.1 */

enum { LNRHO = 0, UX, UY, UZ, SS, AX, AY, AZ };

typedef struct {
  double nu, zeta, eta, mu0, cs0, cp, gamma, K, H, C, lnrho0, lnT0;
} oracle_params;

/* ---- grid indexing (M = N + 2r per axis) ---------------------- */
typedef struct { int nx, ny, nz, r; } dims3;

static size_t gidx(dims3 d, int x, int y, int z) {
  /* x, y, z are halo-inclusive coordinates in [0, n+2r) */
  return ((size_t)z * (size_t)(d.ny + 2 * d.r) + (size_t)y) * (size_t)(d.nx + 2 * d.r) + (size_t)x;
}

size_t oracle_grid_cells(int nx, int ny, int nz, int r) {
  return (size_t)(nx + 2 * r) * (size_t)(ny + 2 * r) * (size_t)(nz + 2 * r);
}

/* ---- periodic halo (s'_i = ((s_i - r) mod n'_i) + r; P:418 periodic) -
 * Every halo cell, sides, edges and corners alike, takes the value of the
 * interior cell at the wrapped index along each axis. */
static int wrap(int s, int n, int r) { int m = (s - r) % n; if (m < 0) m += n; return m + r; }

void oracle_periodic_fill(real* f, int nx, int ny, int nz, int r) {
  dims3 d = {nx, ny, nz, r};
  for (int z = 0; z < nz + 2 * r; ++z)
    for (int y = 0; y < ny + 2 * r; ++y)
      for (int x = 0; x < nx + 2 * r; ++x) {
        int inside = x >= r && x < nx + r && y >= r && y < ny + r && z >= r && z < nz + r;
        if (!inside) f[gidx(d, x, y, z)] = f[gidx(d, wrap(x, nx, r), wrap(y, ny, r), wrap(z, nz, r))];
      }
}

/* ---- central differences of order 2r (weights R#1, R#2) --------
 * First derivative:  D1 f = sum_i c_i (f(+i) - f(-i)) / ds
 * Second derivative: D2 f = sum_i d_i ((f(+i) - f0) + (f(-i) - f0)) / ds^2   (difference form)
 * Cross derivative:  DX f = sum_i e_i (f(+i,+i) + f(-i,-i) - f(+i,-i) - f(-i,+i)) / (da db),
 *                    e_i = d_i / 4, using only the in-plane diagonal points z(x +- y) of
 *                    Eq. 14.  Textbook central-difference weights, i = 1..r:
 *   r = 1: c = (1/2)                         d = (1)
 *   r = 2: c = (2/3, -1/12)                  d = (4/3, -1/12)
 *   r = 3: c = (3/4, -3/20, 1/60)            d = (3/2, -3/20, 1/90)
 *   r = 4: c = (4/5, -1/5, 4/105, -1/280)    d = (8/5, -1/5, 8/315, -1/560) */
static const real C1T[RMAX + 1][RMAX + 1] = {
    {0},
    {0, (real)1 / 2},
    {0, (real)2 / 3, -(real)1 / 12},
    {0, (real)3 / 4, -(real)3 / 20, (real)1 / 60},
    {0, (real)4 / 5, -(real)1 / 5, (real)4 / 105, -(real)1 / 280}};
static const real C2T[RMAX + 1][RMAX + 1] = {
    {0},
    {0, 1},
    {0, (real)4 / 3, -(real)1 / 12},
    {0, (real)3 / 2, -(real)3 / 20, (real)1 / 90},
    {0, (real)8 / 5, -(real)1 / 5, (real)8 / 315, -(real)1 / 560}};

typedef struct { const real* f; dims3 d; } fieldv;

static real at(fieldv g, int x, int y, int z) { return g.f[gidx(g.d, x, y, z)]; }

static void axis_step(int axis, int i, int* dx, int* dy, int* dz) {
  *dx = axis == 0 ? i : 0; *dy = axis == 1 ? i : 0; *dz = axis == 2 ? i : 0;
}

static real d1(fieldv g, int x, int y, int z, int axis, const double ds[3]) {
  real acc = 0;
  for (int i = 1; i <= g.d.r; ++i) {
    int a, b, c; axis_step(axis, i, &a, &b, &c);
    acc += C1T[g.d.r][i] * (at(g, x + a, y + b, z + c) - at(g, x - a, y - b, z - c));
  }
  return acc / (real)ds[axis];
}

static real d2(fieldv g, int x, int y, int z, int axis, const double ds[3]) {
  real f0 = at(g, x, y, z), acc = 0;
  for (int i = 1; i <= g.d.r; ++i) {
    int a, b, c; axis_step(axis, i, &a, &b, &c);
    acc += C2T[g.d.r][i] * ((at(g, x + a, y + b, z + c) - f0) + (at(g, x - a, y - b, z - c) - f0));
  }
  return acc / ((real)ds[axis] * (real)ds[axis]);
}

static real dx2(fieldv g, int x, int y, int z, int ax1, int ax2, const double ds[3]) {
  real acc = 0;
  for (int i = 1; i <= g.d.r; ++i) {
    int a1, b1, c1, a2, b2, c2;
    axis_step(ax1, i, &a1, &b1, &c1);
    axis_step(ax2, i, &a2, &b2, &c2);
    real pp = at(g, x + a1 + a2, y + b1 + b2, z + c1 + c2);
    real mm = at(g, x - a1 - a2, y - b1 - b2, z - c1 - c2);
    real pm = at(g, x + a1 - a2, y + b1 - b2, z + c1 - c2);
    real mp = at(g, x - a1 + a2, y - b1 + b2, z - c1 + c2);
    acc += C2T[g.d.r][i] / 4 * (pp + mm - pm - mp);
  }
  return acc / ((real)ds[ax1] * (real)ds[ax2]);
}

/* Second derivative d^2/(da db): D2 on the diagonal a == b, DX otherwise. */
static real dd(fieldv g, int x, int y, int z, int a, int b, const double ds[3]) {
  return a == b ? d2(g, x, y, z, a, ds) : dx2(g, x, y, z, a, b, ds);
}

/* Operator on a halo-filled field, evaluated at every interior cell.
 * op: 1 = D1 along a1; 2 = D2 along a1; 3 = cross derivative (a1, a2). */
void oracle_apply_op(const real* f, int nx, int ny, int nz, int r, const double ds[3],
                     int op, int a1, int a2, real* out) {
  dims3 d = {nx, ny, nz, r};
  const int R = r;
  fieldv g = {f, d};
  for (int z = 0; z < nz; ++z)
    for (int y = 0; y < ny; ++y)
      for (int x = 0; x < nx; ++x) {
        real v;
        if (op == 1) v = d1(g, x + R, y + R, z + R, a1, ds);
        else if (op == 2) v = d2(g, x + R, y + R, z + R, a1, ds);
        else v = dx2(g, x + R, y + R, z + R, a1, a2, ds);
        out[((size_t)z * ny + y) * nx + x] = v;
      }
}

/* ---- right-hand side, Appendix B, Eqs. B.1-B.4 --------------
 * Evaluated at one interior cell (halo-inclusive coordinates x, y, z) of the
 * halo-filled fields f[0..7].  Writes the 8 time derivatives to out[0..7]. */
static void rhs_cell(fieldv g[NF], int x, int y, int z, const double ds[3],
                     const oracle_params* p, real out[NF]) {
  const int U[3] = {UX, UY, UZ}, A[3] = {AX, AY, AZ};

  real lnrho = at(g[LNRHO], x, y, z), s = at(g[SS], x, y, z);
  real u[3], Av[3];
  for (int i = 0; i < 3; ++i) { u[i] = at(g[U[i]], x, y, z); Av[i] = at(g[A[i]], x, y, z); }

  /* first derivatives: grad lnrho, grad s, du_i/dx_j, dA_i/dx_j */
  real glnrho[3], gs[3], gu[3][3], gA[3][3];
  for (int j = 0; j < 3; ++j) {
    glnrho[j] = d1(g[LNRHO], x, y, z, j, ds);
    gs[j] = d1(g[SS], x, y, z, j, ds);
    for (int i = 0; i < 3; ++i) {
      gu[i][j] = d1(g[U[i]], x, y, z, j, ds);
      gA[i][j] = d1(g[A[i]], x, y, z, j, ds);
    }
  }

  /* Laplacians (Table B.2 "Laplace operator") */
  real lap_lnrho = 0, lap_s = 0, lap_u[3] = {0, 0, 0}, lap_A[3] = {0, 0, 0};
  for (int j = 0; j < 3; ++j) {
    lap_lnrho += d2(g[LNRHO], x, y, z, j, ds);
    lap_s += d2(g[SS], x, y, z, j, ds);
    for (int i = 0; i < 3; ++i) {
      lap_u[i] += d2(g[U[i]], x, y, z, j, ds);
      lap_A[i] += d2(g[A[i]], x, y, z, j, ds);
    }
  }

  /* grad(div v)_i = sum_j d^2 v_j / (dx_i dx_j) — uses only the Eq. 14 points */
  real graddiv_u[3] = {0, 0, 0}, graddiv_A[3] = {0, 0, 0};
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) {
      graddiv_u[i] += dd(g[U[j]], x, y, z, i, j, ds);
      graddiv_A[i] += dd(g[A[j]], x, y, z, i, j, ds);
    }

  real divu = gu[0][0] + gu[1][1] + gu[2][2];

  /* B = curl A (Table B.2) */
  real B[3] = {gA[2][1] - gA[1][2], gA[0][2] - gA[2][0], gA[1][0] - gA[0][1]};
  /* j = mu0^-1 curl B = mu0^-1 (grad div A - lap A)  (Table B.2; reading R#7) */
  real jv[3];
  for (int i = 0; i < 3; ++i) jv[i] = (graddiv_A[i] - lap_A[i]) / (real)p->mu0;

  /* Traceless rate-of-shear tensor S (Table B.2; reading R#9) */
  real S[3][3];
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j)
      S[i][j] = (real)0.5 * (gu[i][j] + gu[j][i]) - (i == j ? divu / 3 : 0);

  /* Equation of state (reading R#5): lnT = lnT0 + gamma s/cp + (gamma-1)(lnrho - lnrho0),
   * cs^2 = cs0^2 T/T0 */
  real gamma = (real)p->gamma, cp = (real)p->cp;
  real theta = gamma * s / cp + (gamma - 1) * (lnrho - (real)p->lnrho0);
  real rho = EXP(lnrho);
  real T = EXP((real)p->lnT0 + theta);
  real cs2 = (real)p->cs0 * (real)p->cs0 * EXP(theta);

  /* (B.1) D lnrho / Dt = -div u,  D/Dt = d/dt + u.grad (Table B.2) */
  real udotglnrho = u[0] * glnrho[0] + u[1] * glnrho[1] + u[2] * glnrho[2];
  out[LNRHO] = -udotglnrho - divu;

  /* (B.2) Du/Dt = -cs^2 grad(s/cp + lnrho) + j x B / rho
   *               + nu [lap u + 1/3 grad div u + 2 S.grad lnrho] + zeta grad div u */
  real jxB[3] = {jv[1] * B[2] - jv[2] * B[1], jv[2] * B[0] - jv[0] * B[2], jv[0] * B[1] - jv[1] * B[0]};
  for (int i = 0; i < 3; ++i) {
    real adv = u[0] * gu[i][0] + u[1] * gu[i][1] + u[2] * gu[i][2];
    real Sglnrho = S[i][0] * glnrho[0] + S[i][1] * glnrho[1] + S[i][2] * glnrho[2];
    out[U[i]] = -adv
              - cs2 * (gs[i] / cp + glnrho[i])
              + jxB[i] / rho
              + (real)p->nu * (lap_u[i] + graddiv_u[i] / 3 + 2 * Sglnrho)
              + (real)p->zeta * graddiv_u[i];
  }

  /* (B.3) rho T Ds/Dt = H - C + div(K grad T) + eta mu0 j^2 + 2 rho nu S:S + zeta rho (div u)^2
   * with div(K grad T)/(rho T) = (K/rho)(lap lnT + |grad lnT|^2)  (reading R#6) */
  real SS2 = 0;
  for (int i = 0; i < 3; ++i) for (int j = 0; j < 3; ++j) SS2 += S[i][j] * S[i][j];
  real j2 = jv[0] * jv[0] + jv[1] * jv[1] + jv[2] * jv[2];
  real gtheta[3];
  for (int i = 0; i < 3; ++i) gtheta[i] = gamma / cp * gs[i] + (gamma - 1) * glnrho[i];
  real lap_theta = gamma / cp * lap_s + (gamma - 1) * lap_lnrho;
  real gtheta2 = gtheta[0] * gtheta[0] + gtheta[1] * gtheta[1] + gtheta[2] * gtheta[2];
  real udotgs = u[0] * gs[0] + u[1] * gs[1] + u[2] * gs[2];
  real heat = (real)p->H - (real)p->C + (real)p->eta * (real)p->mu0 * j2
            + 2 * rho * (real)p->nu * SS2 + (real)p->zeta * rho * divu * divu;
  out[SS] = -udotgs + heat / (rho * T) + (real)p->K / rho * (lap_theta + gtheta2);

  /* (B.4) dA/dt = u x B + eta lap A */
  real uxB[3] = {u[1] * B[2] - u[2] * B[1], u[2] * B[0] - u[0] * B[2], u[0] * B[1] - u[1] * B[0]};
  for (int i = 0; i < 3; ++i) out[A[i]] = uxB[i] + (real)p->eta * lap_A[i];
}

/* RHS at every interior cell.  f: 8 halo-filled fields; rhs: 8 interior arrays. */
void oracle_rhs(real* const f[NF], int nx, int ny, int nz, int r, const double ds[3],
                const oracle_params* p, real* const rhs[NF]) {
  dims3 d = {nx, ny, nz, r};
  const int R = r;
  fieldv g[NF];
  for (int k = 0; k < NF; ++k) { g[k].f = f[k]; g[k].d = d; }
#pragma omp parallel for schedule(static)
  for (int z = 0; z < nz; ++z)
    for (int y = 0; y < ny; ++y)
      for (int x = 0; x < nx; ++x) {
        real out[NF];
        rhs_cell(g, x + R, y + R, z + R, ds, p, out);
        for (int k = 0; k < NF; ++k) rhs[k][((size_t)z * ny + y) * nx + x] = out[k];
      }
}

/* ---- Williamson (1980) 2N-storage RK3 (coefficients reading R#3) ----
 *   w <- alpha_k w + dt * RHS(f);   f <- f + beta_k w,   k = 0, 1, 2 */
static const real RK_ALPHA[3] = {0, -(real)5 / 9, -(real)153 / 128};
static const real RK_BETA[3] = {(real)1 / 3, (real)15 / 16, (real)8 / 15};

void oracle_rk3_update(real* f, real* w, const real* rhs, size_t n, int k, double dt) {
  for (size_t i = 0; i < n; ++i) {
    w[i] = RK_ALPHA[k] * w[i] + (real)dt * rhs[i];
    f[i] = f[i] + RK_BETA[k] * w[i];
  }
}

/* The same RK3 update applied to y' = lambda y (a pin on the coefficients:
 * one step must equal R(lambda dt) y with R(z) = 1 + z + z^2/2 + z^3/6). */
void oracle_rk3_linear(real* y, size_t n, double lambda, double dt, int nsteps) {
  real* w = (real*)calloc(n, sizeof(real));
  real* rhs = (real*)malloc(n * sizeof(real));
  for (int s = 0; s < nsteps; ++s)
    for (int k = 0; k < 3; ++k) {
      for (size_t i = 0; i < n; ++i) rhs[i] = (real)lambda * y[i];
      oracle_rk3_update(y, w, rhs, n, k, dt);
    }
  free(w); free(rhs);
}

/* The same 2N scheme in the two-state form of reading R#4 (the form the GPU path stores): with
 * w_k = (f_{k+1} - f_k) / beta_k eliminated,
 *   f_{k+1} = f_k + (beta_k alpha_k / beta_{k-1}) (f_k - f_{k-1}) + beta_k dt RHS(f_k),
 * evaluated as t = fma(beta_k dt, RHS, f_k); f_{k+1} = fma(beta_k alpha_k / beta_{k-1}, f_k - f_{k-1}, t).
 * Algebraically identical to oracle_rk3_update (R(z) pinned in tests); it differs only in rounding,
 * and exists to attribute the last ulps of the GPU/oracle difference to the form. */
#ifdef ORACLE_LONG_DOUBLE
#define FMA fmal
#else
#define FMA fma
#endif
void oracle_rk3_update_w2(real* f, real* fprev, const real* rhs, size_t n, int k, double dt) {
  const real b = (real)((double)RK_BETA[k] * dt);
  const real a = k == 0 ? 0 : (real)((double)RK_BETA[k] * (double)RK_ALPHA[k] / (double)RK_BETA[k - 1]);
  for (size_t i = 0; i < n; ++i) {
    const real t = FMA(b, rhs[i], f[i]);
    const real fn = k == 0 ? t : FMA(a, f[i] - fprev[i], t);
    fprev[i] = f[i];
    f[i] = fn;
  }
}

/* ---- one full integration: nsteps RK3 steps of the MHD system --------------
 * state: 8 interior arrays (nz*ny*nx, x fastest), updated in place.
 * stop_substep: if >= 0, stop after that many substeps in total (for substep-level
 * parity), else run 3*nsteps substeps.
 * rhs_out: optional 8 interior arrays receiving the RHS of the last substep run. */
static int integrate_form(real* const state[NF], int nx, int ny, int nz, int r, const double ds[3],
                          const oracle_params* p, double dt, int nsteps, int stop_substep,
                          real* const rhs_out[NF], int form) {
  size_t ncell = (size_t)nx * ny * nz, ngrid = oracle_grid_cells(nx, ny, nz, r);
  dims3 d = {nx, ny, nz, r};
  const int R = r;
  real* f[NF]; real* w[NF]; real* rhs[NF];
  for (int k = 0; k < NF; ++k) {
    f[k] = (real*)calloc(ngrid, sizeof(real));
    w[k] = (real*)calloc(ncell, sizeof(real));   /* w = 0 at the start of a step */
    rhs[k] = (real*)malloc(ncell * sizeof(real));
    if (!f[k] || !w[k] || !rhs[k]) return -1;
  }
  int total = stop_substep >= 0 ? stop_substep : 3 * nsteps;
  for (int sub = 0; sub < total; ++sub) {
    int k = sub % 3;
    for (int q = 0; q < NF; ++q) {
      for (int z = 0; z < nz; ++z)
        for (int y = 0; y < ny; ++y)
          memcpy(&f[q][gidx(d, R, y + R, z + R)], &state[q][((size_t)z * ny + y) * nx], nx * sizeof(real));
      oracle_periodic_fill(f[q], nx, ny, nz, r);     /* halo exchange */
    }
    oracle_rhs(f, nx, ny, nz, r, ds, p, rhs);          /* all cells before any update */
    for (int q = 0; q < NF; ++q) {
      if (form == 0)
        oracle_rk3_update(state[q], w[q], rhs[q], ncell, k, dt);
      else  /* w holds f_{k-1} in the two-state form */
        oracle_rk3_update_w2(state[q], w[q], rhs[q], ncell, k, dt);
    }
  }
  if (rhs_out)
    for (int q = 0; q < NF; ++q) memcpy(rhs_out[q], rhs[q], ncell * sizeof(real));
  for (int k = 0; k < NF; ++k) { free(f[k]); free(w[k]); free(rhs[k]); }
  return 0;
}

int oracle_integrate(real* const state[NF], int nx, int ny, int nz, int r, const double ds[3],
                     const oracle_params* p, double dt, int nsteps, int stop_substep,
                     real* const rhs_out[NF]) {
  return integrate_form(state, nx, ny, nz, r, ds, p, dt, nsteps, stop_substep, rhs_out, 0);
}
/* The same integration with the two-state RK3 form of R#4 (oracle_rk3_update_w2). */
int oracle_integrate_w2(real* const state[NF], int nx, int ny, int nz, int r, const double ds[3],
                        const oracle_params* p, double dt, int nsteps, int stop_substep,
                        real* const rhs_out[NF]) {
  return integrate_form(state, nx, ny, nz, r, ds, p, dt, nsteps, stop_substep, rhs_out, 1);
}

/* RHS of an interior state (periodic), without any update: the `debug_rhs` check. */
int oracle_rhs_of_state(real* const state[NF], int nx, int ny, int nz, int r, const double ds[3],
                        const oracle_params* p, real* const rhs_out[NF]) {
  size_t ngrid = oracle_grid_cells(nx, ny, nz, r);
  dims3 d = {nx, ny, nz, r};
  const int R = r;
  real* f[NF];
  for (int q = 0; q < NF; ++q) {
    f[q] = (real*)calloc(ngrid, sizeof(real));
    if (!f[q]) return -1;
    for (int z = 0; z < nz; ++z)
      for (int y = 0; y < ny; ++y)
        memcpy(&f[q][gidx(d, R, y + R, z + R)], &state[q][((size_t)z * ny + y) * nx], nx * sizeof(real));
    oracle_periodic_fill(f[q], nx, ny, nz, r);
  }
  oracle_rhs(f, nx, ny, nz, r, ds, p, rhs_out);
  for (int q = 0; q < NF; ++q) free(f[q]);
  return 0;
}

int oracle_real_bytes(void) { return (int)sizeof(real); }

/* OpenMP thread count of oracle_rhs (per-cell results do not depend on it). */
#ifdef _OPENMP
#include <omp.h>
void oracle_set_threads(int n) { omp_set_num_threads(n); }
int oracle_get_threads(void) { return omp_get_max_threads(); }
#else
void oracle_set_threads(int n) { (void)n; }
int oracle_get_threads(void) { return 1; }
#endif
