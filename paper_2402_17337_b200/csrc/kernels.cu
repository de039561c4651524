// sm_100a fp64 kernels of the IBM fractional-step hot path.
//
// Arithmetic contract (reading R13): compiled with --fmad=false;
// every expression keeps the parenthesisation written in DESIGN.md §3 so the
// results are bit-identical to the CPU oracle; IEEE division and sqrt; no
// transcendental functions on the device (sin/cos are evaluated on the host).
//
// Citations: P:NN = PAPER.md line NN, S:NN = SPEC.md line NN.
#include <cstdint>

#include "ibm_internal.h"

namespace ibm {

__device__ __forceinline__ double ld(const double *__restrict__ p, const Geo &g, int i, int jl) {
  if (i < 0 || i >= g.ni || jl < -kGhost || jl >= g.nj + kGhost) return 0.0;
  return __ldg(p + g.off(i, jl));
}

__device__ __forceinline__ double2 ld2(const double *__restrict__ p, const Geo &g, int i, int jl) {
  double2 r = make_double2(0.0, 0.0);
  if (jl < -kGhost || jl >= g.nj + kGhost) return r;
  const double *row = p + (long)(jl + kGhost) * g.pitch;
  if (i >= 0 && i + 1 < g.ni) return __ldg(reinterpret_cast<const double2 *>(row + i));
  if (i >= 0 && i < g.ni) r.x = __ldg(row + i);
  if (i + 1 >= 0 && i + 1 < g.ni) r.y = __ldg(row + i + 1);
  return r;
}

// a / b for b > 0, bit-identical to IEEE division: a zero dividend (the common
// case in uniform-flow regions) would send div.rn.f64 down its slow path, so a
// safe 1.0 is divided instead (hidden behind an opaque move, otherwise the
// compiler folds the substitution away) and the exact +-0 = a is selected.
__device__ __forceinline__ double pdiv(double a, double b) {
  const bool zero = (a == 0.0);
  double d = zero ? 1.0 : a;
  asm("mov.b64 %0, %0;" : "+d"(d));
  const double q = d / b;
  return zero ? a : q;
}

// ---------------------------------------------------------------- a1: classification
// Solid = inside the ellipse (boundary inclusive); Forcing = Solid
// with at least one in-range 4-neighbour outside.  Recomputed analytically for the
// neighbours, so one pass; runs over the body envelope box only (R12, R15).
__global__ void k_classify(uint8_t *__restrict__ tag, Geo g, BBox box, const double *__restrict__ xs,
                           const double *__restrict__ ys, double a, double b, double xb, double yb) {
  int i = box.i0 + blockIdx.x * blockDim.x + threadIdx.x;
  int jl = box.j0 + blockIdx.y * blockDim.y + threadIdx.y;
  if (i >= box.i1 || jl >= box.j1) return;
  int gj = g.gj0 + jl;
  auto ins = [&](int ii, int jj) -> bool {
    double dxn = (xs[ii] - xb) / a;
    double dyn = (ys[jj] - yb) / b;
    double s = dxn * dxn + dyn * dyn;
    return s <= 1.0;
  };
  uint8_t t = FLUID;
  if (ins(i, gj)) {
    bool fl = false;
    if (i + 1 < g.ni && !ins(i + 1, gj)) fl = true;
    if (i - 1 >= 0 && !ins(i - 1, gj)) fl = true;
    if (gj + 1 < g.NJ && !ins(i, gj + 1)) fl = true;
    if (gj - 1 >= 0 && !ins(i, gj - 1)) fl = true;
    t = fl ? FORCING : SOLID;
  }
  tag[g.off(i, jl)] = t;
}

// ---------------------------------------------------------------- a5 masks (R16-R18)
__global__ void k_pflags(uint8_t *__restrict__ pf, const uint8_t *__restrict__ tp, const uint8_t *__restrict__ tu,
                         const uint8_t *__restrict__ tv, Geo gp, Geo gu, Geo gv, BBox box, Metric m, int nx,
                         int ny) {
  int i = box.i0 + blockIdx.x * blockDim.x + threadIdx.x;
  int jl = box.j0 + blockIdx.y * blockDim.y + threadIdx.y;
  if (i >= box.i1 || jl >= box.j1) return;
  int gj = gp.gj0 + jl;
  // rows beyond the stored ghost rows: treated as inactive (only the outermost
  // ghost row's flags depend on them, and that row is never updated)
  auto act0 = [&](int ii, int jj) -> bool { return jj >= -kGhost && jj < gp.nj + kGhost && tp[gp.off(ii, jj)] == FLUID; };
  bool a0 = act0(i, jl);
  bool oE = (i + 1 <= nx - 1) && tu[gu.off(i + 1, jl)] == FLUID && a0 && act0(i + 1, jl);
  bool oW = (i >= 1) && tu[gu.off(i, jl)] == FLUID && act0(i - 1, jl) && a0;
  bool oN = (gj + 1 <= ny - 1) && jl + 1 < gv.nj + kGhost && tv[gv.off(i, jl + 1)] == FLUID && a0 && act0(i, jl + 1);
  bool oS = (gj >= 1) && tv[gv.off(i, jl)] == FLUID && act0(i, jl - 1) && a0;
  uint8_t f = 0;
  if (i + 1 <= nx - 1 && !oE) f |= PF_E;
  if (i >= 1 && !oW) f |= PF_W;
  if (gj + 1 <= ny - 1 && !oN) f |= PF_N;
  if (gj >= 1 && !oS) f |= PF_S;
  bool act = a0;
  if (act) {  // R18: zero Poisson diagonal -> inactive
    double aE = oE ? m.cEp[i] : 0.0;
    double aW = oW ? m.cWp[i] : 0.0;
    double aN = oN ? m.cNp[gj] : 0.0;
    double aS = oS ? m.cSp[gj] : 0.0;
    double aP = ((aE + aW) + (aN + aS)) + m.cDp[i];
    if (aP == 0.0) act = false;
  }
  if (!act) f |= PF_INACTIVE;
  pf[gp.off(i, jl)] = f;
}

// ---------------------------------------------------------------- a3: forcing targets
struct BodyNow {
  double a, b, xb, yb, vb;
};

// R14 / R14b: average over E, W, N, S fluid neighbours of the 1-D
// linear extrapolation from the boundary intercept B through the neighbour N
// (through N2 = N + (N - F) when dN < dF), using u^n.
__device__ double forcing_target(const double *__restrict__ x, const uint8_t *__restrict__ tag, const Geo &g,
                                 const BBox &box, int i, int jl, const double *__restrict__ xs,
                                 const double *__restrict__ ys, const BodyNow &B, double uB) {
  const int gj = g.gj0 + jl;
  const double xF = xs[i], yF = ys[gj];
  double sum = 0.0;
  int cnt = 0;
#pragma unroll 1
  for (int d = 0; d < 4; ++d) {
    const int di = (d == 0) ? 1 : (d == 1) ? -1 : 0;
    const int dj = (d == 2) ? 1 : (d == 3) ? -1 : 0;
    int in_ = i + di, jn = gj + dj;
    if (in_ < 0 || jn < 0 || in_ >= g.ni || jn >= g.NJ) continue;
    int jnl = jn - g.gj0;
    uint8_t tn = box.contains(in_, jnl) ? tag[g.off(in_, jnl)] : (uint8_t)FLUID;
    if (tn != FLUID) continue;
    double xN = xs[in_], yN = ys[jn];
    double dF, dN;
    if (d < 2) {
      double eta = (yF - B.yb) / B.b;
      double w = B.a * sqrt(1.0 - eta * eta);
      double xB = di > 0 ? B.xb + w : B.xb - w;
      dF = fabs(xB - xF);
      dN = fabs(xN - xB);
    } else {
      double zeta = (xF - B.xb) / B.a;
      double w = B.b * sqrt(1.0 - zeta * zeta);
      double yB = dj > 0 ? B.yb + w : B.yb - w;
      dF = fabs(yB - yF);
      dN = fabs(yN - yB);
    }
    double uN = x[g.off(in_, jnl)];
    if (dN < dF) {
      int i2 = in_ + di, j2 = jn + dj;
      if (i2 >= 0 && j2 >= 0 && i2 < g.ni && j2 < g.NJ) {
        int j2l = j2 - g.gj0;
        uint8_t t2 = box.contains(i2, j2l) ? tag[g.off(i2, j2l)] : (uint8_t)FLUID;
        if (t2 == FLUID) {
          dN = (d < 2) ? dN + fabs(xs[i2] - xN) : dN + fabs(ys[j2] - yN);
          uN = x[g.off(i2, j2l)];
        }
      }
    }
    sum = sum + (uB - (uN - uB) * (dF / dN));
    cnt = cnt + 1;
  }
  return sum / (double)cnt;
}

// ---------------------------------------------------------------- a2/a3: predictor
struct PredArgs {
  const double *u, *v, *p, *cup, *cvp;
  double *cu, *cv, *ru, *rv, *us, *vs, *fu, *fv;
  const uint8_t *tu, *tv, *pf;
  Geo gu, gv, gp;
  BBox bu, bv, bp;
  Metric m;
  BodyNow B;
  int nx, ny, have_hist;
  double dt, halfnu, nu;
};

// u family: convection, AB2 (R8), grad p^n, explicit half of CN
// (S:245), Helmholtz rhs at Fluid nodes; targets at Forcing nodes, the body
// velocity at Solid nodes, and the momentum forcing f at both (R19, R19b).
__global__ void k_pred_u(PredArgs A) {
  const Geo &g = A.gu;
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  int jl = blockIdx.y * blockDim.y + threadIdx.y;
  if (i >= g.ni || jl >= g.nj) return;
  const long o = g.off(i, jl);
  const int gj = g.gj0 + jl, nx = A.nx, ny = A.ny;
  const double *dx = A.m.dx, *dy = A.m.dy, *hxc = A.m.hxc;
  if (i == 0 || i == nx) {
    A.us[o] = A.u[o];
    A.cu[o] = 0.0;
    A.ru[o] = 0.0;
    return;
  }
  const bool inbox = A.bu.contains(i, jl);
  const uint8_t t = inbox ? A.tu[o] : (uint8_t)FLUID;
  const Geo &gv = A.gv, &gp = A.gp;
  const double *u = A.u, *v = A.v;
  const double uC = ld(u, g, i, jl);
  const double uE = ld(u, g, i + 1, jl), uW = ld(u, g, i - 1, jl);
  const double uN = ld(u, g, i, jl + 1), uS = ld(u, g, i, jl - 1);
  // convection
  double ue = 0.5 * (uC + uE);
  double uw = 0.5 * (uW + uC);
  double tn, ts;
  if (gj == ny - 1) {
    tn = 0.0;
  } else {
    double un = pdiv(dy[gj + 1] * uC + dy[gj] * uN, dy[gj] + dy[gj + 1]);
    double vn = pdiv(dx[i] * ld(v, gv, i - 1, jl + 1) + dx[i - 1] * ld(v, gv, i, jl + 1), dx[i - 1] + dx[i]);
    tn = un * vn;
  }
  if (gj == 0) {
    ts = 0.0;
  } else {
    double us_ = pdiv(dy[gj] * uS + dy[gj - 1] * uC, dy[gj - 1] + dy[gj]);
    double vs_ = pdiv(dx[i] * ld(v, gv, i - 1, jl) + dx[i - 1] * ld(v, gv, i, jl), dx[i - 1] + dx[i]);
    ts = us_ * vs_;
  }
  const double C = pdiv(ue * ue - uw * uw, hxc[i]) + pdiv(tn - ts, dy[gj]);
  const double Cp = A.have_hist ? A.cup[o] : C;
  const double G = pdiv(ld(A.p, gp, i, jl) - ld(A.p, gp, i - 1, jl), hxc[i]);
  const double cE = A.m.cEu[i], cW = A.m.cWu[i], cD = A.m.cDu[i], cN = A.m.cNu[gj], cS = A.m.cSu[gj];
  const double L = ((cE * (uE - uC) + cW * (uW - uC)) + (cN * (uN - uC) + cS * (uS - uC))) - cD * uC;
  A.cu[o] = C;
  if (t == FLUID) {
    // R9b: the pressure gradient acts on open faces only (closed faces are Neumann)
    const double Gf = (A.bp.contains(i, jl) && (A.pf[gp.off(i, jl)] & PF_W)) ? 0.0 : G;
    A.ru[o] = uC + A.dt * ((-(1.5 * C - 0.5 * Cp) - Gf) + A.halfnu * L);
    A.us[o] = uC;
    if (inbox) A.fu[o] = 0.0;
  } else {  // R19b: Forcing -> target, Solid -> body velocity; f recorded at both
    double tgt = (t == FORCING) ? forcing_target(u, A.tu, g, A.bu, i, jl, A.m.xn, A.m.yc, A.B, 0.0) : 0.0;
    double uhat = uC + A.dt * ((-(1.5 * C - 0.5 * Cp) - G) + A.nu * L);
    A.us[o] = tgt;
    A.fu[o] = pdiv(tgt - uhat, A.dt);
    A.ru[o] = 0.0;
  }
}

__global__ void k_pred_v(PredArgs A) {
  const Geo &g = A.gv;
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  int jl = blockIdx.y * blockDim.y + threadIdx.y;
  if (i >= g.ni || jl >= g.nj) return;
  const long o = g.off(i, jl);
  const int gj = g.gj0 + jl, nx = A.nx, ny = A.ny;
  const double *dx = A.m.dx, *dy = A.m.dy, *hyc = A.m.hyc;
  if (gj == 0 || gj == ny) {
    A.vs[o] = A.v[o];
    A.cv[o] = 0.0;
    A.rv[o] = 0.0;
    return;
  }
  const bool inbox = A.bv.contains(i, jl);
  const uint8_t t = inbox ? A.tv[o] : (uint8_t)FLUID;
  const Geo &gu = A.gu, &gp = A.gp;
  const double *u = A.u, *v = A.v;
  const double vC = ld(v, g, i, jl);
  const double vE = ld(v, g, i + 1, jl), vW = ld(v, g, i - 1, jl);
  const double vN = ld(v, g, i, jl + 1), vS = ld(v, g, i, jl - 1);
  double vn = 0.5 * (vC + vN);
  double vs_ = 0.5 * (vS + vC);
  double ue = pdiv(dy[gj] * ld(u, gu, i + 1, jl - 1) + dy[gj - 1] * ld(u, gu, i + 1, jl), dy[gj - 1] + dy[gj]);
  double ve = (i == nx - 1) ? vC : pdiv(dx[i + 1] * vC + dx[i] * vE, dx[i] + dx[i + 1]);
  double te = ue * ve, tw;
  if (i == 0) {
    tw = 0.0;  // inlet corner: u = 1, v = 0
  } else {
    double uw = pdiv(dy[gj] * ld(u, gu, i, jl - 1) + dy[gj - 1] * ld(u, gu, i, jl), dy[gj - 1] + dy[gj]);
    double vw = pdiv(dx[i] * vW + dx[i - 1] * vC, dx[i - 1] + dx[i]);
    tw = uw * vw;
  }
  const double C = pdiv(te - tw, dx[i]) + pdiv(vn * vn - vs_ * vs_, hyc[gj]);
  const double Cp = A.have_hist ? A.cvp[o] : C;
  const double G = pdiv(ld(A.p, gp, i, jl) - ld(A.p, gp, i, jl - 1), hyc[gj]);
  const double cE = A.m.cEv[i], cW = A.m.cWv[i], cD = A.m.cDv[i], cN = A.m.cNv[gj], cS = A.m.cSv[gj];
  const double L = ((cE * (vE - vC) + cW * (vW - vC)) + (cN * (vN - vC) + cS * (vS - vC))) - cD * vC;
  A.cv[o] = C;
  if (t == FLUID) {
    const double Gf = (A.bp.contains(i, jl) && (A.pf[gp.off(i, jl)] & PF_S)) ? 0.0 : G;
    A.rv[o] = vC + A.dt * ((-(1.5 * C - 0.5 * Cp) - Gf) + A.halfnu * L);
    A.vs[o] = vC;
    if (inbox) A.fv[o] = 0.0;
  } else {  // R19b
    double tgt = (t == FORCING) ? forcing_target(v, A.tv, g, A.bv, i, jl, A.m.xc, A.m.yn, A.B, A.B.vb) : A.B.vb;
    double vhat = vC + A.dt * ((-(1.5 * C - 0.5 * Cp) - G) + A.nu * L);
    A.vs[o] = tgt;
    A.fv[o] = pdiv(tgt - vhat, A.dt);
    A.rv[o] = 0.0;
  }
}

// ---------------------------------------------------------------- outlet fill (R10b)
// u*_{nx} = u*_{nx-1} - dx_{nx-1} (v*_N - v*_S)/dy: discrete continuity of the last
// cell column (the v* halo row is exchanged before this kernel on slabs).
__global__ void k_outlet_fill(double *__restrict__ us, const double *__restrict__ vs, Geo gu, Geo gv, Metric m,
                              int nx) {
  int jl = blockIdx.x * blockDim.x + threadIdx.x;
  if (jl >= gu.nj) return;
  const int gj = gu.gj0 + jl;
  us[gu.off(nx, jl)] = us[gu.off(nx - 1, jl)] -
                       m.dx[nx - 1] * pdiv(vs[gv.off(nx - 1, jl + 1)] - vs[gv.off(nx - 1, jl)], m.dy[gj]);
}

// ---------------------------------------------------------------- a5: Poisson rhs and q
// S:269-277, R16: rhs = D_open(u*)/dt with domain-boundary faces always
// counted; q = closed-face flux / V; b = -rhs; phi := 0 on inactive cells (R17).
__global__ void k_prhs(const double *__restrict__ us, const double *__restrict__ vs, double *__restrict__ bp,
                       double *__restrict__ q, double *__restrict__ phi0, const uint8_t *__restrict__ pf, Geo gp,
                       Geo gu, Geo gv, BBox box, Metric m, int nx, int ny, double dt) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  int jl = blockIdx.y * blockDim.y + threadIdx.y;
  if (i >= gp.ni || jl >= gp.nj) return;
  const long o = gp.off(i, jl);
  const int gj = gp.gj0 + jl;
  const uint8_t f = box.contains(i, jl) ? pf[o] : (uint8_t)0;
  if (f & PF_INACTIVE) {
    q[o] = 0.0;
    bp[o] = 0.0;
    phi0[o] = 0.0;
    return;
  }
  const double uE = us[gu.off(i + 1, jl)], uW = us[gu.off(i, jl)];
  const double vN = vs[gv.off(i, jl + 1)], vS = vs[gv.off(i, jl)];
  const double mE = (i + 1 == nx) ? 1.0 : ((f & PF_E) ? 0.0 : 1.0);
  const double mW = (i == 0) ? 1.0 : ((f & PF_W) ? 0.0 : 1.0);
  const double mN = (gj + 1 == ny) ? 1.0 : ((f & PF_N) ? 0.0 : 1.0);
  const double mS = (gj == 0) ? 1.0 : ((f & PF_S) ? 0.0 : 1.0);
  const double dxi = m.dx[i], dyj = m.dy[gj];
  const double rhs = pdiv(pdiv(mE * uE - mW * uW, dxi) + pdiv(mN * vN - mS * vS, dyj), dt);
  q[o] = pdiv((1.0 - mE) * uE - (1.0 - mW) * uW, dxi) + pdiv((1.0 - mN) * vN - (1.0 - mS) * vS, dyj);
  bp[o] = -rhs;
}

// ---------------------------------------------------------------- a7: projection
// S:296-304, R9, R16: open faces u = u* - dt (phi_E - phi_W)/h; the outlet face
// uses phi = 0 at the face; closed faces keep u*; p += phi on active cells.
// Non-finite results raise the NaN flag.
__global__ void k_correct_u(double *__restrict__ u, const double *__restrict__ us, const double *__restrict__ phi,
                            const uint8_t *__restrict__ pf, Geo gu, Geo gp, BBox pbox, Metric m, int nx, double dt,
                            int *nanflag) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  int jl = blockIdx.y * blockDim.y + threadIdx.y;
  if (i >= gu.ni || jl >= gu.nj) return;
  const long o = gu.off(i, jl);
  double val = us[o];
  if (i >= 1 && i <= nx - 1) {
    const uint8_t f = pbox.contains(i, jl) ? pf[gp.off(i, jl)] : (uint8_t)0;
    if (!(f & PF_W)) val = us[o] - dt * pdiv(phi[gp.off(i, jl)] - phi[gp.off(i - 1, jl)], m.hxc[i]);
  } else if (i == nx) {
    const uint8_t f = pbox.contains(nx - 1, jl) ? pf[gp.off(nx - 1, jl)] : (uint8_t)0;
    if (!(f & PF_INACTIVE)) val = us[o] - dt * pdiv(0.0 - phi[gp.off(nx - 1, jl)], 0.5 * m.dx[nx - 1]);
  }
  u[o] = val;
  if (!isfinite(val)) atomicOr(nanflag, 1);
}

__global__ void k_correct_v(double *__restrict__ v, const double *__restrict__ vs, const double *__restrict__ phi,
                            const uint8_t *__restrict__ pf, Geo gv, Geo gp, BBox pbox, Metric m, int ny, double dt,
                            int *nanflag) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  int jl = blockIdx.y * blockDim.y + threadIdx.y;
  if (i >= gv.ni || jl >= gv.nj) return;
  const long o = gv.off(i, jl);
  const int gj = gv.gj0 + jl;
  double val = vs[o];
  if (gj >= 1 && gj <= ny - 1) {
    const uint8_t f = pbox.contains(i, jl) ? pf[gp.off(i, jl)] : (uint8_t)0;
    if (!(f & PF_S)) val = vs[o] - dt * pdiv(phi[gp.off(i, jl)] - phi[gp.off(i, jl - 1)], m.hyc[gj]);
  }
  v[o] = val;
  if (!isfinite(val)) atomicOr(nanflag, 1);
}

__global__ void k_correct_p(double *__restrict__ p, const double *__restrict__ phi, const uint8_t *__restrict__ pf,
                            Geo gp, BBox pbox, int *nanflag) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  int jl = blockIdx.y * blockDim.y + threadIdx.y;
  if (i >= gp.ni || jl >= gp.nj) return;
  const long o = gp.off(i, jl);
  const uint8_t f = pbox.contains(i, jl) ? pf[o] : (uint8_t)0;
  double val = p[o];
  if (!(f & PF_INACTIVE)) val = p[o] + phi[o];
  p[o] = val;
  if (!isfinite(val)) atomicOr(nanflag, 1);
}

// ---------------------------------------------------------------- R17b: pressure extension
// An inactive cell with at least one active 4-neighbour takes the mean of their
// p^{n+1} (E, W, N, S order, left fold from 0.0); deeper inactive cells keep p.
// Runs after k_correct_p.  A neighbour in a ghost row (another slab) still holds
// p^n there (exchanged at the start of the step), so its p^{n+1} = p^n + phi is
// formed here -- the same IEEE addition its own slab performed.
__global__ void k_pext(double *__restrict__ p, const double *__restrict__ phi, const uint8_t *__restrict__ pf,
                       Geo gp, BBox pbox, int nx, int ny) {
  const int i = pbox.i0 + blockIdx.x * blockDim.x + threadIdx.x;
  const int jl = max(pbox.j0, 0) + blockIdx.y * blockDim.y + threadIdx.y;
  if (i >= pbox.i1 || jl >= min(pbox.j1, gp.nj)) return;
  if (!(pf[gp.off(i, jl)] & PF_INACTIVE)) return;
  double sum = 0.0;
  int cnt = 0;
#pragma unroll
  for (int d = 0; d < 4; ++d) {
    const int di = (d == 0) ? 1 : (d == 1) ? -1 : 0;
    const int dj = (d == 2) ? 1 : (d == 3) ? -1 : 0;
    const int in_ = i + di, jn = jl + dj, gjn = gp.gj0 + jn;
    if (in_ < 0 || in_ >= nx || gjn < 0 || gjn >= ny) continue;
    const uint8_t fn = pbox.contains(in_, jn) ? pf[gp.off(in_, jn)] : (uint8_t)0;
    if (fn & PF_INACTIVE) continue;
    const long o = gp.off(in_, jn);
    const double pn = (jn >= 0 && jn < gp.nj) ? p[o] : p[o] + phi[o];
    sum = sum + pn;
    cnt = cnt + 1;
  }
  if (cnt > 0) p[gp.off(i, jl)] = pdiv(sum, (double)cnt);
}

// ---------------------------------------------------------------- a8: forces (R20, R19b)
// red[0] = sum_{Solid,Forcing} f_u dV, red[1] = sum_{Solid,Forcing} u dV, red[2], red[3] for v.
// Deterministic two-level reduction: CTA b of kForceParts sums a fixed contiguous
// chunk of the body boxes' nodes (fixed tree order) into part[q][b]; one CTA then
// sums the parts in order.
constexpr int kForceParts = 64, kForceThreads = 256;
__global__ void __launch_bounds__(kForceThreads) k_forces_part(const double *__restrict__ u,
                                                               const double *__restrict__ v,
                                                               const double *__restrict__ fu,
                                                               const double *__restrict__ fv,
                                                               const uint8_t *__restrict__ tu,
                                                               const uint8_t *__restrict__ tv, Geo gu, Geo gv,
                                                               BBox bu, BBox bv, Metric m, int nx, int ny,
                                                               double *part) {
  __shared__ double sh[4][kForceThreads];
  const int wu = bu.i1 - bu.i0, nu = wu > 0 ? wu * (bu.j1 - bu.j0) : 0;
  const int wv = bv.i1 - bv.i0, nv = wv > 0 ? wv * (bv.j1 - bv.j0) : 0;
  const int n = nu + nv, chunk = (n + kForceParts - 1) / kForceParts;
  const int lo = blockIdx.x * chunk, hi = min(n, lo + chunk);
  double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
  for (int idx = lo + threadIdx.x; idx < hi; idx += kForceThreads) {
    if (idx < nu) {
      const int i = bu.i0 + idx % wu, jl = bu.j0 + idx / wu;
      if (i < 1 || i > nx - 1 || jl < 0 || jl >= gu.nj) continue;
      const long o = gu.off(i, jl);
      if (tu[o] == FLUID) continue;
      const double dV = m.hxc[i] * m.dy[gu.gj0 + jl];
      s1 = s1 + u[o] * dV;
      s0 = s0 + fu[o] * dV;
    } else {
      const int k = idx - nu;
      const int i = bv.i0 + k % wv, jl = bv.j0 + k / wv;
      const int gj = gv.gj0 + jl;
      if (gj < 1 || gj > ny - 1 || jl < 0 || jl >= gv.nj) continue;
      const long o = gv.off(i, jl);
      if (tv[o] == FLUID) continue;
      const double dV = m.dx[i] * m.hyc[gj];
      s3 = s3 + v[o] * dV;
      s2 = s2 + fv[o] * dV;
    }
  }
  sh[0][threadIdx.x] = s0;
  sh[1][threadIdx.x] = s1;
  sh[2][threadIdx.x] = s2;
  sh[3][threadIdx.x] = s3;
  __syncthreads();
  for (int st = kForceThreads / 2; st > 0; st >>= 1) {
    if (threadIdx.x < st)
      for (int q = 0; q < 4; ++q) sh[q][threadIdx.x] = sh[q][threadIdx.x] + sh[q][threadIdx.x + st];
    __syncthreads();
  }
  if (threadIdx.x < 4) part[threadIdx.x * kForceParts + blockIdx.x] = sh[threadIdx.x][0];
}

__global__ void k_forces_final(const double *__restrict__ part, double *red) {
  const int q = threadIdx.x;
  if (q >= 4) return;
  double s = 0.0;
  for (int b = 0; b < kForceParts; ++b) s = s + part[q * kForceParts + b];
  red[q] = s;
}

// fill the owned rows of a family with a constant (initial condition)
__global__ void k_fill(double *__restrict__ p, Geo g, double val) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  int jl = blockIdx.y * blockDim.y + threadIdx.y;
  if (i >= g.ni || jl >= g.nj) return;
  p[g.off(i, jl)] = val;
}

// ================================================================ launchers
static dim3 grid2(int ni, int nj, dim3 b) { return dim3((ni + b.x - 1) / b.x, (nj + b.y - 1) / b.y); }

int launch_classify(const Ctx &c, const Slab &s, double yb) {
  int n = 0;
  const Body &B = c.body;
  struct F {
    uint8_t *t;
    const Geo *g;
    const BBox *b;
    const double *xs, *ys;
  } fams[3] = {{s.tu, &s.gu, &s.bu, c.m.xn, c.m.yc}, {s.tv, &s.gv, &s.bv, c.m.xc, c.m.yn},
               {s.tp, &s.gp, &s.bpb, c.m.xc, c.m.yc}};
  for (auto &f : fams) {
    if (f.b->empty()) continue;
    // classification also covers the ghost rows inside the box (analytic, no exchange)
    const BBox box = *f.b;
    dim3 blk(32, 8);
    k_classify<<<grid2(box.i1 - box.i0, box.j1 - box.j0, blk), blk, 0, c.stream>>>(f.t, *f.g, box, f.xs, f.ys, B.a,
                                                                                     B.b, B.x0, yb);
    ++n;
  }
  return n;
}

int launch_pflags(const Ctx &c, const Slab &s) {
  if (s.bpb.empty()) return 0;
  // flags are needed on the owned rows and on the ghost rows a decomposed pass
  // updates: one for the one-iteration pass, 2m - 1 <= kGhost - 1 for a pass fusing m
  BBox box = s.bpb;
  box.j0 = box.j0 < 1 - kGhost ? 1 - kGhost : box.j0;
  box.j1 = box.j1 > s.gp.nj + kGhost - 1 ? s.gp.nj + kGhost - 1 : box.j1;
  if (box.empty()) return 0;
  dim3 blk(32, 8);
  k_pflags<<<grid2(box.i1 - box.i0, box.j1 - box.j0, blk), blk, 0, c.stream>>>(s.pf, s.tp, s.tu, s.tv, s.gp, s.gu,
                                                                                s.gv, box, c.m, c.nx, c.ny);
  return 1;
}

int launch_predictor(const Ctx &c, const Slab &s, double yb, double vb) {
  PredArgs A;
  A.u = s.u; A.v = s.v; A.p = s.p; A.cup = s.cup; A.cvp = s.cvp;
  A.cu = s.cu; A.cv = s.cv; A.ru = s.ru; A.rv = s.rv; A.us = s.us[0]; A.vs = s.vs[0]; A.fu = s.fu; A.fv = s.fv;
  A.tu = s.tu; A.tv = s.tv; A.pf = s.pf;
  A.gu = s.gu; A.gv = s.gv; A.gp = s.gp;
  A.bu = s.bu; A.bv = s.bv; A.bp = s.bpb;
  A.m = c.m;
  A.B.a = c.body.a; A.B.b = c.body.b; A.B.xb = c.body.x0; A.B.yb = yb; A.B.vb = vb;
  A.nx = c.nx; A.ny = c.ny; A.have_hist = c.have_hist;
  A.dt = c.cfg.dt;
  A.halfnu = 0.5 / c.cfg.Re;
  A.nu = 1.0 / c.cfg.Re;
  dim3 blk(128, 2);
  k_pred_u<<<grid2(s.gu.ni, s.gu.nj, blk), blk, 0, c.stream>>>(A);
  k_pred_v<<<grid2(s.gv.ni, s.gv.nj, blk), blk, 0, c.stream>>>(A);
  return 2;
}

int launch_outlet_fill(const Ctx &c, const Slab &s, double *us, const double *vs) {
  k_outlet_fill<<<(s.gu.nj + 127) / 128, 128, 0, c.stream>>>(us, vs, s.gu, s.gv, c.m, c.nx);
  return 1;
}

int launch_prhs(const Ctx &c, const Slab &s, const double *us, const double *vs, double *phi_start) {
  dim3 blk(128, 2);
  k_prhs<<<grid2(s.gp.ni, s.gp.nj, blk), blk, 0, c.stream>>>(us, vs, s.bp, s.q, phi_start, s.pf, s.gp, s.gu, s.gv,
                                                             s.bpb, c.m, c.nx, c.ny, c.cfg.dt);
  return 1;
}

int launch_pext(const Ctx &c, const Slab &s, const double *phi) {
  const BBox &b = s.bpb;
  const int j0 = b.j0 > 0 ? b.j0 : 0, j1 = b.j1 < s.gp.nj ? b.j1 : s.gp.nj;
  if (b.empty() || j1 <= j0) return 0;
  dim3 blk(32, 8);
  k_pext<<<grid2(b.i1 - b.i0, j1 - j0, blk), blk, 0, c.stream>>>(s.p, phi, s.pf, s.gp, b, c.nx, c.ny);
  return 1;
}

int launch_correct(const Ctx &c, const Slab &s, const double *us, const double *vs, const double *phi) {
  dim3 blk(128, 2);
  k_correct_u<<<grid2(s.gu.ni, s.gu.nj, blk), blk, 0, c.stream>>>(s.u, us, phi, s.pf, s.gu, s.gp, s.bpb, c.m, c.nx,
                                                                  c.cfg.dt, c.nanflag);
  k_correct_v<<<grid2(s.gv.ni, s.gv.nj, blk), blk, 0, c.stream>>>(s.v, vs, phi, s.pf, s.gv, s.gp, s.bpb, c.m, c.ny,
                                                                  c.cfg.dt, c.nanflag);
  k_correct_p<<<grid2(s.gp.ni, s.gp.nj, blk), blk, 0, c.stream>>>(s.p, phi, s.pf, s.gp, s.bpb, c.nanflag);
  return 3;
}

void launch_fill(double *p, const Geo &g, double val, cudaStream_t st) {
  dim3 blk(128, 2);
  k_fill<<<grid2(g.ni, g.nj, blk), blk, 0, st>>>(p, g, val);
}

int launch_forces(const Ctx &c, const Slab &s) {
  k_forces_part<<<kForceParts, kForceThreads, 0, c.stream>>>(s.u, s.v, s.fu, s.fv, s.tu, s.tv, s.gu, s.gv, s.bu, s.bv,
                                                             c.m, c.nx, c.ny, s.red + 4);
  k_forces_final<<<1, 32, 0, c.stream>>>(s.red + 4, s.red);
  return 2;
}

}  // namespace ibm
