/*
 * oracle/ibm_oracle.c -- CPU fp64 ORACLE for the per-time-step hot path of the
 * discrete-forcing IBM fractional-step solver of arXiv 2402.17337.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference leg may load this library.  The
 * product path (paper_2402_17337_b200/) never imports, links or calls it, and
 * this file shares no code, header, table or constant generator with it.
 *
 * Form: plain loops, one thread, no blocking, no fusion, full-array temporaries,
 * compiled with -O2 -ffp-contract=off (no FMA contraction, IEEE / and sqrt).
 * Every expression is written exactly as parenthesised in DESIGN.md §3 (the
 * arithmetic contract, reading R13), evaluated left to right inside a
 * parenthesis.
 *
 * Citations: P:NN = /root/reference/PAPER.md line NN, S:NN = SPEC.md line NN,
 * Rnn = reading nn of DESIGN.md §2 (same numbering as SURVEY.md §8(c)).
 *
 * Pins (tests/test_oracle_pins.py) -- what fixes each function from outside:
 *   orc_plunge            closed form / FD consistency / periodicity
 *   orc_inside/classify   brute force + S:174 worked example + area ~ pi a b
 *   orc_intercept         bisection within 1e-10, ellipse residual
 *   orc_target_dir        numpy.polyfit line through (B,uB),(N,uN) at F
 *   orc_convection        uniform flow -> 0 exactly; smooth field -> 2nd order
 *   orc_laplacian         smooth fields -> 2nd order (interior and BC nodes)
 *   orc_sor_generic       16x16 Dirichlet Poisson vs dense numpy solve
 *   orc_poisson           manufactured closed form, 2nd-order decay
 *   orc_step              uniform-flow fixed point, projection identity,
 *                         mirror symmetry, zero-force cases,
 *                         temporal order (AB2/CN/projection self-convergence)
 *   forcing_target        all four directions: linear fields through N / N2,
 *                         brute force (bisection + polyfit) at every node
 *   forces (a8)           Archimedes -V grad p, viscous 2V/Re of u = y^2,
 *                         cancellation for a body started from rest, discrete
 *                         momentum budget (tests/test_oracle_force_pins.py)
 */
#define _POSIX_C_SOURCE 199309L /* clock_gettime (region timers only) */
#include <math.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

enum { FLUID = 0, SOLID = 1, FORCING = 2 };
enum { ORC_OK = 0, ORC_WARN_NOCONV = 1, ORC_ERR_CONFIG = 2, ORC_ERR_DIVERGED = 3 };

typedef struct {
    /* grid (S:36-42, P:54 staggered MAC arrangement) */
    int nx, ny;
    double *xn, *yn;              /* nodes, nx+1 / ny+1 */
    double *dx, *dy;              /* cell widths */
    double *xc, *yc;              /* cell centres */
    double *hxc, *hyc;            /* centre spacings, index 1..n-1 (index 0 unused) */
    /* parameters */
    double Re, dt, omega_p, tol_p, omega_uv, tol_uv;
    int maxit_p, maxit_uv, check_every;
    /* body */
    int has_body;
    double a, b, x0, y0, hbar, k;
    /* state */
    double *u, *v, *p, *phi;
    double *cu, *cv, *cu_prev, *cv_prev;
    double *fu, *fv, *q;
    double *us, *vs, *rhs_u, *rhs_v, *bp;
    unsigned char *tu, *tv, *tp;
    unsigned char *act, *open_u, *open_v;
    int step, have_hist;
    double Mx, My;
    /* last-step outputs */
    double t, yb, vb, cd, cl;
    int it_uv, it_p;
    double rho_uv, rho_p;
    /* region wall times (s), accumulated over steps, in the layout of the paper's
     * Table 1: flagging, predictor + forcing, U-V solver, Poisson rhs,
     * P solver, correction, forces.  Timing only: no effect on the arithmetic. */
    double tm[7];
} orc_ctx;

/* ---------------- indexing ---------------- */
#define UI(c, i, j) ((size_t)(j) * (size_t)((c)->nx + 1) + (size_t)(i))
#define VI(c, i, j) ((size_t)(j) * (size_t)(c)->nx + (size_t)(i))
#define PI_(c, i, j) ((size_t)(j) * (size_t)(c)->nx + (size_t)(i))

static double now_s(void)
{
    struct timespec ts;
    clock_gettime(CLOCK_MONOTONIC, &ts);
    return (double)ts.tv_sec + 1e-9 * (double)ts.tv_nsec;
}
/* adds the time since *t0 to region r and restarts the clock */
static void tick(orc_ctx *c, int r, double *t0)
{
    double t = now_s();
    c->tm[r] += t - *t0;
    *t0 = t;
}

/* ORC_PAR: row loops whose iterations write disjoint elements (the OpenMP build,
 * -fopenmp, splits them over threads; without it the pragma is ignored and the
 * oracle is the plain one-thread program).  Sum reductions (forces, solid
 * momentum) are never parallelised, so both builds are bitwise identical. */
#ifdef _OPENMP
#define ORC_PAR _Pragma("omp parallel for schedule(static)")
#else
#define ORC_PAR
#endif

static double *dalloc(size_t n) { return (double *)calloc(n ? n : 1, sizeof(double)); }
static unsigned char *balloc(size_t n) { return (unsigned char *)calloc(n ? n : 1, 1); }

/* ---------------- kinematics, Eqs. (1)-(2), P:34-37 ---------------- */
void orc_plunge(double t, double hbar, double k, double *out2)
{
    out2[0] = hbar * sin(k * t);          /* ybar(t) = h sin(k t)      Eq. 1 */
    out2[1] = (k * hbar) * cos(k * t);    /* ydot(t) = k h cos(k t)    Eq. 2 */
}

/* ---------------- geometry: boundary-inclusive ellipse test, S:166-174 -------- */
int orc_inside(double x, double y, double a, double b, double xb, double yb)
{
    double dxn = (x - xb) / a;
    double dyn = (y - yb) / b;
    double s = dxn * dxn + dyn * dyn;
    return s <= 1.0;
}

/* Closed-form intercept of an axis-aligned segment from an inside node F toward
 * an outside node N with the ellipse.  axis 0: horizontal segment at
 * y = yF, returns x_B; axis 1: vertical segment at x = xF, returns y_B.
 * dir = +1 toward increasing coordinate, -1 toward decreasing. */
double orc_intercept(int axis, int dir, double xF, double yF,
                     double a, double b, double xb, double yb)
{
    if (axis == 0) {
        double eta = (yF - yb) / b;
        double w = a * sqrt(1.0 - eta * eta);
        return dir > 0 ? xb + w : xb - w;
    } else {
        double zeta = (xF - xb) / a;
        double w = b * sqrt(1.0 - zeta * zeta);
        return dir > 0 ? yb + w : yb - w;
    }
}

/* One-direction forcing target (R14): linear extrapolation from the
 * boundary intercept B (value uB) through the fluid neighbour N (value uN) to
 * the forcing node F, which lies on the other side of B at distance dF. */
double orc_target_dir(double uB, double uN, double dF, double dN)
{
    return uB - (uN - uB) * (dF / dN);
}

/* ---------------- grid metrics ---------------- */
static void build_metrics(orc_ctx *c)
{
    int nx = c->nx, ny = c->ny;
    for (int i = 0; i < nx; ++i) {
        c->dx[i] = c->xn[i + 1] - c->xn[i];
        c->xc[i] = 0.5 * (c->xn[i] + c->xn[i + 1]);
    }
    for (int j = 0; j < ny; ++j) {
        c->dy[j] = c->yn[j + 1] - c->yn[j];
        c->yc[j] = 0.5 * (c->yn[j] + c->yn[j + 1]);
    }
    c->hxc[0] = 0.0;
    c->hyc[0] = 0.0;
    for (int i = 1; i < nx; ++i) c->hxc[i] = c->xc[i] - c->xc[i - 1];
    for (int j = 1; j < ny; ++j) c->hyc[j] = c->yc[j] - c->yc[j - 1];
}

/* Five-point operator coefficients of the viscous / pressure Laplacians on each
 * staggered family (readings R10).  fam: 0=u, 1=v, 2=p. */
static void coef(const orc_ctx *c, int fam, int i, int j,
                 double *cE, double *cW, double *cN, double *cS, double *cD)
{
    int nx = c->nx, ny = c->ny;
    const double *dx = c->dx, *dy = c->dy, *hxc = c->hxc, *hyc = c->hyc;
    *cE = *cW = *cN = *cS = *cD = 0.0;
    if (fam == 0) {               /* u at (xn_i, yc_j), interior 1 <= i <= nx-1 */
        if (i < 1 || i > nx - 1) return;
        if (i <= nx - 2) *cE = 1.0 / (hxc[i] * dx[i]);     /* outlet: zero gradient */
        *cW = 1.0 / (hxc[i] * dx[i - 1]);
        if (j <= ny - 2) *cN = 1.0 / (dy[j] * hyc[j + 1]); /* slip top wall */
        if (j >= 1) *cS = 1.0 / (dy[j] * hyc[j]);          /* slip bottom wall */
    } else if (fam == 1) {        /* v at (xc_i, yn_j), interior 1 <= j <= ny-1 */
        if (j < 1 || j > ny - 1) return;
        if (i <= nx - 2) *cE = 1.0 / (dx[i] * hxc[i + 1]); /* outlet: zero gradient */
        if (i >= 1) *cW = 1.0 / (dx[i] * hxc[i]);
        if (i == 0) *cD = 2.0 / (dx[0] * dx[0]);           /* v = 0 on the inlet face */
        *cN = 1.0 / (hyc[j] * dy[j]);
        *cS = 1.0 / (hyc[j] * dy[j - 1]);
    } else {                      /* p / phi at (xc_i, yc_j) */
        if (i <= nx - 2) *cE = 1.0 / (dx[i] * hxc[i + 1]);
        if (i >= 1) *cW = 1.0 / (dx[i] * hxc[i]);
        if (i == nx - 1) *cD = 2.0 / (dx[nx - 1] * dx[nx - 1]); /* phi = 0 on the outlet face */
        if (j <= ny - 2) *cN = 1.0 / (dy[j] * hyc[j + 1]);
        if (j >= 1) *cS = 1.0 / (dy[j] * hyc[j]);
    }
}

static int fam_ni(const orc_ctx *c, int fam) { return fam == 0 ? c->nx + 1 : c->nx; }
static int fam_nj(const orc_ctx *c, int fam) { return fam == 1 ? c->ny + 1 : c->ny; }

/* field value with 0 outside the family's index range */
static double fv_at(const double *x, int ni, int nj, int i, int j)
{
    if (i < 0 || j < 0 || i >= ni || j >= nj) return 0.0;
    return x[(size_t)j * (size_t)ni + (size_t)i];
}

/* L x at one node: ((cE(xE-xC) + cW(xW-xC)) + (cN(xN-xC) + cS(xS-xC))) - cD xC */
static double lap_at(const orc_ctx *c, int fam, const double *x, int i, int j)
{
    int ni = fam_ni(c, fam), nj = fam_nj(c, fam);
    double cE, cW, cN, cS, cD;
    coef(c, fam, i, j, &cE, &cW, &cN, &cS, &cD);
    double xC = fv_at(x, ni, nj, i, j);
    double xE = fv_at(x, ni, nj, i + 1, j), xW = fv_at(x, ni, nj, i - 1, j);
    double xN = fv_at(x, ni, nj, i, j + 1), xS = fv_at(x, ni, nj, i, j - 1);
    return ((cE * (xE - xC) + cW * (xW - xC)) + (cN * (xN - xC) + cS * (xS - xC))) - cD * xC;
}

/* ---------------- classification, S:175-183, P:52 (R12, R15) ---------------- */
static void node_xy(const orc_ctx *c, int fam, int i, int j, double *x, double *y)
{
    if (fam == 0) { *x = c->xn[i]; *y = c->yc[j]; }
    else if (fam == 1) { *x = c->xc[i]; *y = c->yn[j]; }
    else { *x = c->xc[i]; *y = c->yc[j]; }
}

static void classify_family(const orc_ctx *c, int fam, double yb, unsigned char *tag)
{
    int ni = fam_ni(c, fam), nj = fam_nj(c, fam);
    size_t n = (size_t)ni * (size_t)nj;
    unsigned char *in = balloc(n);
    ORC_PAR
    for (int j = 0; j < nj; ++j)
        for (int i = 0; i < ni; ++i) {
            double x, y;
            node_xy(c, fam, i, j, &x, &y);
            in[(size_t)j * ni + i] = c->has_body ? (unsigned char)orc_inside(x, y, c->a, c->b, c->x0, yb) : 0;
        }
    ORC_PAR
    for (int j = 0; j < nj; ++j)
        for (int i = 0; i < ni; ++i) {
            size_t id = (size_t)j * ni + i;
            if (!in[id]) { tag[id] = FLUID; continue; }
            int fluid_nb = 0;
            if (i + 1 < ni && !in[id + 1]) fluid_nb = 1;
            if (i - 1 >= 0 && !in[id - 1]) fluid_nb = 1;
            if (j + 1 < nj && !in[id + ni]) fluid_nb = 1;
            if (j - 1 >= 0 && !in[id - ni]) fluid_nb = 1;
            tag[id] = fluid_nb ? FORCING : SOLID;
        }
    free(in);
}

static void body_at(orc_ctx *c, double t)
{
    double yv[2] = {0.0, 0.0};
    if (c->has_body) orc_plunge(t, c->hbar, c->k, yv);
    c->yb = c->y0 + yv[0];
    c->vb = yv[1];
}

/* classify all three families for the body at time t; writes ctx tags */
void orc_classify_at(orc_ctx *c, double t)
{
    body_at(c, t);
    classify_family(c, 0, c->yb, c->tu);
    classify_family(c, 1, c->yb, c->tv);
    classify_family(c, 2, c->yb, c->tp);
}

/* ---------------- convection, S:233-241 (R7) ----------------
 * Evaluated at every interior node, Solid ones included: C at a Solid node only
 * enters u_hat of the momentum forcing there (R19b), never a Fluid row. */
static void convection(const orc_ctx *c, const double *u, const double *v, double *cu, double *cv)
{
    int nx = c->nx, ny = c->ny;
    const double *dx = c->dx, *dy = c->dy, *hxc = c->hxc, *hyc = c->hyc;
    size_t nu = (size_t)(nx + 1) * ny, nv = (size_t)nx * (ny + 1);
    for (size_t id = 0; id < nu; ++id) cu[id] = 0.0;
    for (size_t id = 0; id < nv; ++id) cv[id] = 0.0;
#define U(i, j) u[UI(c, i, j)]
#define V(i, j) v[VI(c, i, j)]
    ORC_PAR
    for (int j = 0; j < ny; ++j)
        for (int i = 1; i <= nx - 1; ++i) {
            double ue = 0.5 * (U(i, j) + U(i + 1, j));
            double uw = 0.5 * (U(i - 1, j) + U(i, j));
            double tn, ts;
            if (j == ny - 1) tn = 0.0;
            else {
                double un = (dy[j + 1] * U(i, j) + dy[j] * U(i, j + 1)) / (dy[j] + dy[j + 1]);
                double vn = (dx[i] * V(i - 1, j + 1) + dx[i - 1] * V(i, j + 1)) / (dx[i - 1] + dx[i]);
                tn = un * vn;
            }
            if (j == 0) ts = 0.0;
            else {
                double us = (dy[j] * U(i, j - 1) + dy[j - 1] * U(i, j)) / (dy[j - 1] + dy[j]);
                double vs = (dx[i] * V(i - 1, j) + dx[i - 1] * V(i, j)) / (dx[i - 1] + dx[i]);
                ts = us * vs;
            }
            cu[UI(c, i, j)] = (ue * ue - uw * uw) / hxc[i] + (tn - ts) / dy[j];
        }
    ORC_PAR
    for (int j = 1; j <= ny - 1; ++j)
        for (int i = 0; i < nx; ++i) {
            double vn = 0.5 * (V(i, j) + V(i, j + 1));
            double vs = 0.5 * (V(i, j - 1) + V(i, j));
            double ue = (dy[j] * U(i + 1, j - 1) + dy[j - 1] * U(i + 1, j)) / (dy[j - 1] + dy[j]);
            double ve = (i == nx - 1) ? V(i, j)
                                      : (dx[i + 1] * V(i, j) + dx[i] * V(i + 1, j)) / (dx[i] + dx[i + 1]);
            double te = ue * ve, tw;
            if (i == 0) tw = 0.0; /* inlet corner: u = 1, v = 0 */
            else {
                double uw = (dy[j] * U(i, j - 1) + dy[j - 1] * U(i, j)) / (dy[j - 1] + dy[j]);
                double vw = (dx[i] * V(i - 1, j) + dx[i - 1] * V(i, j)) / (dx[i - 1] + dx[i]);
                tw = uw * vw;
            }
            cv[VI(c, i, j)] = (te - tw) / dx[i] + (vn * vn - vs * vs) / hyc[j];
        }
#undef U
#undef V
}

/* ---------------- generic red-black SOR, S:278-286 (R1-R5) ---------------- */
/* 0: the arithmetic contract R13 (default, what the GPU evaluates); 1: the plain
 * IEEE form of SURVEY 8(c), kept only so a pin can show that the contract is a
 * rounding choice (tests/test_oracle_pins.py::test_sor_contract_vs_plain_ieee) */
static int g_sor_plain = 0;
void orc_set_sor_form(int plain) { g_sor_plain = plain ? 1 : 0; }

typedef struct {
    int ni, nj;
    double *x;
    const double *b, *aP, *aE, *aW, *aN, *aS;
    const unsigned char *upd;
} sor_sys;

/* Runs red-black SOR on nsys independent systems jointly: one iteration = red
 * sweep of every system, then black sweep of every system; rho_k = max over all
 * updates of |gs - x_old|.  Node update (R2, R13):
 *   n = fma(aN, xN, fma(aE, xE, fma(aW, xW, fma(aS, xS, b))));  r = 1/aP;
 *   d = fma(n, r, -x_old) (= gs - x_old, gs = n/aP, one rounding);
 *   x = fma(omega, d, x_old) (= (1-omega) x_old + omega gs);  e = |d|.
 *   fma is C99 fma (one rounding); 1/aP is the correctly rounded reciprocal (one
 *   IEEE division) -- reading R13.  Colour red = (i+j) even.  Returns iterations; status
 * ORC_ERR_DIVERGED if rho is NaN, ORC_WARN_NOCONV if maxit reached above tol. */
static int sor_run(int nsys, sor_sys *sys, double omega, double tol, int maxit,
                   int check_every, double *rho_out, int *status)
{
    double rho = 0.0;
    int k;
    *status = ORC_OK;
    for (k = 1;; ++k) {
        rho = 0.0;
        int rho_nan = 0;
        for (int colour = 0; colour < 2; ++colour)
            for (int s = 0; s < nsys; ++s) {
                sor_sys *S = &sys[s];
                /* rows of one colour are independent: the OpenMP build splits them over
                 * threads; max and NaN are order-independent, so both builds agree bitwise */
#ifdef _OPENMP
#pragma omp parallel
#endif
                {
                double trho = 0.0;
                int tnan = 0;
#ifdef _OPENMP
#pragma omp for schedule(static)
#endif
                for (int j = 0; j < S->nj; ++j)
                    for (int i = 0; i < S->ni; ++i) {
                        if (((i + j) & 1) != colour) continue;
                        size_t id = (size_t)j * S->ni + i;
                        if (!S->upd[id]) continue;
                        double xE = fv_at(S->x, S->ni, S->nj, i + 1, j);
                        double xW = fv_at(S->x, S->ni, S->nj, i - 1, j);
                        double xN = fv_at(S->x, S->ni, S->nj, i, j + 1);
                        double xS = fv_at(S->x, S->ni, S->nj, i, j - 1);
                        double xo = S->x[id], d;
                        if (!g_sor_plain) {
                            /* R13: b + sum of the neighbour terms as a chain of fused multiply-adds
                             * (C99 fma, one rounding each), S, W, E, N */
                            double num = fma(S->aN[id], xN, fma(S->aE[id], xE, fma(S->aW[id], xW,
                                             fma(S->aS[id], xS, S->b[id]))));
                            double rcp = 1.0 / S->aP[id];
                            d = fma(num, rcp, -xo); /* gs - x_old, gs = num * rcp (R13) */
                            S->x[id] = fma(omega, d, xo);
                        } else {
                            /* SURVEY 8(c) plain IEEE form (cross-check only, never the
                             * contract): s, gs = (b + s)/aP, x = (1-w) x + w gs */
                            double sn = (S->aE[id] * xE + S->aW[id] * xW) + (S->aN[id] * xN + S->aS[id] * xS);
                            double gs = (S->b[id] + sn) / S->aP[id];
                            d = gs - xo;
                            S->x[id] = (1.0 - omega) * xo + omega * gs;
                        }
                        double e = fabs(d);
                        if (isnan(e)) tnan = 1;
                        else if (e > trho) trho = e;
                    }
#ifdef _OPENMP
#pragma omp critical
#endif
                {
                    if (tnan) rho_nan = 1;
                    if (trho > rho) rho = trho;
                }
                }
            }
        if (rho_nan) rho = NAN;
        if (isnan(rho)) { *status = ORC_ERR_DIVERGED; break; }
        if ((k % check_every == 0 && rho <= tol)) break;
        if (k == maxit) { *status = ORC_WARN_NOCONV; break; }
    }
    *rho_out = rho;
    return k;
}

/* exported single-system SOR over explicit per-node coefficient arrays */
int orc_sor_generic(int ni, int nj, const double *aP, const double *aE, const double *aW,
                    const double *aN, const double *aS, const double *b,
                    const unsigned char *upd, double *x, double omega, double tol,
                    int maxit, int check_every, double *rho_out, int *status)
{
    sor_sys s = {ni, nj, x, b, aP, aE, aW, aN, aS, upd};
    return sor_run(1, &s, omega, tol, maxit, check_every, rho_out, status);
}

/* ---------------- pressure masks (R16-R18) ---------------- */
static void build_masks(orc_ctx *c)
{
    int nx = c->nx, ny = c->ny;
    ORC_PAR
    for (int j = 0; j < ny; ++j)
        for (int i = 0; i < nx; ++i) c->act[PI_(c, i, j)] = (c->tp[PI_(c, i, j)] == FLUID);
    ORC_PAR
    for (int j = 0; j < ny; ++j)
        for (int i = 0; i <= nx; ++i) {
            int o = 0;
            if (i >= 1 && i <= nx - 1)
                o = c->tu[UI(c, i, j)] == FLUID && c->act[PI_(c, i - 1, j)] && c->act[PI_(c, i, j)];
            c->open_u[UI(c, i, j)] = (unsigned char)o;
        }
    ORC_PAR
    for (int j = 0; j <= ny; ++j)
        for (int i = 0; i < nx; ++i) {
            int o = 0;
            if (j >= 1 && j <= ny - 1)
                o = c->tv[VI(c, i, j)] == FLUID && c->act[PI_(c, i, j - 1)] && c->act[PI_(c, i, j)];
            c->open_v[VI(c, i, j)] = (unsigned char)o;
        }
    /* R18: an active cell whose Poisson diagonal is 0 (no open face, no Dirichlet face) is inactive */
    ORC_PAR
    for (int j = 0; j < ny; ++j)
        for (int i = 0; i < nx; ++i) {
            if (!c->act[PI_(c, i, j)]) continue;
            double cE, cW, cN, cS, cD;
            coef(c, 2, i, j, &cE, &cW, &cN, &cS, &cD);
            double aE = c->open_u[UI(c, i + 1, j)] ? cE : 0.0;
            double aW = c->open_u[UI(c, i, j)] ? cW : 0.0;
            double aN = c->open_v[VI(c, i, j + 1)] ? cN : 0.0;
            double aS = c->open_v[VI(c, i, j)] ? cS : 0.0;
            double aP = ((aE + aW) + (aN + aS)) + cD;
            if (aP == 0.0) c->act[PI_(c, i, j)] = 0;
        }
}

/* Poisson SOR on the current masks: A phi = b, (A x)_C = aP x_C - [(aE xE + aW xW) + (aN xN + aS xS)]
 * with aX = m_X cX, aP = ((aE + aW) + (aN + aS)) + cD. phi is the warm start. */
static int poisson_solve(orc_ctx *c, const double *b, double *phi, double *rho, int *status)
{
    int nx = c->nx, ny = c->ny;
    size_t n = (size_t)nx * ny;
    double *aP = dalloc(n), *aE = dalloc(n), *aW = dalloc(n), *aN = dalloc(n), *aS = dalloc(n);
    ORC_PAR
    for (int j = 0; j < ny; ++j)
        for (int i = 0; i < nx; ++i) {
            size_t id = PI_(c, i, j);
            if (!c->act[id]) { aP[id] = 1.0; phi[id] = 0.0; continue; }
            double cE, cW, cN, cS, cD;
            coef(c, 2, i, j, &cE, &cW, &cN, &cS, &cD);
            aE[id] = c->open_u[UI(c, i + 1, j)] ? cE : 0.0;
            aW[id] = c->open_u[UI(c, i, j)] ? cW : 0.0;
            aN[id] = c->open_v[VI(c, i, j + 1)] ? cN : 0.0;
            aS[id] = c->open_v[VI(c, i, j)] ? cS : 0.0;
            aP[id] = ((aE[id] + aW[id]) + (aN[id] + aS[id])) + cD;
        }
    sor_sys s = {nx, ny, phi, b, aP, aE, aW, aN, aS, c->act};
    int it = sor_run(1, &s, c->omega_p, c->tol_p, c->maxit_p, c->check_every, rho, status);
    free(aP); free(aE); free(aW); free(aN); free(aS);
    return it;
}

/* ---------------- forcing targets, S:251-259 (R14, R15) ---------------- */
static double forcing_target(const orc_ctx *c, int fam, const double *x, const unsigned char *tag,
                             int i, int j, double uB)
{
    int ni = fam_ni(c, fam), nj = fam_nj(c, fam);
    double xF, yF;
    node_xy(c, fam, i, j, &xF, &yF);
    double sum = 0.0;
    int cnt = 0;
    static const int di[4] = {1, -1, 0, 0}, dj[4] = {0, 0, 1, -1}; /* E, W, N, S */
    for (int d = 0; d < 4; ++d) {
        int in_ = i + di[d], jn = j + dj[d];
        if (in_ < 0 || jn < 0 || in_ >= ni || jn >= nj) continue;
        if (tag[(size_t)jn * ni + in_] != FLUID) continue;
        double xN, yN;
        node_xy(c, fam, in_, jn, &xN, &yN);
        double dF, dN;
        if (d < 2) {
            double xB = orc_intercept(0, di[d], xF, yF, c->a, c->b, c->x0, c->yb);
            dF = fabs(xB - xF);
            dN = fabs(xN - xB);
        } else {
            double yB = orc_intercept(1, dj[d], xF, yF, c->a, c->b, c->x0, c->yb);
            dF = fabs(yB - yF);
            dN = fabs(yN - yB);
        }
        double uN = x[(size_t)jn * ni + in_];
        /* R14b (stability): when the fluid neighbour is closer to the boundary than
         * the forcing node (dN < dF, extrapolation ratio > 1), extrapolate through
         * the second node N2 = N + (N - F) instead, if it is in range and Fluid. */
        if (dN < dF) {
            int i2 = in_ + di[d], j2 = jn + dj[d];
            if (i2 >= 0 && j2 >= 0 && i2 < ni && j2 < nj && tag[(size_t)j2 * ni + i2] == FLUID) {
                double x2, y2;
                node_xy(c, fam, i2, j2, &x2, &y2);
                dN = (d < 2) ? dN + fabs(x2 - xN) : dN + fabs(y2 - yN);
                uN = x[(size_t)j2 * ni + i2];
            }
        }
        sum = sum + orc_target_dir(uB, uN, dF, dN);
        cnt = cnt + 1;
    }
    return sum / (double)cnt;
}

/* ---------------- context ---------------- */
orc_ctx *orc_create(int nx, int ny, const double *xn, const double *yn, double Re, double dt,
                    double omega_p, double tol_p, int maxit_p, double omega_uv, double tol_uv,
                    int maxit_uv, int check_every)
{
    if (nx < 4 || ny < 4) return NULL;
    orc_ctx *c = (orc_ctx *)calloc(1, sizeof(orc_ctx));
    c->nx = nx; c->ny = ny;
    c->xn = dalloc(nx + 1); c->yn = dalloc(ny + 1);
    memcpy(c->xn, xn, sizeof(double) * (nx + 1));
    memcpy(c->yn, yn, sizeof(double) * (ny + 1));
    c->dx = dalloc(nx); c->dy = dalloc(ny); c->xc = dalloc(nx); c->yc = dalloc(ny);
    c->hxc = dalloc(nx); c->hyc = dalloc(ny);
    build_metrics(c);
    c->Re = Re; c->dt = dt; c->omega_p = omega_p; c->tol_p = tol_p; c->maxit_p = maxit_p;
    c->omega_uv = omega_uv; c->tol_uv = tol_uv; c->maxit_uv = maxit_uv;
    c->check_every = check_every < 1 ? 1 : check_every;
    size_t nu = (size_t)(nx + 1) * ny, nv = (size_t)nx * (ny + 1), np = (size_t)nx * ny;
    c->u = dalloc(nu); c->v = dalloc(nv); c->p = dalloc(np); c->phi = dalloc(np);
    c->cu = dalloc(nu); c->cv = dalloc(nv); c->cu_prev = dalloc(nu); c->cv_prev = dalloc(nv);
    c->fu = dalloc(nu); c->fv = dalloc(nv); c->q = dalloc(np);
    c->us = dalloc(nu); c->vs = dalloc(nv); c->rhs_u = dalloc(nu); c->rhs_v = dalloc(nv);
    c->bp = dalloc(np);
    c->tu = balloc(nu); c->tv = balloc(nv); c->tp = balloc(np);
    c->act = balloc(np); c->open_u = balloc(nu); c->open_v = balloc(nv);
    /* impulsive start u = 1, v = p = 0 (R11) */
    for (size_t id = 0; id < nu; ++id) c->u[id] = 1.0;
    return c;
}

void orc_destroy(orc_ctx *c)
{
    if (!c) return;
    double *ds[] = {c->xn, c->yn, c->dx, c->dy, c->xc, c->yc, c->hxc, c->hyc, c->u, c->v, c->p,
                    c->phi, c->cu, c->cv, c->cu_prev, c->cv_prev, c->fu, c->fv, c->q, c->us,
                    c->vs, c->rhs_u, c->rhs_v, c->bp};
    for (size_t i = 0; i < sizeof(ds) / sizeof(ds[0]); ++i) free(ds[i]);
    unsigned char *bs[] = {c->tu, c->tv, c->tp, c->act, c->open_u, c->open_v};
    for (size_t i = 0; i < sizeof(bs) / sizeof(bs[0]); ++i) free(bs[i]);
    free(c);
}

/* solid-region momentum M = sum over Solid u Forcing interior nodes of u dV (R20) */
static void solid_momentum(const orc_ctx *c, double *Mx, double *My)
{
    int nx = c->nx, ny = c->ny;
    double mx = 0.0, my = 0.0;
    for (int j = 0; j < ny; ++j)
        for (int i = 1; i <= nx - 1; ++i)
            if (c->tu[UI(c, i, j)] != FLUID) mx = mx + c->u[UI(c, i, j)] * (c->hxc[i] * c->dy[j]);
    for (int j = 1; j <= ny - 1; ++j)
        for (int i = 0; i < nx; ++i)
            if (c->tv[VI(c, i, j)] != FLUID) my = my + c->v[VI(c, i, j)] * (c->dx[i] * c->hyc[j]);
    *Mx = mx;
    *My = my;
}

static void refresh_time0(orc_ctx *c)
{
    orc_classify_at(c, (double)c->step * c->dt);
    solid_momentum(c, &c->Mx, &c->My);
}

int orc_set_body(orc_ctx *c, double a, double b, double x0, double y0, double hbar, double k)
{
    if (!(a > 0.0) || !(b > 0.0) || !(k > 0.0) || !(hbar >= 0.0)) return ORC_ERR_CONFIG;
    c->has_body = 1;
    c->a = a; c->b = b; c->x0 = x0; c->y0 = y0; c->hbar = hbar; c->k = k;
    refresh_time0(c);
    return ORC_OK;
}

int orc_clear_body(orc_ctx *c)
{
    c->has_body = 0;
    refresh_time0(c);
    return ORC_OK;
}

/* set state fields (any may be NULL); step counter and history reset */
int orc_set_fields(orc_ctx *c, const double *u, const double *v, const double *p)
{
    size_t nu = (size_t)(c->nx + 1) * c->ny, nv = (size_t)c->nx * (c->ny + 1), np = (size_t)c->nx * c->ny;
    if (u) memcpy(c->u, u, nu * sizeof(double));
    if (v) memcpy(c->v, v, nv * sizeof(double));
    if (p) memcpy(c->p, p, np * sizeof(double));
    memset(c->phi, 0, np * sizeof(double));
    c->step = 0;
    c->have_hist = 0;
    refresh_time0(c);
    return ORC_OK;
}

/* ---------------- one time step n -> n+1, S:305-313 order ---------------- */
static int step_once(orc_ctx *c)
{
    int nx = c->nx, ny = c->ny;
    size_t nu = (size_t)(nx + 1) * ny, nv = (size_t)nx * (ny + 1), np = (size_t)nx * ny;
    const double dt = c->dt;
    const double halfnu = 0.5 / c->Re, nu_ = 1.0 / c->Re, beta = dt * halfnu;
    int status = ORC_OK, st;
    double t0 = now_s();

    /* a0: t^{n+1} = (n+1) dt, body at t^{n+1} (R13, R15) ; a1: classification */
    c->t = (double)(c->step + 1) * dt;
    orc_classify_at(c, c->t);

    /* a5 masks (R16-R18) depend only on the tags, so they are built here: the
     * predictor's pressure gradient at Fluid nodes uses open faces only (R9b) */
    build_masks(c);
    tick(c, 0, &t0);

    /* a2: convection C^n at Fluid+Forcing nodes; first step Euler (R8) */
    convection(c, c->u, c->v, c->cu, c->cv);
    if (!c->have_hist) {
        memcpy(c->cu_prev, c->cu, nu * sizeof(double));
        memcpy(c->cv_prev, c->cv, nv * sizeof(double));
    }

    /* a2/a3: Helmholtz rhs (Fluid), targets (Forcing), body velocity (Solid), f (R19) */
    for (size_t id = 0; id < nu; ++id) { c->us[id] = c->u[id]; c->rhs_u[id] = 0.0; c->fu[id] = 0.0; }
    for (size_t id = 0; id < nv; ++id) { c->vs[id] = c->v[id]; c->rhs_v[id] = 0.0; c->fv[id] = 0.0; }
    ORC_PAR
    for (int j = 0; j < ny; ++j)
        for (int i = 1; i <= nx - 1; ++i) {
            size_t id = UI(c, i, j);
            double C = c->cu[id], Cp = c->cu_prev[id];
            double G = (c->p[PI_(c, i, j)] - c->p[PI_(c, i - 1, j)]) / c->hxc[i];
            double Lu = lap_at(c, 0, c->u, i, j);
            if (c->tu[id] == FLUID) {
                if (!c->open_u[id]) G = 0.0; /* R9b: closed (solid-adjacent) face, Neumann */
                c->rhs_u[id] = c->u[id] + dt * ((-(1.5 * C - 0.5 * Cp) - G) + halfnu * Lu);
            } else {
                /* R19b: Forcing nodes take the target, Solid nodes the body velocity; the
                 * momentum forcing f = (u*_prescribed - u_hat)/dt is recorded at both */
                double tgt = (c->tu[id] == FORCING) ? forcing_target(c, 0, c->u, c->tu, i, j, 0.0) : 0.0;
                double uhat = c->u[id] + dt * ((-(1.5 * C - 0.5 * Cp) - G) + nu_ * Lu);
                c->us[id] = tgt;
                c->fu[id] = (tgt - uhat) / dt;
            }
        }
    ORC_PAR
    for (int j = 1; j <= ny - 1; ++j)
        for (int i = 0; i < nx; ++i) {
            size_t id = VI(c, i, j);
            double C = c->cv[id], Cp = c->cv_prev[id];
            double G = (c->p[PI_(c, i, j)] - c->p[PI_(c, i, j - 1)]) / c->hyc[j];
            double Lv = lap_at(c, 1, c->v, i, j);
            if (c->tv[id] == FLUID) {
                if (!c->open_v[id]) G = 0.0; /* R9b */
                c->rhs_v[id] = c->v[id] + dt * ((-(1.5 * C - 0.5 * Cp) - G) + halfnu * Lv);
            } else {  /* R19b */
                double tgt = (c->tv[id] == FORCING) ? forcing_target(c, 1, c->v, c->tv, i, j, c->vb) : c->vb;
                double vhat = c->v[id] + dt * ((-(1.5 * C - 0.5 * Cp) - G) + nu_ * Lv);
                c->vs[id] = tgt;
                c->fv[id] = (tgt - vhat) / dt;
            }
        }

    tick(c, 1, &t0);
    /* a4: CN Helmholtz (I - beta L) u* = rhs, u and v jointly by red-black SOR (R5, R6) */
    {
        double *aPu = dalloc(nu), *aEu = dalloc(nu), *aWu = dalloc(nu), *aNu = dalloc(nu), *aSu = dalloc(nu);
        double *aPv = dalloc(nv), *aEv = dalloc(nv), *aWv = dalloc(nv), *aNv = dalloc(nv), *aSv = dalloc(nv);
        unsigned char *updu = balloc(nu), *updv = balloc(nv);
        ORC_PAR
        for (int j = 0; j < ny; ++j)
            for (int i = 0; i <= nx; ++i) {
                size_t id = UI(c, i, j);
                double cE, cW, cN, cS, cD;
                coef(c, 0, i, j, &cE, &cW, &cN, &cS, &cD);
                aEu[id] = beta * cE; aWu[id] = beta * cW; aNu[id] = beta * cN; aSu[id] = beta * cS;
                aPu[id] = 1.0 + beta * (((cE + cW) + (cN + cS)) + cD);
                updu[id] = (i >= 1 && i <= nx - 1 && c->tu[id] == FLUID);
            }
        ORC_PAR
        for (int j = 0; j <= ny; ++j)
            for (int i = 0; i < nx; ++i) {
                size_t id = VI(c, i, j);
                double cE, cW, cN, cS, cD;
                coef(c, 1, i, j, &cE, &cW, &cN, &cS, &cD);
                aEv[id] = beta * cE; aWv[id] = beta * cW; aNv[id] = beta * cN; aSv[id] = beta * cS;
                aPv[id] = 1.0 + beta * (((cE + cW) + (cN + cS)) + cD);
                updv[id] = (j >= 1 && j <= ny - 1 && c->tv[id] == FLUID);
            }
        sor_sys sys[2] = {{nx + 1, ny, c->us, c->rhs_u, aPu, aEu, aWu, aNu, aSu, updu},
                          {nx, ny + 1, c->vs, c->rhs_v, aPv, aEv, aWv, aNv, aSv, updv}};
        c->it_uv = sor_run(2, sys, c->omega_uv, c->tol_uv, c->maxit_uv, c->check_every, &c->rho_uv, &st);
        free(aPu); free(aEu); free(aWu); free(aNu); free(aSu);
        free(aPv); free(aEv); free(aWv); free(aNv); free(aSv);
        free(updu); free(updv);
        if (st == ORC_ERR_DIVERGED) return ORC_ERR_DIVERGED;
        if (st == ORC_WARN_NOCONV) status = ORC_WARN_NOCONV;
    }
    /* outlet fill (R10b): u*_{nx} from discrete continuity of the last cell column,
     * u*_{nx} = u*_{nx-1} - dx_{nx-1} (v*_N - v*_S)/dy.  The SPEC-literal
     * zero-gradient fill injects divergence wherever dv/dy != 0 at the
     * outlet and makes the time integration non-convergent. */
    for (int j = 0; j < ny; ++j)
        c->us[UI(c, nx, j)] = c->us[UI(c, nx - 1, j)] -
                              c->dx[nx - 1] * ((c->vs[VI(c, nx - 1, j + 1)] - c->vs[VI(c, nx - 1, j)]) / c->dy[j]);

    tick(c, 2, &t0);
    /* a5: mass source q and Poisson rhs on the masks built above (R16) */
    ORC_PAR
    for (int j = 0; j < ny; ++j)
        for (int i = 0; i < nx; ++i) {
            size_t id = PI_(c, i, j);
            if (!c->act[id]) { c->q[id] = 0.0; c->bp[id] = 0.0; continue; }
            double uE = c->us[UI(c, i + 1, j)], uW = c->us[UI(c, i, j)];
            double vN = c->vs[VI(c, i, j + 1)], vS = c->vs[VI(c, i, j)];
            double mE = (i + 1 == nx) ? 1.0 : (double)c->open_u[UI(c, i + 1, j)];
            double mW = (i == 0) ? 1.0 : (double)c->open_u[UI(c, i, j)];
            double mN = (j + 1 == ny) ? 1.0 : (double)c->open_v[VI(c, i, j + 1)];
            double mS = (j == 0) ? 1.0 : (double)c->open_v[VI(c, i, j)];
            double rhs = (((mE * uE - mW * uW) / c->dx[i]) + ((mN * vN - mS * vS) / c->dy[j])) / dt;
            c->q[id] = (((1.0 - mE) * uE - (1.0 - mW) * uW) / c->dx[i]) +
                       (((1.0 - mN) * vN - (1.0 - mS) * vS) / c->dy[j]);
            c->bp[id] = -rhs;
        }

    tick(c, 3, &t0);
    /* a6: Poisson red-black SOR, warm start phi^{n-1}, phi = 0 on inactive cells (R6, R17) */
    c->it_p = poisson_solve(c, c->bp, c->phi, &c->rho_p, &st);
    if (st == ORC_ERR_DIVERGED) return ORC_ERR_DIVERGED;
    if (st == ORC_WARN_NOCONV) status = ORC_WARN_NOCONV;

    tick(c, 4, &t0);
    /* a7: projection / correction (R9, R16, R17) */
    ORC_PAR
    for (int j = 0; j < ny; ++j)
        for (int i = 0; i <= nx; ++i) {
            size_t id = UI(c, i, j);
            double val = c->us[id];
            if (i >= 1 && i <= nx - 1) {
                if (c->open_u[id])
                    val = c->us[id] - dt * ((c->phi[PI_(c, i, j)] - c->phi[PI_(c, i - 1, j)]) / c->hxc[i]);
            } else if (i == nx) {
                if (c->act[PI_(c, nx - 1, j)])
                    val = c->us[id] - dt * ((0.0 - c->phi[PI_(c, nx - 1, j)]) / (0.5 * c->dx[nx - 1]));
            }
            c->u[id] = val;
        }
    ORC_PAR
    for (int j = 0; j <= ny; ++j)
        for (int i = 0; i < nx; ++i) {
            size_t id = VI(c, i, j);
            double val = c->vs[id];
            if (j >= 1 && j <= ny - 1 && c->open_v[id])
                val = c->vs[id] - dt * ((c->phi[PI_(c, i, j)] - c->phi[PI_(c, i, j - 1)]) / c->hyc[j]);
            c->v[id] = val;
        }
    for (size_t id = 0; id < np; ++id)
        if (c->act[id]) c->p[id] = c->p[id] + c->phi[id];
    /* R17b: an inactive cell with at least one active 4-neighbour takes the mean of
     * their p^{n+1} (E, W, N, S order, left fold); deeper inactive cells keep p.  Reads
     * active cells only, so the result does not depend on the loop order. */
    ORC_PAR
    for (int j = 0; j < ny; ++j)
        for (int i = 0; i < nx; ++i) {
            if (c->act[PI_(c, i, j)]) continue;
            static const int di[4] = {1, -1, 0, 0}, dj[4] = {0, 0, 1, -1};
            double sum = 0.0;
            int cnt = 0;
            for (int d = 0; d < 4; ++d) {
                int in_ = i + di[d], jn = j + dj[d];
                if (in_ < 0 || jn < 0 || in_ >= nx || jn >= ny || !c->act[PI_(c, in_, jn)]) continue;
                sum = sum + c->p[PI_(c, in_, jn)];
                cnt = cnt + 1;
            }
            if (cnt > 0) c->p[PI_(c, i, j)] = sum / (double)cnt;
        }

    /* history rotation */
    memcpy(c->cu_prev, c->cu, nu * sizeof(double));
    memcpy(c->cv_prev, c->cv, nv * sizeof(double));
    c->have_hist = 1;

    tick(c, 5, &t0);
    /* a8: forces, S:352-360 (R20, R19b): F = -sum_{Solid u Forcing} f dV + (M^{n+1} - M^n)/dt,
     * the forcing summed over every node where the scheme replaces the momentum
     * equation, consistently with M (for unchanged tags F = sum_body (u_hat - u^n)/dt dV) */
    {
        double sfx = 0.0, sfy = 0.0;
        for (int j = 0; j < ny; ++j)
            for (int i = 1; i <= nx - 1; ++i)
                if (c->tu[UI(c, i, j)] != FLUID) sfx = sfx + c->fu[UI(c, i, j)] * (c->hxc[i] * c->dy[j]);
        for (int j = 1; j <= ny - 1; ++j)
            for (int i = 0; i < nx; ++i)
                if (c->tv[VI(c, i, j)] != FLUID) sfy = sfy + c->fv[VI(c, i, j)] * (c->dx[i] * c->hyc[j]);
        double Mx1, My1;
        solid_momentum(c, &Mx1, &My1);
        double Fx = -sfx + (Mx1 - c->Mx) / dt;
        double Fy = -sfy + (My1 - c->My) / dt;
        c->Mx = Mx1;
        c->My = My1;
        c->cd = 2.0 * Fx;
        c->cl = 2.0 * Fy;
    }

    c->step += 1;

    tick(c, 6, &t0);
    /* NaN guard */
    for (size_t id = 0; id < nu; ++id) if (!isfinite(c->u[id])) return ORC_ERR_DIVERGED;
    for (size_t id = 0; id < nv; ++id) if (!isfinite(c->v[id])) return ORC_ERR_DIVERGED;
    for (size_t id = 0; id < np; ++id) if (!isfinite(c->p[id])) return ORC_ERR_DIVERGED;
    return status;
}

/* stats: per step 8 doubles: t, it_uv, it_p, rho_uv, rho_p, cd, cl, status */
int orc_step(orc_ctx *c, int nsteps, double *stats)
{
    int worst = ORC_OK;
    for (int s = 0; s < nsteps; ++s) {
        int st = step_once(c);
        if (stats) {
            double *o = stats + 8 * s;
            o[0] = c->t; o[1] = c->it_uv; o[2] = c->it_p; o[3] = c->rho_uv; o[4] = c->rho_p;
            o[5] = c->cd; o[6] = c->cl; o[7] = st;
        }
        if (st == ORC_ERR_DIVERGED) return st;
        if (st > worst) worst = st;
    }
    return worst;
}

/* ---------------- field access for tests ---------------- */
/* which: 0 u, 1 v, 2 p, 3 phi, 4 fu, 5 fv, 6 q, 7 cu_prev, 8 cv_prev, 9 us, 10 vs, 11 bp,
 *        12 rhs_u, 13 rhs_v */
int orc_get(const orc_ctx *c, int which, double *out)
{
    size_t nu = (size_t)(c->nx + 1) * c->ny, nv = (size_t)c->nx * (c->ny + 1), np = (size_t)c->nx * c->ny;
    const double *src[] = {c->u, c->v, c->p, c->phi, c->fu, c->fv, c->q, c->cu_prev, c->cv_prev,
                           c->us, c->vs, c->bp, c->rhs_u, c->rhs_v};
    size_t n[] = {nu, nv, np, np, nu, nv, np, nu, nv, nu, nv, np, nu, nv};
    if (which < 0 || which > 13) return ORC_ERR_CONFIG;
    memcpy(out, src[which], n[which] * sizeof(double));
    return ORC_OK;
}

/* which: 0 tu, 1 tv, 2 tp, 3 act, 4 open_u, 5 open_v */
int orc_get_tags(const orc_ctx *c, int which, unsigned char *out)
{
    size_t nu = (size_t)(c->nx + 1) * c->ny, nv = (size_t)c->nx * (c->ny + 1), np = (size_t)c->nx * c->ny;
    const unsigned char *src[] = {c->tu, c->tv, c->tp, c->act, c->open_u, c->open_v};
    size_t n[] = {nu, nv, np, np, nu, nv};
    if (which < 0 || which > 5) return ORC_ERR_CONFIG;
    memcpy(out, src[which], n[which]);
    return ORC_OK;
}

/* accumulated region times (s) since the last call, Table 1 layout (see orc_ctx.tm); resets them */
void orc_timers(orc_ctx *c, double *out7)
{
    for (int r = 0; r < 7; ++r) { out7[r] = c->tm[r]; c->tm[r] = 0.0; }
}

void orc_forces(const orc_ctx *c, double *out3)
{
    out3[0] = c->t;
    out3[1] = c->cd;
    out3[2] = c->cl;
}

/* ---------------- operator entry points for pins ---------------- */
/* convection of given fields with the ctx's current tags */
void orc_convection(const orc_ctx *c, const double *u, const double *v, double *cu, double *cv)
{
    convection(c, u, v, cu, cv);
}

/* explicit L on family fam at every interior node (0 elsewhere) */
void orc_laplacian(const orc_ctx *c, int fam, const double *x, double *out)
{
    int ni = fam_ni(c, fam), nj = fam_nj(c, fam);
    for (int j = 0; j < nj; ++j)
        for (int i = 0; i < ni; ++i) {
            int interior = (fam == 0) ? (i >= 1 && i <= c->nx - 1) : (fam == 1) ? (j >= 1 && j <= c->ny - 1) : 1;
            out[(size_t)j * ni + i] = interior ? lap_at(c, fam, x, i, j) : 0.0;
        }
}

/* Poisson solve L phi = rhs on the ctx's current masks (built from the current
 * tags); phi in/out is the warm start.  Returns iterations. */
int orc_poisson(orc_ctx *c, const double *rhs, double *phi, double *rho, int *status)
{
    size_t np = (size_t)c->nx * c->ny;
    build_masks(c);
    double *b = dalloc(np);
    for (size_t id = 0; id < np; ++id) b[id] = c->act[id] ? -rhs[id] : 0.0;
    int it = poisson_solve(c, b, phi, rho, status);
    free(b);
    return it;
}

/* forcing target of node (i,j) of family fam with the ctx's current tags/body */
double orc_forcing_target(const orc_ctx *c, int fam, const double *x, int i, int j)
{
    const unsigned char *tag = fam == 0 ? c->tu : c->tv;
    double uB = fam == 0 ? 0.0 : c->vb;
    return forcing_target(c, fam, x, tag, i, j, uB);
}
