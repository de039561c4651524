/*
 * include/ibm.h -- C ABI of the B200-native hot path of the discrete-forcing
 * immersed-boundary fractional-step solver of arXiv 2402.17337 (2-D
 * incompressible flow past a plunging elliptic foil).
 *
 * The problem the calls follow (citations: P:NN = PAPER.md line, S:NN = SPEC.md):
 *   Eq. (3)  du/dt + div(uu) = -grad p + Re^-1 lap u + f
 *   Eq. (4)  div u - q = 0
 *   discrete forcing f and mass source q at points classified fluid/solid every
 *   step; finite-volume semi-implicit fractional step on a staggered
 *   grid, Adams-Bashforth convection + Crank-Nicolson diffusion;
 *   red-black Gauss-Seidel SOR for the velocity and pressure equations;
 *   plunge ybar = h sin(k t), ydot = k h cos(k t) (Eqs. 1-2).
 * The discretisation, boundary conditions and every reading of a silent or
 * ambiguous passage are written out in DESIGN.md §2-§3; the arithmetic is
 * identical (bit for bit on one GPU) to the CPU oracle in oracle/.
 *
 * Grid and layouts.  nx x ny cells; node coordinates xn[0..nx], yn[0..ny]
 * (strictly increasing, uniform or stretched).  Staggered (MAC) families, all
 * global row-major with x fastest:
 *   u [ny][nx+1] at (xn_i, yc_j),   v [ny+1][nx] at (xc_i, yn_j),
 *   p, phi, q [ny][nx] at (xc_i, yc_j),   tags: uint8 0 Fluid, 1 Solid, 2 Forcing.
 * With nranks > 1 the grid is split into slabs along y; each rank owns rows
 * [j0, j1) of every family (the last rank also owns v row ny) and
 * ibm_get_fields / ibm_set_fields transfer only those rows.
 *
 * Ownership.  The caller allocates the device workspace (ibm_workspace_size)
 * and keeps it alive until ibm_destroy; the caller owns the CUDA stream.  The
 * library owns the ctx, its metric arrays and (nranks > 1) the NCCL
 * communicator.  Host arrays passed in (xn, yn, fields) are copied during the
 * call.  Every call is stream-ordered on the stream given to ibm_init; calls
 * that return host data synchronise that stream.  A ctx is not thread-safe.
 *
 * Errors.  Every function returns an int status (enum below).  On an error the
 * state is left as it was at detection and ibm_last_error(ctx) names the cause.
 */
#ifndef IBM_H
#define IBM_H

#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

#ifndef IBM_API
#define IBM_API __attribute__((visibility("default")))
#endif

typedef struct ibm_ctx ibm_ctx; /* opaque; owned by the library */

enum {
    IBM_OK = 0,
    IBM_WARN_NOCONV = 1,   /* step completed; an SOR solve stopped at max_iters */
    IBM_ERR_CONFIG = 2,    /* invalid configuration or body (S:552 exit code 2) */
    IBM_ERR_DIVERGED = 3,  /* NaN/Inf in a residual or a field (S:309, S:552 exit code 3) */
    IBM_ERR_ARG = 4,       /* bad argument (NULL pointer, bad mask, short workspace) */
    IBM_ERR_CUDA = 5,      /* CUDA runtime failure */
    IBM_ERR_NCCL = 6,      /* NCCL failure or NCCL not available */
    IBM_ERR_STATE = 7      /* call out of order (e.g. step before init) */
};

/* field-selection bits for ibm_get_fields / ibm_set_fields; dst/src arrays are
 * indexed by bit position (dst[0] for IBM_U, dst[1] for IBM_V, ...). */
enum {
    IBM_U = 1u << 0, IBM_V = 1u << 1, IBM_P = 1u << 2, IBM_PHI = 1u << 3,
    IBM_FU = 1u << 4, IBM_FV = 1u << 5, IBM_Q = 1u << 6,
    IBM_TU = 1u << 7, IBM_TV = 1u << 8, IBM_TP = 1u << 9,      /* uint8 tags */
    IBM_CU_PREV = 1u << 10, IBM_CV_PREV = 1u << 11,            /* AB2 history C^{n-1} */
    IBM_NFIELDS = 12
};
enum { IBM_HOST = 0, IBM_DEVICE = 1 };

typedef struct {
    int nx, ny;                 /* global cells, >= 4 each */
    const double *xn, *yn;      /* host, nx+1 / ny+1 node coordinates (copied) */
    double Re, dt;              /* Reynolds number, time step */
    double omega_p, tol_p;      /* Poisson SOR relaxation in [1,2), tolerance on max|gs - x| */
    int maxit_p;                /* Poisson iteration cap (S:327 default 10000) */
    double omega_uv, tol_uv;    /* velocity (Helmholtz) SOR, S:327 defaults 1.2, 1e-8 */
    int maxit_uv;               /* velocity iteration cap (default 1000, reading R25) */
    int check_every;            /* convergence-test cadence in iterations (R4; default 1) */
    int rank, nranks;           /* slab decomposition along y; nranks = 1 for one GPU */
    const unsigned char *nccl_id; /* 128 B from ibm_nccl_unique_id (rank 0), NULL if nranks == 1 */
    int device;                 /* CUDA device ordinal */
    int sor_batch;              /* SOR iterations launched between convergence polls (0 = auto) */
    int loopback;               /* 1: all nranks slabs live in this ctx on one device, halos and
                                   reductions by device copies (decomposition test mode; rank
                                   ignored, get/set_fields cover the whole grid) */
    int sor_fuse;               /* Poisson red-black iterations fused per HBM pass (temporal
                                   blocking): 0 = default (3), 1 = one iteration
                                   per pass, 2..4; slabs of fewer than 2m rows use 1 */
} ibm_config;

typedef struct {
    int step;                   /* step index n+1 just completed */
    double t_bar;               /* t^{n+1} = (n+1) dt */
    int it_uv, it_p;            /* SOR iterations of the velocity / pressure solves */
    double rho_uv, rho_p;       /* final max-norm update |gs - x_old| (reading R2) */
    double cd, cl;              /* force coefficients of this step */
    float ms[8];                /* device ms (CUDA events on the solver stream): [0] classify+predictor,
                                   [1] uv-SOR (+ outlet fill), [2] Poisson rhs, [3] p-SOR, [4] correct,
                                   [5] forces, [6] of [0]: classification and Poisson masks (a1, the
                                   paper's "flagging", Table 1), [7] whole step */
    int status;                 /* IBM_OK / IBM_WARN_NOCONV / IBM_ERR_DIVERGED */
    int launches;               /* CUDA kernels this library launched for the step (incl.
                                   early-exit SOR iterations past convergence) */
} ibm_step_stats;

/* Bytes of device workspace ibm_init needs for this configuration. */
IBM_API int ibm_workspace_size(const ibm_config *cfg, size_t *bytes);

/* Rank 0 only: NCCL unique id (128 B) to broadcast to every rank before ibm_init.
 * Returns IBM_ERR_NCCL when the library was built without NCCL. */
IBM_API int ibm_nccl_unique_id(unsigned char out[128]);

/* Validates cfg (IBM_ERR_CONFIG: nx,ny < 4, non-monotone axes, Re or dt <= 0,
 * omega outside [1,2), tol <= 0, maxit < 1, rank/nranks inconsistent, slab of
 * fewer than 4 rows), carves d_workspace (>= ibm_workspace_size bytes, 256-B
 * aligned, device memory of cfg->device), uploads metric arrays and sets the
 * impulsive start u = 1, v = p = phi = 0 (R11) at step 0 with no body.
 * cuda_stream is a cudaStream_t (NULL = legacy default stream). */
IBM_API int ibm_init(const ibm_config *cfg, void *d_workspace, size_t bytes, void *cuda_stream,
             ibm_ctx **out);

/* Elliptic foil of semi-axes a (chord/2) and b (thickness/2), centre (x0, y0),
 * plunging ybar = h_bar sin(k t), ydot = k h_bar cos(k t) (Eqs. 1-2).
 * a = b is a cylinder (reading R22).  IBM_ERR_CONFIG if a, b, k <= 0, h_bar < 0,
 * or the body envelope [x0 +- a] x [y0 +- (b + h_bar)] is not inside the domain
 * by >= 3 cells.  Re-classifies at the current time and resets the solid
 * momentum used by the force time-derivative. */
IBM_API int ibm_set_body(ibm_ctx *ctx, double a, double b, double x0, double y0, double h_bar, double k);

/* Removes the body (uniform-flow and channel checks). */
IBM_API int ibm_clear_body(ibm_ctx *ctx);

/* Copies the selected fields (IBM_U, IBM_V, IBM_P, IBM_PHI, IBM_CU_PREV,
 * IBM_CV_PREV; other bits -> IBM_ERR_ARG) from host (where = IBM_HOST) or device
 * buffers in the global layouts above (this rank's rows only).  Does not change
 * the step counter: call ibm_set_step afterwards to restart the time history. */
IBM_API int ibm_set_fields(ibm_ctx *ctx, unsigned mask, const void *const *src, int where);

/* Sets the step counter n (time t = n dt) and whether C^{n-1} is valid
 * (have_history = 0 -> the next step uses Euler convection, reading R8);
 * re-classifies at t and recomputes the solid momentum. */
IBM_API int ibm_set_step(ibm_ctx *ctx, int step, int have_history);

/* Advances nsteps time steps (S:305-313 order).  stats (nullable)
 * receives one record per step.  Returns the worst status; stops at the first
 * IBM_ERR_DIVERGED, leaving the state of the diverged step. */
IBM_API int ibm_step(ibm_ctx *ctx, int nsteps, ibm_step_stats *stats);

/* Copies the selected fields of this rank's slab (rows [*j0, *j1) of the global
 * index space of each family) to caller buffers on the host or device.  j0/j1
 * (nullable) receive the p-row range. */
IBM_API int ibm_get_fields(ibm_ctx *ctx, unsigned mask, void *const *dst, int where, int *j0, int *j1);

/* out = {t_bar, c_d, c_l} of the last completed step (globally reduced). */
IBM_API int ibm_forces(ibm_ctx *ctx, double out[3]);

/* Runs exactly `iters` Poisson red-black iterations (tolerance ignored) on the
 * current right-hand side and masks -- the SOR micro-benchmark of DESIGN.md §7.
 * phi is left as computed.  rho_out (nullable) receives the last residual. */
IBM_API int ibm_poisson_iterate(ibm_ctx *ctx, int iters, double *rho_out);

/* Launch configuration the library chose, for reporting (bench roofline labels):
 *   IBM_QUERY_WF_M  Poisson red-black iterations per HBM pass (1 = the one-iteration
 *                   pass k_sor, 2..4 = the temporally blocked k_sor_wf)
 *   IBM_QUERY_WF_L  segment length (owned rows per work item) of the fused pass, 0
 *                   until the online tuner has chosen one
 *   IBM_QUERY_SLABS slabs held by this ctx (loopback: nranks, else 1)
 *   IBM_QUERY_TB_M  Poisson iterations per grid barrier of the resident persistent
 *                   solve used on mid-size single-slab grids (0 = not used)
 *   IBM_QUERY_PEER_HALO 1 if the decomposed fused Poisson pass stores its boundary
 *                   rows directly into the neighbouring slabs' ghost rows (loopback
 *                   slabs, or ranks whose neighbours' buffers were mapped by CUDA IPC;
 *                   SURVEY 8(f) f3; IBM_PEER_HALO=0 disables), 0 if the rows go
 *                   through NCCL send/recv
 * IBM_ERR_ARG for an unknown key or NULL pointers.  No device work. */
enum { IBM_QUERY_WF_M = 0, IBM_QUERY_WF_L = 1, IBM_QUERY_SLABS = 2, IBM_QUERY_TB_M = 3, IBM_QUERY_PEER_HALO = 4 };
IBM_API int ibm_query(const ibm_ctx *ctx, int key, int *out);

/* Human-readable cause of the last error on ctx (never NULL). */
IBM_API const char *ibm_last_error(const ibm_ctx *ctx);

/* Frees library-owned resources (not the caller's workspace or stream). */
IBM_API int ibm_destroy(ibm_ctx *ctx);

#ifdef __cplusplus
}
#endif
#endif /* IBM_H */
