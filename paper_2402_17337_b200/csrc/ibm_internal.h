// Internal declarations of the B200 library (not part of the C ABI).
// Layout of every staggered family in HBM: row-major, x fastest,
// row pitch a multiple of 32 doubles (256 B, padded off 4 KB multiples), kGhost
// ghost rows below and above the slab's owned rows; out-of-range
// columns are never stored -- kernels treat them as 0 with coefficient 0,
// exactly like the oracle's out-of-range reads.
#pragma once
#include <cstddef>
#include <cstdint>
#include <string>
#include <map>
#include <vector>

#include <cuda.h>  // CUtensorMap (TMA descriptors); no libcuda link
#include <cuda_runtime.h>

#include "../../include/ibm.h"

namespace ibm {

// ghost rows per side: 2 for the one-iteration passes, 2m for a pass fusing m
// red-black iterations on a decomposed grid (m <= 4)
constexpr int kGhost = 8;
enum Tag : uint8_t { FLUID = 0, SOLID = 1, FORCING = 2 };
// Poisson cell flags; 0 = active cell with all four faces open (the default
// outside the body envelope box).  Closed bits are only set on interior faces.
enum PFlag : uint8_t { PF_INACTIVE = 1, PF_E = 2, PF_W = 4, PF_N = 8, PF_S = 16 };

struct Geo {
  int ni;      // columns of the family (global == local)
  int nj;      // owned rows of the slab
  int gj0;     // global row index of local row 0
  int NJ;      // global rows of the family
  long pitch;  // elements per stored row
  __host__ __device__ long off(int i, int jl) const { return (long)(jl + kGhost) * pitch + i; }
  __host__ __device__ long elems() const { return (long)(nj + 2 * kGhost) * pitch; }
};

struct BBox {  // half-open node-index box: global columns, LOCAL rows
  int i0, i1, j0, j1;
  __host__ __device__ bool contains(int i, int jl) const { return i >= i0 && i < i1 && jl >= j0 && jl < j1; }
  __host__ __device__ bool empty() const { return i0 >= i1 || j0 >= j1; }
};

// One family of one red-black SOR system (Poisson: phi; Helmholtz: u* or v*).
struct SorFam {
  CUtensorMap tmx;      // TMA map of the input iterate (box SW x SH)
  CUtensorMap tmb;      // TMA map of the right-hand side (box SW x SH-2)
  CUtensorMap tmc[5];   // 1-D maps of the coefficients: cE, cW, cD (box SW columns), cN, cS (box SH global rows)
  const double *xin;
  double *xout;
  double *xb[2];        // both ping-pong buffers (persistent cooperative solve)
  CUtensorMap tmxb[2];  // their TMA maps
  const double *b;
  const uint8_t *flag;  // pflags (Poisson) or tags (Helmholtz)
  Geo g;
  BBox box;
  const double *cE, *cW, *cD;  // per global column
  const double *cN, *cS;       // per global row
  int ui0, ui1, uj0, uj1;      // updatable global index ranges [ui0, ui1) x [uj0, uj1)
  int tiles_x, tiles_y;
};

struct SorCtl {  // per-solve device control block
  unsigned long long rho_final;  // bits of rho at k_done
  int k_done;                    // -1 until converged / stopped
  int status;                    // 0 converged, 1 maxit, 3 NaN, 4 provisional (k_sor_wf lower bound; host confirms)
  unsigned ticket;               // last-block counter
  int buf;                       // k_sor_tb: ping-pong buffer holding the result
  unsigned long long rho3[3];    // persistent (cooperative) solve: residual of iteration k in slot k % 3
};

struct SorArgs {
  SorFam f[2];
  int nfam;
  int helmholtz;  // 0: Poisson coefficients from flags; 1: beta * metric coefficients
  double beta, omega, omc, tol;
  int k, maxit, check_every;
  int total_tiles;
  unsigned long long *rho_bits;  // [maxit + 2], zeroed per solve
  SorCtl *ctl;
  int multi;  // 1: several slabs / ranks -> decision in k_sor_check after the reduction
  int fixup;  // 1: replay of iterations already decided (no early exit, no residual, no decision)
};

// Temporally blocked Poisson pass (sor_wf.cu): WM red-black iterations per HBM
// pass.  One warp = one work item = a strip of 64 stored columns (64 - 4 WM
// owned) x a segment of L owned rows, streamed top to bottom.
// Per-segment data of the fused pass (host-built for each slab and segment
// length, wf_seg_table): the segment's reference row coefficients and the range
// [irr0, irr1] of its streamed local rows that are irregular apart from the body
// box -- outside the family's updatable rows or with other row coefficients
// (irr0 > irr1: none).
struct WfSeg {
  double cN0, cS0;
  int irr0, irr1;
};
struct WfArgs {
  CUtensorMap tmx;      // iterate, box 64 x (2 WM + 2) rows
  CUtensorMap tmb;      // right-hand side, same box
  double *xout;
  const uint8_t *flag;  // Poisson cell flags
  Geo g;
  BBox box;             // body envelope (local rows)
  const double *cE, *cW, *cD, *cN, *cS;
  int ui0, ui1, uj0, uj1;
  int strips, segs, L, items;
  int order, order_mul, order_g;  // item -> (strip, segment) order: 2 strip-major (default), 0 row-major, 1 scattered
  // segment subset of this launch (decomposed grids overlap the halo exchange with
  // the interior): 0 all segments; 1 the edge segments -- the e_lo first and e_hi
  // last ones, whose streamed rows reach the ghost rows; 2 the interior ones
  int seg_mode, e_lo, e_hi;
  int multi;            // several slabs / ranks: the decision runs after the residual reduction
  double omega, omc, tol;
  int k, maxit, check_every;
  unsigned long long *rho_bits;
  SorCtl *ctl;
  const WfSeg *seg;     // [segs] (wf_seg_table for this slab and L)
  // Device-initiated halo: the pass also stores its output rows
  // [0, peer_rows) at peer_lo + (row + kGhost) * pitch -- the top ghost rows of the
  // slab below, in that slab's buffer for the next pass -- and rows [nj - peer_rows,
  // nj) at peer_hi + (row + kGhost) * pitch -- the bottom ghost rows of the slab
  // above (bases pre-offset by the host; nullptr: no such neighbour).  On one GPU
  // (loopback slabs) the neighbours are plain device buffers; across processes they
  // are CUDA-IPC mappings of the neighbours' buffers over NVLink.
  double *peer_lo, *peer_hi;
  int peer_rows;
};
constexpr int kWfMaxM = 4;  // fused iterations per pass: 2..kWfMaxM instantiated

// Persistent shared-memory-resident Poisson solve with m iterations per grid
// barrier (sor_tb.cu; mid-size grids, one slab).  One CTA per tile of tx x ty
// owned cells (ntx x nty tiles), for the whole solve.
struct TbArgs {
  double *xb[2];        // ping-pong iterate buffers
  const double *b;
  const uint8_t *flag;  // Poisson cell flags (valid inside box)
  Geo g;
  BBox box;
  const double *cE, *cW, *cD, *cN, *cS;
  int ui0, ui1, uj0, uj1;
  int tx, ty, ntx, nty, m;
  int rc;               // 1: reciprocal diagonals stored in shared memory, 0: recomputed per update
  int s0;               // buffer holding the initial iterate
  double omega, tol;
  int maxit, check_every;
  unsigned long long *rho_bits;
  SorCtl *ctl;
};
bool tb_plan(TbArgs &a, int nx, int nj, int m, int sms);
cudaError_t launch_sor_tb(const TbArgs &a, cudaStream_t st);

struct Metric {  // device pointers, global index space
  double *xn, *yn, *dx, *dy, *xc, *yc, *hxc, *hyc;
  double *cEu, *cWu, *cDu, *cNu, *cSu;
  double *cEv, *cWv, *cDv, *cNv, *cSv;
  double *cEp, *cWp, *cDp, *cNp, *cSp;
};

struct Body {
  int has;
  double a, b, x0, y0, hbar, k;
};

struct Slab {
  int rank;          // global slab index
  int pj0, pj1;      // owned global p rows
  Geo gu, gv, gp;
  double *u, *v, *p, *phi[2], *cu, *cv, *cup, *cvp, *us[2], *vs[2], *ru, *rv, *bp, *fu, *fv, *q;
  uint8_t *tu, *tv, *tp, *pf;
  BBox bu, bv, bpb;  // body envelope boxes (local rows incl. ghosts), empty without body
  double *red;       // force sums [4], then the 4 x 64 per-CTA parts of k_forces_part
  // TMA descriptors of the SOR operands (built once at init)
  CUtensorMap tm_phi[2], tm_bp, tm_us[2], tm_ru, tm_vs[2], tm_rv;
  CUtensorMap tm_wphi[2], tm_wbp;  // boxes of the temporally blocked Poisson pass (rows 2 wf_m + 2)
};

struct Ctx {
  ibm_config cfg;
  int nx, ny, nranks, device;
  int loopback;      // all slabs in this process (test mode: halos by device copies)
  cudaStream_t stream;
  Metric m;
  std::vector<Slab> sl;
  CUtensorMap tm_coef[3][5];  // [u, v, p][cE, cW, cD, cN, cS] (1-D TMA descriptors)
  unsigned long long *rho_bits;
  SorCtl *ctl;
  int *nanflag;
  double *h_xn, *h_yn;
  SorCtl *h_ctl;   // pinned
  double *h_red;   // pinned [4 * slabs]
  int *h_nan;      // pinned
  Body body;
  int phi_cur;
  int step, have_hist;
  double Mx, My;
  double last_t, last_cd, last_cl;
  int hint_uv, hint_p;
  int wf_m;         // Poisson iterations fused per HBM pass (1 = unfused k_sor)
  int wf_L;         // fused-pass segment length chosen by the online tuner (0: not yet)
  std::vector<double> h_cNp, h_cSp;  // host row coefficients of the p family (wf_seg_table)
  std::map<long, std::pair<std::vector<WfSeg>, WfSeg *>> wf_segs;  // (slab, L) -> host / device table
  int tb_m;         // iterations per grid barrier of the resident mid-grid solve (0: not used)
  TbArgs tb;        // its tile plan (built at init)
  cudaEvent_t tev[24];  // tuner: start / stop of the first fused passes of a run (12 passes)
  int launches;     // kernels launched in the current step
  cudaEvent_t ev[8];
  void *nccl;      // ncclComm_t when nranks > 1 and !loopback
  void *nccl_halo; // its split for the halo exchanges on the comm stream (overlapped with the pass)
  cudaStream_t comm;      // halo-exchange stream of the decomposed fused pass (nranks > 1 or loopback)
  cudaEvent_t ev_edge, ev_halo;  // edge items of a pass done / its output's halo rows exchanged
  // Device-initiated halo of the fused Poisson pass (WfArgs::peer_*): on for
  // loopback slabs, and across ranks when every rank mapped its neighbours' phi
  // buffers by CUDA IPC at init (peer_phi[side][buffer], side 0 = rank - 1,
  // 1 = rank + 1; peer_nj = their owned rows); IBM_PEER_HALO=0 turns it off.
  bool peer_halo;
  double *peer_phi[2][2];
  int peer_nj[2];
  void *peer_map[2];  // cudaIpcOpenMemHandle bases (closed in ibm_destroy)
  std::string err;
};

// kernel launchers (kernels.cu)
int launch_classify(const Ctx &c, const Slab &s, double yb);
int launch_pflags(const Ctx &c, const Slab &s);
int launch_predictor(const Ctx &c, const Slab &s, double yb, double vb);
int sor_grid(const SorArgs &a);
// persistent cooperative solve (small grids): whole SOR loop in one launch with a grid
// barrier per iteration; returns false when the problem does not fit one co-resident grid
bool sor_coop_fits(const SorArgs &a);
cudaError_t launch_sor_coop(const SorArgs &a, int s0, cudaStream_t st);
// TMA box of the SOR tile (x) and of its right-hand side (b)
constexpr int kSorBoxW = 64, kSorBoxHx = 20, kSorBoxHb = 18;
// 1-D box of the row coefficients cN, cS of a tile: the tile's SH = 20 rows from an
// even start row (one row earlier when the tile's first row is odd), 22 rows.  A
// TMA box must start 16-B aligned in its innermost dimension: an odd fp64 start
// (slabs with an odd first global row) raised "illegal instruction".
constexpr int kSorBoxRows1d = kSorBoxHx + 2;
constexpr int kSorTileX = 60, kSorTileY = 16;
void launch_sor_iteration(const SorArgs &a, cudaStream_t st, int grid);
// temporally blocked Poisson pass: rows of the TMA box, segment length, launch
int wf_lag();  // half-sweep lag of the fused pass (1 or 2; sor_wf.cu)
int wf_box_rows(int m);
bool wf_approx();  // the fused pass reports high-word residual bounds (stops are provisional)
int wf_box_cols();
void wf_plan(WfArgs &a, int m, int L_force = 0);
// segment lengths worth trying for this slab (the static choice first)
std::vector<int> wf_candidates(const Geo &g, int m);
// WfSeg of every segment of a plan (a.g, a.L, a.segs, a.uj0/uj1) from the host row coefficients
std::vector<WfSeg> wf_seg_table(const WfArgs &a, int m, const double *cN, const double *cS);
bool wf_viable(int ni, int nj, int m);
cudaError_t launch_sor_wf(const WfArgs &a, int m, cudaStream_t st);
void launch_sor_check(SorCtl *ctl, const unsigned long long *rho_bits, int k, int maxit, int check_every,
                      double tol, cudaStream_t st, int m = 1, int apx = 0);
int launch_outlet_fill(const Ctx &c, const Slab &s, double *us, const double *vs);
int launch_prhs(const Ctx &c, const Slab &s, const double *us, const double *vs, double *phi_start);
int launch_correct(const Ctx &c, const Slab &s, const double *us, const double *vs, const double *phi);
// R17b pressure extension into the inactive cells next to active ones (after launch_correct)
int launch_pext(const Ctx &c, const Slab &s, const double *phi);
int launch_forces(const Ctx &c, const Slab &s);
void launch_fill(double *p, const Geo &g, double val, cudaStream_t st);

}  // namespace ibm
