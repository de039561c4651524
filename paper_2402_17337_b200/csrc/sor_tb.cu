// Persistent, shared-memory-resident, temporally blocked Poisson red-black SOR for
// mid-size grids (row a6; the paper's production meshes M1-M3,
// P:198, and BJ configs[1]/[3] up to ~1e6 cells).
//
// Why: on grids of 1e5-1e6 cells one red-black iteration is a few microseconds of
// work, and the launched passes (sor.cu) or the cooperative loop with one grid
// barrier per iteration (k_sor_coop) spend most of each iteration in launch /
// barrier latency (ncu, cylinder 512x384: 44 % CTA-barrier stalls, 9 us per
// iteration).  Here one cooperative launch runs the whole solve; each CTA owns one
// tile of the grid for the whole solve, keeps its right-hand side, cell flags and
// reciprocal diagonals in shared memory, and advances M red-black iterations per
// grid barrier: it reloads its tile with a halo of 2M cells from the global
// iterate of the previous block, applies 2M half-sweeps (red, black, ...) on a
// region that shrinks by one ring per half-sweep -- the redundant halo
// recomputation of the fused pass (sor_wf.cu) -- and stores its owned cells into
// the other global buffer.  Every stored value and every residual term is the
// oracle's (same updates in the same colour order; cells of one colour are
// independent within a half-sweep).
//
// Convergence: the residual of each of the M iterations (max |gs - x_old| on the
// uint64 bit pattern, owned cells only) is folded into rho_bits[k + i] by one
// atomicMax per CTA; after the grid barrier every CTA reads the M words and takes
// the same decision (first i with NaN, rho <= tol at a check iteration, or
// k + i = maxit).  A stop inside the block is made exact by replaying the block
// from its input buffer (intact: ping-pong per block) up to that iteration.
//
// Arithmetic (R13): n = fma(aN, xN, fma(aE, xE, fma(aW, xW, fma(aS,
// xS, b)))), d = fma(n, RN(1/aP), -x_old), x = fma(omega, d, x_old); aX = open ?
// cX : 0, aP = ((aE + aW) + (aN + aS)) + cD -- bit-identical to the oracle.
#include <algorithm>
#include <cooperative_groups.h>
#include <cstdint>

#include "ibm_internal.h"
#include "sor_common.cuh"

namespace ibm {
namespace {

constexpr int TBT = 256;  // threads per CTA (8 warps)
constexpr int TBW = TBT / 32;

struct TbLayout {  // byte offsets of the shared-memory arrays of one tile region RX x RY
  int RX, RY;
  size_t x, b, rc, fl, rp, cE, cW, cD, cN, cS, red, total;
};

// rc: the reciprocal diagonals are stored per cell (25 B per region cell) or, for
// regions too large for that, recomputed at every update (17 B per cell)
__host__ __device__ inline TbLayout tb_layout(int tx, int ty, int M, bool rc = true) {
  TbLayout L;
  L.RX = tx + 4 * M;
  L.RY = ty + 4 * M;
  const size_t n = (size_t)L.RX * L.RY;
  size_t o = 0;
  L.x = o;  o += n * 8;
  L.b = o;  o += n * 8;
  L.rc = o; o += rc ? n * 8 : 0;
  L.cE = o; o += (size_t)L.RX * 8;
  L.cW = o; o += (size_t)L.RX * 8;
  L.cD = o; o += (size_t)L.RX * 8;
  L.cN = o; o += (size_t)L.RY * 8;
  L.cS = o; o += (size_t)L.RY * 8;
  L.red = o; o += (size_t)TBW * 4 * 8;
  L.fl = o; o += (n + 15) / 16 * 16;
  L.rp = o; o += ((size_t)L.RY + 15) / 16 * 16;
  L.total = o;
  return L;
}

// flag byte in shared memory: the Poisson cell flags (PF_*) of the cell plus
// TB_UPD when the cell is updated by the solve (inside the updatable range, active)
constexpr uint8_t TB_UPD = 0x80;

struct TbCtx {
  double *x, *b, *rc, *cE, *cW, *cD, *cN, *cS;
  unsigned long long *red;
  uint8_t *fl;
  uint8_t *rp;  // per row: 1 if every cell of the row is updated with open faces (no flags to apply)
  int RX, RY, gi0, jl0, gj0;  // region origin: global column gi0, local row jl0 (global row gj0 + jl0)
};

// The region is RX = 64 columns wide (owned tx = 64 - 4M): lane l always holds
// the columns 2l and 2l+1, so in every row and half-sweep each lane updates
// exactly one cell (the one of the half-sweep's colour) and keeps the column
// coefficients of its two columns in registers.  Warp w takes rows w, w+8, ...
// Shared-memory rows are stored de-interleaved -- the 32 even columns, then the
// 32 odd ones -- so that the lanes' accesses to a cell and to each of its four
// neighbours are 32 consecutive doubles (no bank conflicts; the interleaved
// layout had 2-way conflicts on every access).
constexpr int TB_RX = 64;
__device__ __forceinline__ int tb_ix(int x, int y) { return y * TB_RX + ((x & 1) << 5) + (x >> 1); }

#ifndef TB_R
#define TB_R 2
#endif

// One half-sweep h (colour h & 1: red = (i + j) even) over rows h+1 .. RY-2-h.
// Rows of a warp are 8 apart, so the colour's column parity e (column 2 lane + e)
// is the same in all of them.  In the de-interleaved layout the cell is at
// y*64 + 32e + lane and its west / east neighbours at o - 1 + e / o + e with
// o = y*64 + 32(1-e) + lane.  Cells past the region's outermost ring are
// recomputed from stale halo values like every other halo cell (never stored or
// counted), so only x = 0 / 63 (lane 0 with e = 0, lane 31 with e = 1) are
// skipped.  Rows whose 64 cells are all updated with open faces (rp) take the
// flag-free path.  RES: fold |d| of owned cells into t.
template <bool RES, bool RC>
__device__ __forceinline__ void tb_half(const TbCtx &T, int h, int M, double omega, const double (&cE2)[2],
                                        const double (&cW2)[2], const double (&cD2)[2], unsigned long long &t) {
  constexpr int R = TB_R;  // rows per pass of a warp: their loads are issued before any store (ILP)
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int y0 = h + 1, y1 = T.RY - 2 - h;
  const int H = 2 * M;
  const int e = (T.gi0 + T.gj0 + T.jl0 + (h & 1) + y0 + w) & 1;
  const bool act = e ? lane != 31 : lane != 0;
  const bool lres = RES && lane >= H / 2 && lane < 32 - H / 2;  // owned columns (x in [H, 64-H))
  const double cE = e ? cE2[1] : cE2[0], cW = e ? cW2[1] : cW2[0], cD = e ? cD2[1] : cD2[0];
  const int offC = (e << 5) + lane, offO = ((e ^ 1) << 5) + lane + e;  // cell; east neighbour (west = -1)
  for (int yb = y0 + w; yb <= y1; yb += TBW * R) {
    double xo[R], nm[R], rcp[R];
    bool upd[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int y = min(yb + r * TBW, y1);  // (a duplicate of the last row when past it: not stored)
      const int iC = y * TB_RX + offC, iE = y * TB_RX + offO;
      double aE = cE, aW = cW, aN = T.cN[y], aS = T.cS[y];
      bool u = act && yb + r * TBW <= y1;
      if (!T.rp[y]) {
        const uint8_t f = T.fl[iC];
        u = u && (f & TB_UPD);
        aE = (f & PF_E) ? 0.0 : aE;
        aW = (f & PF_W) ? 0.0 : aW;
        aN = (f & PF_N) ? 0.0 : aN;
        aS = (f & PF_S) ? 0.0 : aS;
      }
      upd[r] = u;
      if (RC)
        rcp[r] = T.rc[iC];
      else  // the same IEEE operations as the stored reciprocal (setup below)
        rcp[r] = __drcp_rn(((aE + aW) + (aN + aS)) + cD);
      xo[r] = T.x[iC];
      nm[r] = __fma_rn(aN, T.x[iC + TB_RX],
                       __fma_rn(aE, T.x[iE], __fma_rn(aW, T.x[iE - 1], __fma_rn(aS, T.x[iC - TB_RX], T.b[iC]))));
    }
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int y = min(yb + r * TBW, y1);
      const int iC = y * TB_RX + offC;
      const double d = __fma_rn(nm[r], rcp[r], -xo[r]);
      if (upd[r]) {
        T.x[iC] = __fma_rn(omega, d, xo[r]);
        if (RES && lres && y >= H && y < T.RY - H) t = umax64(t, abs_bits(d));
      }
    }
  }
}

// value of the iterate at region cell (x, y) from global (0 outside the family / stored rows)
__device__ __forceinline__ double tb_src(const TbCtx &T, const double *__restrict__ src, const Geo &g, int x, int y) {
  const int gi = T.gi0 + x, jl = T.jl0 + y;
  return (gi >= 0 && gi < g.ni && jl >= -kGhost && jl < g.nj + kGhost) ? src[g.off(gi, jl)] : 0.0;
}

// load the region (ring = false) or only its halo ring of width H (ring = true:
// the owned cells in shared memory are already the block's input) from global
__device__ __forceinline__ void tb_load_x(const TbCtx &T, const double *__restrict__ src, const Geo &g, int H,
                                          bool ring) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int y = w; y < T.RY; y += TBW) {
    const bool full = !ring || y < H || y >= T.RY - H;
    if (!full && lane >= H / 2 && lane < 32 - H / 2) continue;  // owned columns of an owned row
    const int x = 2 * lane;
    T.x[tb_ix(x, y)] = tb_src(T, src, g, x, y);
    T.x[tb_ix(x + 1, y)] = tb_src(T, src, g, x + 1, y);
  }
}

// store the owned cells of the region (inside the family) into dst
__device__ __forceinline__ void tb_store_x(const TbCtx &T, double *__restrict__ dst, const Geo &g, int M) {
  const int H = 2 * M, lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (lane < H / 2 || lane >= 32 - H / 2) return;
  for (int y = H + w; y < T.RY - H; y += TBW) {
    const int x = 2 * lane, gi = T.gi0 + x, jl = T.jl0 + y;
    if (jl >= g.nj) break;
    double *row = dst + g.off(gi, jl);
    const double2 v = make_double2(T.x[tb_ix(x, y)], T.x[tb_ix(x + 1, y)]);
    if (gi + 1 < g.ni)
      *reinterpret_cast<double2 *>(row) = v;
    else if (gi < g.ni)
      row[0] = v.x;
  }
}

template <int M, bool RC>
__global__ void __launch_bounds__(TBT, 2) k_sor_tb(const __grid_constant__ TbArgs A) {
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  extern __shared__ __align__(16) unsigned char smraw[];
  const TbLayout L = tb_layout(A.tx, A.ty, M, RC);
  TbCtx T;
  T.x = reinterpret_cast<double *>(smraw + L.x);
  T.b = reinterpret_cast<double *>(smraw + L.b);
  T.rc = reinterpret_cast<double *>(smraw + L.rc);
  T.cE = reinterpret_cast<double *>(smraw + L.cE);
  T.cW = reinterpret_cast<double *>(smraw + L.cW);
  T.cD = reinterpret_cast<double *>(smraw + L.cD);
  T.cN = reinterpret_cast<double *>(smraw + L.cN);
  T.cS = reinterpret_cast<double *>(smraw + L.cS);
  T.red = reinterpret_cast<unsigned long long *>(smraw + L.red);
  T.fl = smraw + L.fl;
  T.rp = smraw + L.rp;
  T.RX = L.RX;  // == TB_RX (tb_plan)
  T.RY = L.RY;
  const Geo &g = A.g;
  const int H = 2 * M;
  const int bx = blockIdx.x % A.ntx, by = blockIdx.x / A.ntx;
  T.gi0 = bx * A.tx - H;
  T.jl0 = by * A.ty - H;
  T.gj0 = g.gj0;
  SorCtl *ctl = A.ctl;

  // ---- once per solve: coefficients, right-hand side, flags, reciprocal diagonals
  for (int x = threadIdx.x; x < T.RX; x += TBT) {
    const int gi = T.gi0 + x;
    const bool in = gi >= 0 && gi < g.ni;  // 0 outside the family (the oracle's out-of-range coefficient)
    T.cE[x] = in ? A.cE[gi] : 0.0;
    T.cW[x] = in ? A.cW[gi] : 0.0;
    T.cD[x] = in ? A.cD[gi] : 0.0;
  }
  for (int y = threadIdx.x; y < T.RY; y += TBT) {
    const int gj = T.gj0 + T.jl0 + y;
    const bool in = gj >= 0 && gj < g.NJ;
    T.cN[y] = in ? A.cN[gj] : 0.0;
    T.cS[y] = in ? A.cS[gj] : 0.0;
  }
  __syncthreads();
  {
    const int n = T.RX * T.RY;
    for (int id = threadIdx.x; id < n; id += TBT) {
      const int y = id / T.RX, x = id - y * T.RX;
      const int gi = T.gi0 + x, jl = T.jl0 + y, gj = T.gj0 + jl;
      const bool stored = gi >= 0 && gi < g.ni && jl >= -kGhost && jl < g.nj + kGhost;
      uint8_t f = 0;
      double bb = 0.0, rc = 0.0;
      if (stored) {
        bb = A.b[g.off(gi, jl)];
        if (A.box.contains(gi, jl)) f = A.flag[g.off(gi, jl)];
        const bool upd = gi >= A.ui0 && gi < A.ui1 && gj >= A.uj0 && gj < A.uj1 && !(f & PF_INACTIVE);
        if (upd) {
          const double aE = (f & PF_E) ? 0.0 : T.cE[x];
          const double aW = (f & PF_W) ? 0.0 : T.cW[x];
          const double aN = (f & PF_N) ? 0.0 : T.cN[y];
          const double aS = (f & PF_S) ? 0.0 : T.cS[y];
          rc = __drcp_rn(((aE + aW) + (aN + aS)) + T.cD[x]);
          f |= TB_UPD;
        }
      }
      const int si = tb_ix(x, y);
      T.b[si] = bb;
      if (RC) T.rc[si] = rc;
      T.fl[si] = f;
    }
  }

  // column coefficients of the lane's two columns (registers for the whole solve)
  double cE2[2], cW2[2], cD2[2];
  {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    __syncthreads();
    for (int e = 0; e < 2; ++e) {
      cE2[e] = T.cE[2 * lane + e];
      cW2[e] = T.cW[2 * lane + e];
      cD2[e] = T.cD[2 * lane + e];
    }
    for (int y = w; y < T.RY; y += TBW) {  // rows without flags to apply
      const bool plain = T.fl[tb_ix(2 * lane, y)] == TB_UPD && T.fl[tb_ix(2 * lane + 1, y)] == TB_UPD;
      const bool all = __all_sync(0xffffffffu, plain);
      if (lane == 0) T.rp[y] = all ? 1 : 0;
    }
    __syncthreads();
  }
  // ---- blocks of M iterations, one grid barrier each
  for (int k = 1;; k += M) {
    const int blk = (k - 1) / M;
    const int bin = (A.s0 + blk) & 1;
    tb_load_x(T, A.xb[bin], g, H, blk > 0);  // after the first block only the halo ring is stale
    __syncthreads();
    unsigned long long t[4] = {0ull, 0ull, 0ull, 0ull};
#pragma unroll
    for (int h = 0; h < 2 * M; ++h) {
      tb_half<true, RC>(T, h, M, A.omega, cE2, cW2, cD2, t[h >> 1]);
      __syncthreads();
    }
    tb_store_x(T, A.xb[bin ^ 1], g, M);
    // residuals: warp max -> CTA max -> one atomic per iteration
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
    for (int i = 0; i < M; ++i) {
      unsigned long long v = t[i];
#pragma unroll
      for (int off = 16; off; off >>= 1) v = umax64(v, __shfl_xor_sync(0xffffffffu, v, off));
      if (lane == 0) T.red[w * 4 + i] = v;
    }
    __syncthreads();
    if (threadIdx.x < M && k + (int)threadIdx.x <= A.maxit) {  // (later iterations are never decided on)
      unsigned long long mx = 0ull;
      for (int v = 0; v < TBW; ++v) mx = umax64(mx, T.red[v * 4 + threadIdx.x]);
      if (mx) atomicMax(&A.rho_bits[k + threadIdx.x], mx);
    }
    grid.sync();
    // every CTA takes the same decision from the same words
    int stop = -1;
    unsigned long long rbs = 0ull;
    int status = 0;
    unsigned long long rbw[4];
#pragma unroll
    for (int i = 0; i < M; ++i)  // (independent loads: one L2 round trip, not M)
      rbw[i] = (k + i <= A.maxit) ? *(volatile unsigned long long *)&A.rho_bits[k + i] : 0ull;
    for (int i = 0; i < M; ++i) {
      const int kk = k + i;
      const unsigned long long rb = rbw[i];
      const double rho = __longlong_as_double((long long)rb);
      const bool nan_ = isnan(rho);
      const bool conv = (kk % A.check_every == 0) && rho <= A.tol;
      if (nan_ || conv || kk >= A.maxit) {
        stop = i;
        rbs = rb;
        status = nan_ ? 3 : (conv ? 0 : 1);
        break;
      }
    }
    if (stop < 0) continue;
    if (stop < M - 1) {
      // exact stop inside the block: replay iterations k .. k + stop from the input
      __syncthreads();
      tb_load_x(T, A.xb[bin], g, H, false);
      __syncthreads();
      unsigned long long dummy = 0ull;
      for (int h = 0; h < 2 * (stop + 1); ++h) {
        tb_half<false, RC>(T, h, M, A.omega, cE2, cW2, cD2, dummy);
        __syncthreads();
      }
      tb_store_x(T, A.xb[bin ^ 1], g, M);
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      ctl->rho_final = rbs;
      ctl->status = status;
      ctl->buf = bin ^ 1;  // buffer holding the result
      ctl->k_done = k + stop;
    }
    return;
  }
}

template <int M, bool RC>
bool tb_fits_mr(const TbArgs &a, int *per_sm) {
  const TbLayout L = tb_layout(a.tx, a.ty, M, RC);
  if (L.total > 227 * 1024) return false;
  cudaFuncSetAttribute(k_sor_tb<M, RC>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L.total);
  int per = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_sor_tb<M, RC>, TBT, L.total) != cudaSuccess) return false;
  *per_sm = per;
  return per >= 1;
}
template <int M>
bool tb_fits_m(const TbArgs &a, int *per_sm) {
  return a.rc ? tb_fits_mr<M, true>(a, per_sm) : tb_fits_mr<M, false>(a, per_sm);
}

template <int M, bool RC>
cudaError_t tb_launch_mr(const TbArgs &a, cudaStream_t st) {
  const TbLayout L = tb_layout(a.tx, a.ty, M, RC);
  void *args[] = {const_cast<TbArgs *>(&a)};
  return cudaLaunchCooperativeKernel((void *)k_sor_tb<M, RC>, dim3(a.ntx * a.nty), dim3(TBT), args, L.total, st);
}
template <int M>
cudaError_t tb_launch_m(const TbArgs &a, cudaStream_t st) {
  return a.rc ? tb_launch_mr<M, true>(a, st) : tb_launch_mr<M, false>(a, st);
}

}  // namespace

// Tile plan: the smallest tiles (least redundant halo work) whose count fits the
// co-resident grid.  Returns false when the grid is too large for one resident
// tile per CTA (then the caller keeps the other Poisson paths).
bool tb_plan(TbArgs &a, int nx, int nj, int M, int sms) {
  if (M < 2 || M > 4) return false;
  a.m = M;
  const int tx = TB_RX - 4 * M;
  const int ntx = (nx + tx - 1) / tx;
  for (int variant = 0; variant < 4; ++variant) {  // (rc stored, 2/SM), (stored, 1), (recomputed, 2), (recomputed, 1)
    const int per = 2 - (variant & 1);
    const bool rc = variant < 2;
    const int cap = per * sms;
    if (ntx > cap) continue;
    const int nty0 = std::max(1, std::min(cap / ntx, nj / 8));  // tiles of >= 8 owned rows
    const int ty = (nj + nty0 - 1) / nty0, nty = (nj + ty - 1) / ty;
    TbArgs b = a;
    b.tx = tx;
    b.ty = ty;
    b.ntx = ntx;
    b.nty = nty;
    b.rc = rc ? 1 : 0;
    const TbLayout L = tb_layout(tx, ty, M, rc);
    if (L.total * per > 227 * 1024) continue;
    int got = 0;
    const bool ok = (M == 2) ? tb_fits_m<2>(b, &got) : (M == 3) ? tb_fits_m<3>(b, &got) : tb_fits_m<4>(b, &got);
    if (ok && got * sms >= ntx * nty) {
      a = b;
      return true;
    }
  }
  return false;
}

cudaError_t launch_sor_tb(const TbArgs &a, cudaStream_t st) {
  switch (a.m) {
    case 2: return tb_launch_m<2>(a, st);
    case 3: return tb_launch_m<3>(a, st);
    case 4: return tb_launch_m<4>(a, st);
  }
  return cudaErrorInvalidValue;
}

}  // namespace ibm
