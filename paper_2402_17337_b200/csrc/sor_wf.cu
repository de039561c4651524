// Temporally blocked Poisson red-black SOR (kernel a6-wf): WM full
// red-black iterations (R1-R3) per HBM pass.
//
// Why: the one-iteration pass (sor.cu) is HBM-bound at 24 B per cell per
// iteration (x in, b in, x out).  Streaming WM iterations through registers
// moves the same 24 B per cell once per WM iterations.
//
// Decomposition: one warp = one work item = a strip of 64 stored columns
// (global i0 .. i0+63 with i0 = sx*OW - 2WM; the middle OW = 64 - 4WM columns
// are owned) x a segment of L owned rows [j0, j1).  The warp streams its strip
// in increasing j: row r enters a register window of W = 2WM+2 rows (lane l
// holds columns 2l, 2l+1), then half-sweep h = 0 .. 2WM-1 (red, black, red, ...)
// is applied to row r-1-h.  That is the oracle's sweep order restricted to the
// strip: half-sweep h at row r-1-h reads rows r-2-h .. r-h, which half-sweep
// h-1 has already finished (row r-h earlier in this step) and half-sweep h+1 has
// not yet touched (it reaches row r-2-h later in this step).  Every half-sweep
// invalidates one more column at each strip edge and one more row at each
// segment end (their outside neighbours are not updated here); those cells are
// recomputed by the neighbouring items and are never stored nor counted, so
// every stored value and every residual term is bit-identical to the oracle's.
//
// Rows arrive by TMA in chunks of W rows (x and b, 64 x W boxes; the TMA unit
// zero-fills outside the array, the oracle's "0 outside the family") into a
// per-warp double-buffered stage armed on an mbarrier.  Chunks whose rows are
// all inside the family, away from the body box and carry the segment's
// reference row coefficients take a check-free path with per-column
// reciprocals; the rest (domain edges, body, stretched rows) the predicated one.
// One warp per CTA (one work item), 8 per SM.
//
// Residual (APX): the max of the high word of |d|, a lower bound of rho whose
// stops are provisional and confirmed by the host's exact replay of the pass
// (sor_solve) -- single-slab and decomposed solves alike.
//
// Arithmetic: identical to sor.cu (R13).
#include <algorithm>
#include <climits>
#include <cmath>
#include <cstdlib>
#include <type_traits>
#include <utility>

#include "ibm_internal.h"
#include "sor_common.cuh"

namespace ibm {
namespace {

constexpr unsigned FULL = 0xffffffffu;
// One warp per CTA (measured, 8192^2 m = 3: 0.134 ms/iteration against 0.145 with
// 4 warps per CTA): a CTA's resources are released as soon as its one item is
// done, so slow items (body, edges) do not hold fast ones at the CTA barrier.
#ifndef WF_NW
#define WF_NW 1
#endif
constexpr int WNW = WF_NW;  // warps per CTA (independent work items)
constexpr int WNT = 32 * WNW;
// TMA stages per warp.  A window of W = 2WM+2 rows arrives as two halves of WM+1
// rows, each in its own stage (4 KB at WM = 3); four stages per warp (the 16 KB of
// the old two full-window stages).  Half hc is read by its own steps and -- the b
// of its last row -- by the first step of half hc+1; right after that step (behind
// a __syncwarp: every lane has consumed the values it read) its stage is refilled
// with half hc+4.  So no generic-proxy read of a stage is outstanding when the TMA
// (async proxy) overwrites it -- no cross-proxy write-after-read race and no proxy
// fence (MEMBAR.ALL.CTA + FENCE.VIEW.ASYNC.S, which would also drain the warp's
// stores) -- and three halves (3 x 4 - 1 = 11 rows) are in flight ahead of the one
// being computed (ncu: with one full window of lead, 33 % of the stall samples
// waited for TMA data).
#ifndef WF_NSTG
#define WF_NSTG 4
#endif
template <int WM>
__host__ __device__ constexpr int wf_nstg() {
  return WF_NSTG;
}
// prefetch distance of the four-columns-per-lane kernel below (half windows)
#ifndef WF_PD
#define WF_PD 2
#endif
constexpr int WPD = WF_PD;
#ifndef WF_NS
#define WF_NS 1
#endif
constexpr int NS = WF_NS;   // column pairs per lane: lane l holds pairs l + 32 st
constexpr int SC = 64 * NS;  // stored columns per strip
#ifndef WF_CPL_DEFAULT
#define WF_CPL_DEFAULT 2  // columns per lane of the fused pass (wf_cpl)
#endif

template <int WM>
struct __align__(128) WfStage {  // half a window: rows rb + h (WM+1) .. + WM
  double x[WM + 1][SC];
  double b[WM + 1][SC];
};
template <int WM>
constexpr size_t wf_smem() {
  return (size_t)WNW * wf_nstg<WM>() * (sizeof(WfStage<WM>) + sizeof(unsigned long long));
}
#ifndef WF_MINB
#define WF_MINB (8 / WF_NW)  // 8 resident warps per SM (255 registers per thread)
#endif
// resident CTAs per SM the register budget is sized for (shared memory permitting)
template <int WM>
constexpr int wf_min_blocks() {
  return (int)((220u * 1024u) / wf_smem<WM>()) < WF_MINB ? (int)((220u * 1024u) / wf_smem<WM>()) : WF_MINB;
}

// Per-lane column data of the columns gi = i0 + 2 (l + 32 st) + e.
struct WfCols {
  double aE[NS][2], aW[NS][2], sEW[NS][2], cD[NS][2], yu[NS][2];
  unsigned inm[NS][2];  // all ones if the column is inside the family's updatable range, else 0
};

// Horizontal neighbour outside the pair for element E of window slot Q of every
// pair set: E = 0 -> W from pair p-1 (.y); E = 1 -> E from pair p+1 (.x).  Pair
// 31 / 32 cross between the sets; the strip's outermost neighbours are junk
// (halo columns, never stored or counted).
template <int W, int Q, int E>
__device__ __forceinline__ void wf_nb(const double2 (&X)[NS][W], double (&nb)[NS]) {
  const int l = threadIdx.x & 31;
  if (E == 0) {
    const double t0 = __shfl_sync(FULL, X[0][Q].y, (l + 31) & 31);
    nb[0] = t0;
    if (NS == 2) {
      const double t1 = __shfl_sync(FULL, X[NS - 1][Q].y, (l + 31) & 31);
      nb[NS - 1] = (l == 0) ? t0 : t1;
    }
  } else {
    const double t0 = __shfl_sync(FULL, X[0][Q].x, (l + 1) & 31);
    if (NS == 2) {
      const double t1 = __shfl_sync(FULL, X[NS - 1][Q].x, (l + 1) & 31);
      nb[0] = (l == 31) ? t1 : t0;
      nb[NS - 1] = t1;
    } else {
      nb[0] = t0;
    }
  }
}

// One node update of the check-free path per pair set: element E of window
// slot Q.  EDGE: the strip reaches past the family's columns; cells outside keep
// their value and are not counted.
// Residual accumulation.  Exact (APX = false): max of the 64-bit pattern of |d|
// (LOP3 + 2 ISETP + 2 SEL per node).  Approximate (APX = true): max of the high
// 32 bits only (LOP3 + VIMNMX, which ptxas fuses pairwise into VIMNMX3); the pass
// then reports a lower bound LB = H << 32 <= rho, so a stop is only provisional
// and the host replays that pass with the exact one-iteration kernel (sor_solve).
#ifndef WF_RES2
#define WF_RES2 1
#endif
template <bool APX>
__device__ __forceinline__ void wf_acc(unsigned long long &t, double d, unsigned m) {
  if (APX && WF_RES2) {
    // Two accumulators in the halves of t, no sign clear: lo = signed max of the
    // high words (the largest positive d), hi = unsigned max (the largest-magnitude
    // negative d if there is one, else the largest positive); the magnitude bound
    // is max(lo, hi & 0x7fffffff) (wf_res_word).  One VIMNMX per node each, fused
    // pairwise into VIMNMX3, and no LOP3 where m is the constant all-ones mask.
    unsigned lo, hi;
    asm("mov.b64 {%0, %1}, %2;" : "=r"(lo), "=r"(hi) : "d"(d));
    hi &= m;
    const unsigned tp = (unsigned)max((int)(unsigned)t, (int)hi);
    const unsigned tn = max((unsigned)(t >> 32), hi);
    t = ((unsigned long long)tn << 32) | tp;
  } else if (APX) {
    unsigned lo, hi;
    asm("mov.b64 {%0, %1}, %2;" : "=r"(lo), "=r"(hi) : "d"(d));
    hi &= 0x7fffffffu & m;
    t = (unsigned long long)max((unsigned)t, hi);
  } else {
    const unsigned long long e = abs_bits_masked(d, m);
    t = e > t ? e : t;
  }
}
// comparable residual word of an accumulator: APX -> the high word H of max|d|
// (LB = H << 32 is a lower bound of rho), exact -> the bit pattern of max|d|
template <bool APX>
__device__ __forceinline__ unsigned long long wf_res_word(unsigned long long t) {
  if (APX && WF_RES2) return (unsigned long long)max((unsigned)t, (unsigned)(t >> 32) & 0x7fffffffu);
  return t;
}

// okm: all ones if the row is owned by the item, else 0 (an integer mask, not a
// predicate: ptxas schedules the runtime-ownership chunks as tightly as the
// all-owned ones then).
template <int W, int Q, int E, bool EDGE, bool APX>
__device__ __forceinline__ void wf_fast(double2 (&X)[NS][W], const double2 (&B)[NS][W], const WfCols &C, double aN,
                                        double aS, double omega, double omc, unsigned okm,
                                        unsigned long long (&tmax)[NS]) {
  constexpr int QN = (Q + 1) % W, QS = (Q + W - 1) % W;
  double nb[NS];
  wf_nb<W, Q, E>(X, nb);
#pragma unroll
  for (int st = 0; st < NS; ++st) {
    const double xE = E ? nb[st] : X[st][Q].y;
    const double xW = E ? X[st][Q].x : nb[st];
    const double xo = rd(X[st][Q], E), xN = rd(X[st][QN], E), xS = rd(X[st][QS], E);
    const double nm =
        __fma_rn(aN, xN, __fma_rn(C.aE[st][E], xE, __fma_rn(C.aW[st][E], xW, __fma_rn(aS, xS, rd(B[st][Q], E)))));
    const double d = __fma_rn(nm, C.yu[st][E], -xo);  // gs - x_old, one rounding (R13)
    const double xn = __fma_rn(omega, d, xo);
    wr(X[st][Q], E, (!EDGE || C.inm[st][E]) ? xn : xo);
    // |gs - xo| as a bit pattern (sign cleared on the integer pipe), 0 where not counted
    wf_acc<APX>(tmax[st], d, EDGE ? (okm & C.inm[st][E]) : okm);
  }
}

// One node update of the predicated path (domain edges, body flags, arbitrary
// row coefficients): the same per-cell logic as sor.cu's boundary tiles.
template <int W, int Q, int E, bool APX>
__device__ __forceinline__ void wf_slow(double2 (&X)[NS][W], const double2 (&B)[NS][W], const WfCols &C,
                                        const WfArgs &A, int r, int i0, bool hasf, double omega, double omc, bool own,
                                        unsigned long long (&tmax)[NS]) {
  constexpr int QN = (Q + 1) % W, QS = (Q + W - 1) % W;
  const int l = threadIdx.x & 31;
  const int gj = A.g.gj0 + r;
  double cN = 0.0, cS = 0.0;  // 0 outside the family (oracle: out-of-range coefficient)
  if (gj >= 0 && gj < A.g.NJ) {
    cN = A.cN[gj];
    cS = A.cS[gj];
  }
  double nb[NS];
  wf_nb<W, Q, E>(X, nb);
#pragma unroll
  for (int st = 0; st < NS; ++st) {
    const int gi = i0 + 2 * (l + 32 * st) + E;
    bool u = gi >= A.ui0 && gi < A.ui1 && gj >= A.uj0 && gj < A.uj1;
    uint8_t fl = 0;
    // rows past the stored ghost rows are never read: the cells there are junk
    // recomputation (never stored nor counted), treated as flag 0
    if (hasf && u && r >= -kGhost && r < A.g.nj + kGhost) fl = A.flag[A.g.off(gi, r)];
    u = u && !(fl & PF_INACTIVE);
    double aE = C.aE[st][E], aW = C.aW[st][E], aN = cN, aS = cS, aP;
    if (fl) {
      aE = (fl & PF_E) ? 0.0 : aE;
      aW = (fl & PF_W) ? 0.0 : aW;
      aN = (fl & PF_N) ? 0.0 : aN;
      aS = (fl & PF_S) ? 0.0 : aS;
      aP = ((aE + aW) + (aN + aS)) + C.cD[st][E];
    } else {
      aP = (C.sEW[st][E] + (cN + cS)) + C.cD[st][E];
    }
    const double xE = E ? nb[st] : X[st][Q].y;
    const double xW = E ? X[st][Q].x : nb[st];
    const double xo = rd(X[st][Q], E), xN = rd(X[st][QN], E), xS = rd(X[st][QS], E);
    const double nm = __fma_rn(aN, xN, __fma_rn(aE, xE, __fma_rn(aW, xW, __fma_rn(aS, xS, rd(B[st][Q], E)))));
    const double d = __fma_rn(nm, __drcp_rn(aP), -xo);
    if (u) {
      wr(X[st][Q], E, __fma_rn(omega, d, xo));
      if (own) wf_acc<APX>(tmax[st], d, 0xffffffffu);
    }
  }
}

// predicated global stores (no branch: the warp stays provably converged, so
// the shuffles of the next step need no divergence check and ptxas can
// interleave consecutive steps)
__device__ __forceinline__ void st_pred(bool p, double *a, double2 v) {
  asm volatile("{\n .reg .pred q;\n setp.ne.b32 q, %0, 0;\n @q st.global.v2.f64 [%1], {%2, %3};\n}\n" ::"r"((int)p),
               "l"(a), "d"(v.x), "d"(v.y)
               : "memory");
}
__device__ __forceinline__ void st_pred1(bool p, double *a, double v) {
  asm volatile("{\n .reg .pred q;\n setp.ne.b32 q, %0, 0;\n @q st.global.f64 [%1], %2;\n}\n" ::"r"((int)p), "l"(a),
               "d"(v)
               : "memory");
}

// compile-time loop: f(std::integral_constant<int, i>) for i = 0 .. N-1
template <class F, int... I>
__device__ __forceinline__ void sfor_impl(F &&f, std::integer_sequence<int, I...>) {
  (f(std::integral_constant<int, I>{}), ...);
}
template <int N, class F>
__device__ __forceinline__ void sfor(F &&f) {
  sfor_impl(f, std::make_integer_sequence<int, N>{});
}

// The W steps of one chunk (window slot q = row rb + q).  MODE 2: check-free
// interior strip; 1: check-free edge strip; 0: predicated.  OWN: every row the
// chunk touches is owned by the item (the residual needs no row test; halo
// lanes are dropped once per item).  rb is even and W is even, so the slot and
// the colour element of every half-sweep are compile-time constants.
// (Compile-time ownership classes for the first / last two chunks of a segment
// were measured 14 % slower overall: the extra rarely-run chunk bodies miss in
// the instruction cache.)
// Stage use: the chunk reads its two half-window stages SA, SB and, at step 0, the b row rb-1 from
// the previous half's stage Sp; the hooks wait for the second half's stage and
// refill a stage once it is no longer read (see wf_nstg).
template <int WM, int TP, int MODE, bool OWN, bool APX, class Hooks>
__device__ __forceinline__ void wf_chunk(double2 (&X)[NS][2 * WM + 2], double2 (&B)[NS][2 * WM + 2],
                                         const WfStage<WM> &SA, const WfStage<WM> &SB, const WfStage<WM> &Sp,
                                         const WfCols &C, const WfArgs &A, int rb, int j0, int j1, int i0,
                                         const bool (&lane_own)[NS], bool hasf, double cN0, double cS0,
                                         unsigned long long (&tmax)[WM][NS], Hooks &&hooks) {
  constexpr int W = 2 * WM + 2;
  const int l = threadIdx.x & 31;
  const double omega = A.omega, omc = A.omc;
  const long pitch = A.g.pitch;
  // stored row rb + q - 2WM of this lane's first pair (the second is 64 columns on)
  double *const ob = A.xout + (long)(rb - 2 * WM + kGhost) * pitch + (i0 + 2 * l);
  constexpr int CR = WM + 1;  // rows per half window (stage)
  sfor<W>([&](auto qc) {
    constexpr int q = decltype(qc)::value;
    if constexpr (q == CR) hooks.wait_second();  // second half's stage has landed
    // row rb+q enters the window; the b of row rb+q-1 (first needed in this step)
    // is read now rather than with its x one step earlier (one row less live)
    constexpr int qb = (q + W - 1) % W;
    const WfStage<WM> &Sx = q < CR ? SA : SB;
    const WfStage<WM> &Sb = q == 0 ? Sp : (q - 1 < CR ? SA : SB);
    constexpr int rx = q % CR, rbb = (q + W - 1) % W % CR;
#pragma unroll
    for (int st = 0; st < NS; ++st) {
      X[st][q] = *reinterpret_cast<const double2 *>(&Sx.x[rx][2 * (l + 32 * st)]);
      B[st][qb] = *reinterpret_cast<const double2 *>(&Sb.b[rbb][2 * (l + 32 * st)]);
    }
    sfor<2 * WM>([&](auto hc) {
      constexpr int h = decltype(hc)::value;
      constexpr int Q = ((q - 1 - h) % W + W) % W;  // slot of row rb + q - 1 - h
      constexpr int E = (TP + Q + h) & 1;           // red (h even): (i + j) even
      const int r = rb + q - 1 - h;
      [[maybe_unused]] const bool own = OWN || (r >= j0 && r < j1);
      // owned-row mask from the sign bits of r - j0 and j1 - 1 - r (no predicate)
      unsigned okm = 0xffffffffu;
      if (!OWN)  // (opaque to the compiler, which would otherwise turn it back into selects)
        asm("{\n .reg .b32 t;\n or.b32 t, %1, %2;\n shr.s32 t, t, 31;\n not.b32 %0, t;\n}"
            : "=r"(okm)
            : "r"(r - j0), "r"(j1 - 1 - r));
      if constexpr (MODE > 0)
        wf_fast<W, Q, E, MODE == 1, APX>(X, B, C, cN0, cS0, omega, omc, okm, tmax[h / 2]);
      else
        wf_slow<W, Q, E, APX>(X, B, C, A, r, i0, hasf, omega, omc, own, tmax[h / 2]);
    });
    // row rb + q - 2WM has received its last half-sweep: store the owned columns
    const int ro = rb + q - 2 * WM;
    const bool rowin = OWN || (ro >= j0 && ro < j1);
#pragma unroll
    for (int st = 0; st < NS; ++st) {
      const double2 v = X[st][((q - 2 * WM) % W + W) % W];
      const bool pair_in = MODE == 2 || i0 + 2 * (l + 32 * st) + 1 < A.g.ni;
      st_pred(rowin && lane_own[st] && pair_in, ob + q * pitch + 64 * st, v);
      if (MODE < 2) st_pred1(rowin && lane_own[st] && !pair_in, ob + q * pitch + 64 * st, v.x);
    }
    if constexpr (q == 0) hooks.after_first();  // the previous half's stage is no longer read
    if constexpr (q == CR) hooks.after_second();  // this window's first half: no longer read
  });
}

template <int WM, int TP, bool APX>
__global__ void __launch_bounds__(WNT, wf_min_blocks<WM>()) k_sor_wf(const __grid_constant__ WfArgs A) {
  constexpr int W = 2 * WM + 2, OW = SC - 4 * WM, NSTG = wf_nstg<WM>(), CR = WM + 1;
  constexpr unsigned kBytes = 2u * CR * SC * 8;  // one half window of x and b
  extern __shared__ __align__(1024) unsigned char smraw[];
  __shared__ unsigned long long wmax[WNW][WM];
  const int l = threadIdx.x & 31, w = threadIdx.x >> 5;
  WfStage<WM> *st = reinterpret_cast<WfStage<WM> *>(smraw) + w * NSTG;
  unsigned long long *bar =
      reinterpret_cast<unsigned long long *>(smraw + (size_t)WNW * NSTG * sizeof(WfStage<WM>)) + w * NSTG;
  unsigned long long tmax[WM][NS];
#pragma unroll
  for (int i = 0; i < WM; ++i)
#pragma unroll
    for (int s = 0; s < NS; ++s) tmax[i][s] = 0ull;
  // (one warp per CTA: the item is blockIdx.x, provably warp-uniform, so the TMA
  // coordinates below live in uniform registers)
  const int item = WNW == 1 ? (int)blockIdx.x : (int)blockIdx.x * WNW + w;
  if (item >= A.items && *(volatile int *)&A.ctl->k_done >= 0) return;  // (working warps: below)
  if (item < A.items) {
    const Geo &g = A.g;
    // strip-major item order (consecutive CTAs = the segments of one strip): the
    // warps streaming at the same time cover ~resident/segs strips over the whole
    // height; measured 5-6 % faster than segment-row-major at 8192^2 (DRAM
    // pattern).  IBM_WF_ORDER=0: segment-row-major; 1: scattered rows.
    int sx = item / A.segs, sy = item % A.segs;
    if (A.seg_mode == 1) {  // edge segments only (strip-major)
      const int ne = A.e_lo + A.e_hi, k = item % ne;
      sx = item / ne;
      sy = k < A.e_lo ? k : A.segs - A.e_hi + (k - A.e_lo);
    } else if (A.seg_mode == 2) {  // interior segments only
      const int ni_ = A.segs - A.e_lo - A.e_hi;
      sx = item / ni_;
      sy = A.e_lo + item % ni_;
    } else if (A.order == 0) {
      sx = item % A.strips;
      sy = item / A.strips;
    } else if (A.order == 1) {
      sx = item % A.strips;
      sy = (int)(((long)(item / A.strips) * A.order_mul) % A.segs);
    } else if (A.order == 3) {  // groups of order_g strips, segment-row-major inside a group
      const int gsz = A.order_g * A.segs, g0 = (item / gsz) * A.order_g, r = item % gsz;
      const int gw = min(A.order_g, A.strips - g0);
      sx = g0 + r % gw;
      sy = r / gw;
    }
    const int i0 = sx * OW - 2 * WM;  // global column of stored column 0
    const int j0 = sy * A.L;          // owned local rows [j0, j1)
    const int j1 = min(j0 + A.L, g.nj);
    const int rs = j0 - 2 * WM;       // first streamed row
    const int nch = ((j1 - j0) + 4 * WM + W - 1) / W;
    if (l == 0) {
      for (int s = 0; s < NSTG; ++s) mbar_init(&bar[s], 1);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    for (int hc = 0; hc < NSTG - 1 && hc < 2 * nch; ++hc)  // halves 0..2; half hc+3 is issued in half hc
      tma_load_pair_elect(&bar[hc], kBytes, &st[hc].x[0][0], &A.tmx, &st[hc].b[0][0], &A.tmb, i0,
                          rs + hc * CR + kGhost);
    // converged at an earlier iteration: nothing to do.  Tested after the first
    // TMA issue so that the control-word round trip does not delay the item's
    // first chunk; the loads in flight are waited for before leaving.
    if (*(volatile int *)&A.ctl->k_done >= 0) {
      for (int hc = 0; hc < NSTG - 1 && hc < 2 * nch; ++hc) mbar_wait_warp(&bar[hc], 0);
      return;
    }
    bool lane_own[NS];
#pragma unroll
    for (int s = 0; s < NS; ++s) {
      const int p = l + 32 * s;
      lane_own[s] = p >= WM && p <= 32 * NS - 1 - WM && i0 + 2 * p < g.ni;
    }
    const bool interior = i0 >= A.ui0 && i0 + SC <= A.ui1;
    const bool boxstrip = !A.box.empty() && i0 < A.box.i1 && i0 + SC > A.box.i0;
    // column coefficients (0 outside the family) and the reference row of the segment
    const int jr = min(max(g.gj0 + j0 + A.L / 2, 1), g.NJ - 2);
    const double cN0 = A.cN[jr], cS0 = A.cS[jr];
    WfCols C;
#pragma unroll
    for (int s = 0; s < NS; ++s)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int gi = i0 + 2 * (l + 32 * s) + e;
        const bool in = gi >= 0 && gi < g.ni;
        const double cE = in ? A.cE[gi] : 0.0, cW = in ? A.cW[gi] : 0.0;
        C.cD[s][e] = in ? A.cD[gi] : 0.0;
        C.aE[s][e] = cE;
        C.aW[s][e] = cW;
        C.sEW[s][e] = cE + cW;
        C.yu[s][e] = __drcp_rn((C.sEW[s][e] + (cN0 + cS0)) + C.cD[s][e]);
        C.inm[s][e] = (gi >= A.ui0 && gi < A.ui1) ? 0xffffffffu : 0u;
      }
    double2 X[NS][W], B[NS][W];
#pragma unroll
    for (int s = 0; s < NS; ++s)
#pragma unroll
      for (int q = 0; q < W; ++q) X[s][q] = B[s][q] = make_double2(0.0, 0.0);
    // Irregular rows of the item (outside the family, in the body box, or with
    // row coefficients other than the reference): the chunks whose rows
    // rb-2WM .. rb+W-2 meet [irr0, irr1] take the predicated path.
    // (unconditional loads of clamped rows, unrolled: the loads of several rows
    // are in flight together instead of one dependent L2 round trip per test)
    int irr0 = INT_MAX, irr1 = INT_MIN;
#pragma unroll 4
    for (int r = rs - 2 * WM + l; r <= rs + nch * W - 2; r += 32) {
      const int gj = g.gj0 + r;
      const int gjc = min(max(gj, 0), g.NJ - 1);
      const double cn = __ldg(A.cN + gjc), cs = __ldg(A.cS + gjc);
      const bool reg = (gj >= A.uj0) & (gj < A.uj1) & !(boxstrip & (r >= A.box.j0) & (r < A.box.j1)) &
                       (cn == cN0) & (cs == cS0);
      if (!reg) {
        irr0 = min(irr0, r);
        irr1 = max(irr1, r);
      }
    }
    irr0 = __reduce_min_sync(FULL, irr0);
    irr1 = __reduce_max_sync(FULL, irr1);
    for (int c = 0; c < nch; ++c) {
      const int hA = 2 * c, hB = hA + 1;  // this window's halves
      const int rb = rs + c * W;
      const bool fast = rb + W - 2 < irr0 || rb - 2 * WM > irr1;
      const bool hasf = boxstrip && rb + W - 2 >= A.box.j0 && rb - 2 * WM < A.box.j1;
      mbar_wait_warp(&bar[hA % NSTG], (hA / NSTG) & 1);
      const bool ownall = rb - 2 * WM >= j0 && rb + W - 2 < j1;
      // refill the stage of half h - 1 with half h + 3 once the first step of half h
      // has read its last b row (see wf_nstg; for h = 0 that stage only supplied
      // the b of the junk row rs - 1)
      auto refill = [&](int h) {
        __syncwarp();
        const int hn = h + NSTG - 1;
        if (hn < 2 * nch) {  // (warp-uniform)
          const int sr = hn % NSTG;
          tma_load_pair_elect(&bar[sr], kBytes, &st[sr].x[0][0], &A.tmx, &st[sr].b[0][0], &A.tmb, i0,
                              rs + hn * CR + kGhost);
        }
      };
      struct {
        decltype(refill) &rf;
        unsigned long long *bar;
        int hA, hB;
        __device__ void after_first() { rf(hA); }
        __device__ void wait_second() { mbar_wait_warp(&bar[hB % NSTG], (hB / NSTG) & 1); }
        __device__ void after_second() { rf(hB); }
      } hooks{refill, bar, hA, hB};
      const WfStage<WM> &SA = st[hA % NSTG], &SB = st[hB % NSTG], &Sp = st[(hA + NSTG - 1) % NSTG];
      if (fast && interior && ownall)
        wf_chunk<WM, TP, 2, true, APX>(X, B, SA, SB, Sp, C, A, rb, j0, j1, i0, lane_own, hasf, cN0, cS0, tmax, hooks);
      else if (fast && interior)
        wf_chunk<WM, TP, 2, false, APX>(X, B, SA, SB, Sp, C, A, rb, j0, j1, i0, lane_own, hasf, cN0, cS0, tmax, hooks);
      else if (fast)
        wf_chunk<WM, TP, 1, false, APX>(X, B, SA, SB, Sp, C, A, rb, j0, j1, i0, lane_own, hasf, cN0, cS0, tmax, hooks);
      else
        wf_chunk<WM, TP, 0, false, APX>(X, B, SA, SB, Sp, C, A, rb, j0, j1, i0, lane_own, hasf, cN0, cS0, tmax, hooks);
    }
  }
  // residual of each fused iteration: warp -> CTA -> atomicMax on its bit pattern
  // (halo pairs accumulated recomputed cells: dropped here)
#pragma unroll
  for (int i = 0; i < WM; ++i) {
    unsigned long long t = 0ull;
#pragma unroll
    for (int s = 0; s < NS; ++s) {
      const int p = l + 32 * s;
      if (p >= WM && p <= 32 * NS - 1 - WM) t = umax64(t, wf_res_word<APX>(tmax[i][s]));
    }
#pragma unroll
    for (int off = 16; off; off >>= 1) t = umax64(t, __shfl_xor_sync(FULL, t, off));
    if (l == 0) wmax[w][i] = APX ? t << 32 : t;  // APX: the lower bound LB = H << 32
  }
  __syncthreads();
  if (threadIdx.x == 0) {
#pragma unroll
    for (int i = 0; i < WM; ++i) {
      unsigned long long mx = 0;
#pragma unroll
      for (int v = 0; v < WNW; ++v) mx = umax64(mx, wmax[v][i]);
      if (mx) atomicMax(&A.rho_bits[A.k + i], mx);
    }
    // The stop decision is taken by k_sor_check, launched after the pass (after the
    // cross-slab reduction on decomposed grids): deciding in the pass's last CTA
    // needs a __threadfence per CTA, which waits for the CTA's outstanding stores
    // (ncu: ~5 % of the pass's stall samples at 8192^2).
  }
}

// ============================================================================
// Four contiguous columns per lane (CPL = 4): lane l holds the column pairs
// (4l, 4l+1) and (4l+2, 4l+3) of a 128-column strip (128 - 4WM owned instead of
// 64 - 4WM), so one half-sweep of a row needs one shuffle per two node updates
// (the pair at the lane's other end reads its neighbour from the lane itself)
// and the warp carries two independent updates per row and half-sweep.  The
// register window is the same W = 2WM+2 rows; it arrives by TMA in two halves of
// WM+1 rows (8 KB per half at WM = 3) so that three stages still fit eight warps
// per SM.  Arithmetic, colours and the order of every update are those of the
// CPL = 2 kernel above (and of the oracle): same FMA chain, same reciprocal.
constexpr int SC4 = 128;  // stored columns per strip
template <int WM>
struct __align__(128) Wf4Stage {
  double x[WM + 1][SC4];
  double b[WM + 1][SC4];
};
template <int WM>
constexpr size_t wf4_smem() {
  return (size_t)(WPD + 1) * (sizeof(Wf4Stage<WM>) + sizeof(unsigned long long));
}
template <int WM>
constexpr int wf4_min_blocks() {
  return (int)((220u * 1024u) / wf4_smem<WM>()) < 8 ? (int)((220u * 1024u) / wf4_smem<WM>()) : 8;
}

struct Wf4Cols {  // [pair st][element e] of the lane's columns gi = i0 + 4l + 2st + e
  double aE[2][2], aW[2][2], yu[2][2];
  unsigned inm[2][2];
};

// the four (W, E) neighbours of the two pairs' element E in window slot Q
template <int W, int Q, int E>
__device__ __forceinline__ void wf4_nb(const double2 (&X)[W][2], double (&xw)[2], double (&xe)[2]) {
  const int l = threadIdx.x & 31;
  if (E == 0) {  // columns 4l, 4l+2: west of 4l is lane l-1's column 4l-1
    xw[0] = __shfl_sync(FULL, X[Q][1].y, (l + 31) & 31);
    xe[0] = X[Q][0].y;
    xw[1] = X[Q][0].y;
    xe[1] = X[Q][1].y;
  } else {  // columns 4l+1, 4l+3: east of 4l+3 is lane l+1's column 4l+4
    xw[0] = X[Q][0].x;
    xe[0] = X[Q][1].x;
    xw[1] = X[Q][1].x;
    xe[1] = __shfl_sync(FULL, X[Q][0].x, (l + 1) & 31);
  }
}

template <int W, int Q, int E, bool EDGE, bool APX>
__device__ __forceinline__ void wf4_fast(double2 (&X)[W][2], const double2 (&B)[W][2], const Wf4Cols &C, double aN,
                                         double aS, double omega, unsigned okm, unsigned long long (&tmax)[2]) {
  constexpr int QN = (Q + 1) % W, QS = (Q + W - 1) % W;
  double xw[2], xe[2];
  wf4_nb<W, Q, E>(X, xw, xe);
#pragma unroll
  for (int st = 0; st < 2; ++st) {
    const double xo = rd(X[Q][st], E), xN = rd(X[QN][st], E), xS = rd(X[QS][st], E);
    const double nm = __fma_rn(aN, xN, __fma_rn(C.aE[st][E], xe[st], __fma_rn(C.aW[st][E], xw[st],
                                                                               __fma_rn(aS, xS, rd(B[Q][st], E)))));
    const double d = __fma_rn(nm, C.yu[st][E], -xo);  // gs - x_old, one rounding (R13)
    const double xn = __fma_rn(omega, d, xo);
    wr(X[Q][st], E, (!EDGE || C.inm[st][E]) ? xn : xo);
    wf_acc<APX>(tmax[st], d, EDGE ? (okm & C.inm[st][E]) : okm);
  }
}

template <int W, int Q, int E, bool APX>
__device__ __forceinline__ void wf4_slow(double2 (&X)[W][2], const double2 (&B)[W][2], const Wf4Cols &C,
                                         const WfArgs &A, int r, int i0, bool hasf, double omega, bool own,
                                         unsigned long long (&tmax)[2]) {
  constexpr int QN = (Q + 1) % W, QS = (Q + W - 1) % W;
  const int l = threadIdx.x & 31;
  const int gj = A.g.gj0 + r;
  double cN = 0.0, cS = 0.0;  // 0 outside the family (oracle: out-of-range coefficient)
  if (gj >= 0 && gj < A.g.NJ) {
    cN = A.cN[gj];
    cS = A.cS[gj];
  }
  double xw[2], xe[2];
  wf4_nb<W, Q, E>(X, xw, xe);
#pragma unroll
  for (int st = 0; st < 2; ++st) {
    const int gi = i0 + 4 * l + 2 * st + E;
    const bool in = gi >= 0 && gi < A.g.ni;
    bool u = gi >= A.ui0 && gi < A.ui1 && gj >= A.uj0 && gj < A.uj1;
    uint8_t fl = 0;
    // rows past the stored ghost rows are junk recomputation (never stored nor counted)
    if (hasf && u && r >= -kGhost && r < A.g.nj + kGhost) fl = A.flag[A.g.off(gi, r)];
    u = u && !(fl & PF_INACTIVE);
    const double cD = in ? __ldg(A.cD + gi) : 0.0;
    double aE = C.aE[st][E], aW = C.aW[st][E], aN = cN, aS = cS, aP;
    if (fl) {
      aE = (fl & PF_E) ? 0.0 : aE;
      aW = (fl & PF_W) ? 0.0 : aW;
      aN = (fl & PF_N) ? 0.0 : aN;
      aS = (fl & PF_S) ? 0.0 : aS;
      aP = ((aE + aW) + (aN + aS)) + cD;
    } else {
      aP = ((aE + aW) + (cN + cS)) + cD;
    }
    const double xo = rd(X[Q][st], E), xN = rd(X[QN][st], E), xS = rd(X[QS][st], E);
    const double nm = __fma_rn(aN, xN, __fma_rn(aE, xe[st], __fma_rn(aW, xw[st], __fma_rn(aS, xS, rd(B[Q][st], E)))));
    const double d = __fma_rn(nm, __drcp_rn(aP), -xo);
    if (u) {
      wr(X[Q][st], E, __fma_rn(omega, d, xo));
      if (own) wf_acc<APX>(tmax[st], d, 0xffffffffu);
    }
  }
}

// One half (HALF = 0: slots 0..WM, 1: slots WM+1..2WM+1) of the window of W rows
// rb .. rb+W-1; its rows come from stage S.
template <int WM, int TP, int MODE, bool OWN, bool APX, int HALF>
__device__ __forceinline__ void wf4_half(double2 (&X)[2 * WM + 2][2], double2 (&B)[2 * WM + 2][2],
                                         const Wf4Stage<WM> &S, const Wf4Stage<WM> &Sp, const Wf4Cols &C,
                                         const WfArgs &A, int rb, int j0,
                                         int j1, int i0, const bool (&lane_own)[2], bool hasf, double cN0, double cS0,
                                         unsigned long long (&tmax)[WM][2]) {
  constexpr int W = 2 * WM + 2, CR = WM + 1;
  const int l = threadIdx.x & 31;
  const double omega = A.omega;
  const long pitch = A.g.pitch;
  double *const ob = A.xout + (long)(rb - 2 * WM + kGhost) * pitch + (i0 + 4 * l);
  sfor<CR>([&](auto qc) {
    constexpr int qq = decltype(qc)::value;
    constexpr int q = HALF * CR + qq;  // window slot = row rb + q
    // row rb+q enters the window; b of row rb+q-1 (first needed now) is read now,
    // not with its x, which shortens its live range by one row (registers)
    constexpr int qb = (q + W - 1) % W;
#pragma unroll
    for (int st = 0; st < 2; ++st) {
      X[q][st] = *reinterpret_cast<const double2 *>(&S.x[qq][4 * l + 2 * st]);
      B[qb][st] = *reinterpret_cast<const double2 *>(qq == 0 ? &Sp.b[CR - 1][4 * l + 2 * st]
                                                              : &S.b[qq == 0 ? 0 : qq - 1][4 * l + 2 * st]);
    }
    sfor<2 * WM>([&](auto hc) {
      constexpr int h = decltype(hc)::value;
      constexpr int Q = ((q - 1 - h) % W + W) % W;  // slot of row rb + q - 1 - h
      constexpr int E = (TP + Q + h) & 1;           // red (h even): (i + j) even
      const int r = rb + q - 1 - h;
      [[maybe_unused]] const bool own = OWN || (r >= j0 && r < j1);
      unsigned okm = 0xffffffffu;
      if (!OWN)
        asm("{\n .reg .b32 t;\n or.b32 t, %1, %2;\n shr.s32 t, t, 31;\n not.b32 %0, t;\n}"
            : "=r"(okm)
            : "r"(r - j0), "r"(j1 - 1 - r));
      if constexpr (MODE > 0)
        wf4_fast<W, Q, E, MODE == 1, APX>(X, B, C, cN0, cS0, omega, okm, tmax[h / 2]);
      else
        wf4_slow<W, Q, E, APX>(X, B, C, A, r, i0, hasf, omega, own, tmax[h / 2]);
    });
    const int ro = rb + q - 2 * WM;  // row that has received its last half-sweep
    const bool rowin = OWN || (ro >= j0 && ro < j1);
#pragma unroll
    for (int st = 0; st < 2; ++st) {
      const double2 v = X[((q - 2 * WM) % W + W) % W][st];
      const bool pair_in = MODE == 2 || i0 + 4 * l + 2 * st + 1 < A.g.ni;
      st_pred(rowin && lane_own[st] && pair_in, ob + q * pitch + 2 * st, v);
      if (MODE < 2) st_pred1(rowin && lane_own[st] && !pair_in, ob + q * pitch + 2 * st, v.x);
    }
  });
}

template <int WM, int TP, int MODE, bool OWN, bool APX>
__device__ __forceinline__ void wf4_window(double2 (&X)[2 * WM + 2][2], double2 (&B)[2 * WM + 2][2],
                                           Wf4Stage<WM> *st, unsigned long long *bar, const Wf4Cols &C,
                                           const WfArgs &A, int c, int nhc, int rs, int rb, int j0, int j1, int i0,
                                           const bool (&lane_own)[2], bool hasf, double cN0, double cS0,
                                           unsigned long long (&tmax)[WM][2]) {
  constexpr int NSTG = WPD + 1, CR = WM + 1;
  constexpr unsigned kHalf = 2u * CR * SC4 * 8;
  const int l = threadIdx.x & 31;
  auto refill = [&](int hc) {
    __syncwarp();
    if (l == 0 && hc + WPD < nhc) {
      // stage of half-window hc - 1: every lane consumed its values before the __syncwarp
      const int h2 = hc + WPD, sr = h2 % NSTG;
      mbar_expect_tx(&bar[sr], kHalf);
      tma_load_2d(&st[sr].x[0][0], &A.tmx, i0, rs + h2 * CR + kGhost, &bar[sr]);
      tma_load_2d(&st[sr].b[0][0], &A.tmb, i0, rs + h2 * CR + kGhost, &bar[sr]);
    }
  };
  // (the first window's "previous" stage is its own: the b it supplies there
  // belongs to row rs-1, a junk row never stored nor counted)
  const int h0 = 2 * c, h1 = 2 * c + 1, hp = c > 0 ? h0 - 1 : h0;
  mbar_wait_warp(&bar[h0 % NSTG], (h0 / NSTG) & 1);
  wf4_half<WM, TP, MODE, OWN, APX, 0>(X, B, st[h0 % NSTG], st[hp % NSTG], C, A, rb, j0, j1, i0, lane_own, hasf, cN0,
                                      cS0, tmax);
  refill(h0);
  mbar_wait_warp(&bar[h1 % NSTG], (h1 / NSTG) & 1);
  wf4_half<WM, TP, MODE, OWN, APX, 1>(X, B, st[h1 % NSTG], st[h0 % NSTG], C, A, rb, j0, j1, i0, lane_own, hasf, cN0,
                                      cS0, tmax);
  refill(h1);
}

template <int WM, int TP, bool APX>
__global__ void __launch_bounds__(32, wf4_min_blocks<WM>()) k_sor_wf4(const __grid_constant__ WfArgs A) {
  constexpr int W = 2 * WM + 2, OW = SC4 - 4 * WM, NSTG = WPD + 1, CR = WM + 1;
  constexpr unsigned kHalf = 2u * CR * SC4 * 8;
  extern __shared__ __align__(1024) unsigned char smraw[];
  const int l = threadIdx.x & 31;
  Wf4Stage<WM> *st = reinterpret_cast<Wf4Stage<WM> *>(smraw);
  unsigned long long *bar = reinterpret_cast<unsigned long long *>(smraw + (size_t)NSTG * sizeof(Wf4Stage<WM>));
  unsigned long long tmax[WM][2];
#pragma unroll
  for (int i = 0; i < WM; ++i) tmax[i][0] = tmax[i][1] = 0ull;
  const int item = blockIdx.x;
  const Geo &g = A.g;
  int sx = item / A.segs, sy = item % A.segs;  // strip-major item order
  if (A.seg_mode == 1) {  // edge / interior subsets (decomposed grids), as in k_sor_wf
    const int ne = A.e_lo + A.e_hi, k = item % ne;
    sx = item / ne;
    sy = k < A.e_lo ? k : A.segs - A.e_hi + (k - A.e_lo);
  } else if (A.seg_mode == 2) {
    const int ni_ = A.segs - A.e_lo - A.e_hi;
    sx = item / ni_;
    sy = A.e_lo + item % ni_;
  } else if (A.order == 0) {
    sx = item % A.strips;
    sy = item / A.strips;
  }
  const int i0 = sx * OW - 2 * WM;  // global column of stored column 0
  const int j0 = sy * A.L;          // owned local rows [j0, j1)
  const int j1 = min(j0 + A.L, g.nj);
  const int rs = j0 - 2 * WM;       // first streamed row
  const int nwin = ((j1 - j0) + 4 * WM + W - 1) / W;
  const int nhc = 2 * nwin;
  if (l == 0) {
    for (int s = 0; s < NSTG; ++s) mbar_init(&bar[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (int h = 0; h < WPD && h < nhc; ++h) {
      mbar_expect_tx(&bar[h], kHalf);
      tma_load_2d(&st[h].x[0][0], &A.tmx, i0, rs + h * CR + kGhost, &bar[h]);
      tma_load_2d(&st[h].b[0][0], &A.tmb, i0, rs + h * CR + kGhost, &bar[h]);
    }
  }
  __syncwarp();
  if (*(volatile int *)&A.ctl->k_done >= 0) {  // converged at an earlier iteration
    for (int h = 0; h < WPD && h < nhc; ++h) mbar_wait_warp(&bar[h], 0);
    return;
  }
  bool lane_own[2];
#pragma unroll
  for (int s = 0; s < 2; ++s) {
    const int p = 2 * l + s;  // pair index in the strip
    lane_own[s] = p >= WM && p <= SC4 / 2 - 1 - WM && i0 + 2 * p < g.ni;
  }
  const bool interior = i0 >= A.ui0 && i0 + SC4 <= A.ui1;
  const bool boxstrip = !A.box.empty() && i0 < A.box.i1 && i0 + SC4 > A.box.i0;
  const int jr = min(max(g.gj0 + j0 + A.L / 2, 1), g.NJ - 2);
  const double cN0 = A.cN[jr], cS0 = A.cS[jr];
  Wf4Cols C;
#pragma unroll
  for (int s = 0; s < 2; ++s)
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int gi = i0 + 4 * l + 2 * s + e;
      const bool in = gi >= 0 && gi < g.ni;
      const double cE = in ? A.cE[gi] : 0.0, cW = in ? A.cW[gi] : 0.0, cD = in ? A.cD[gi] : 0.0;
      C.aE[s][e] = cE;
      C.aW[s][e] = cW;
      C.yu[s][e] = __drcp_rn(((cE + cW) + (cN0 + cS0)) + cD);
      C.inm[s][e] = (gi >= A.ui0 && gi < A.ui1) ? 0xffffffffu : 0u;
    }
  double2 X[W][2], B[W][2];
#pragma unroll
  for (int q = 0; q < W; ++q) X[q][0] = X[q][1] = B[q][0] = B[q][1] = make_double2(0.0, 0.0);
  int irr0 = INT_MAX, irr1 = INT_MIN;
#pragma unroll 4
  for (int r = rs - 2 * WM + l; r <= rs + nwin * W - 2; r += 32) {
    const int gj = g.gj0 + r;
    const int gjc = min(max(gj, 0), g.NJ - 1);
    const double cn = __ldg(A.cN + gjc), cs = __ldg(A.cS + gjc);
    const bool reg = (gj >= A.uj0) & (gj < A.uj1) & !(boxstrip & (r >= A.box.j0) & (r < A.box.j1)) &
                     (cn == cN0) & (cs == cS0);
    if (!reg) {
      irr0 = min(irr0, r);
      irr1 = max(irr1, r);
    }
  }
  irr0 = __reduce_min_sync(FULL, irr0);
  irr1 = __reduce_max_sync(FULL, irr1);
  for (int c = 0; c < nwin; ++c) {
    const int rb = rs + c * W;
    const bool fast = rb + W - 2 < irr0 || rb - 2 * WM > irr1;
    const bool hasf = boxstrip && rb + W - 2 >= A.box.j0 && rb - 2 * WM < A.box.j1;
    const bool ownall = rb - 2 * WM >= j0 && rb + W - 2 < j1;
    if (fast && interior && ownall)
      wf4_window<WM, TP, 2, true, APX>(X, B, st, bar, C, A, c, nhc, rs, rb, j0, j1, i0, lane_own, hasf, cN0, cS0, tmax);
    else if (fast && interior)
      wf4_window<WM, TP, 2, false, APX>(X, B, st, bar, C, A, c, nhc, rs, rb, j0, j1, i0, lane_own, hasf, cN0, cS0,
                                        tmax);
    else if (fast)
      wf4_window<WM, TP, 1, false, APX>(X, B, st, bar, C, A, c, nhc, rs, rb, j0, j1, i0, lane_own, hasf, cN0, cS0,
                                        tmax);
    else
      wf4_window<WM, TP, 0, false, APX>(X, B, st, bar, C, A, c, nhc, rs, rb, j0, j1, i0, lane_own, hasf, cN0, cS0,
                                        tmax);
  }
  // residual of each fused iteration: lanes -> warp -> atomicMax on the bit pattern
  // (halo pairs accumulated recomputed cells: dropped here); the stop decision is
  // k_sor_check's, after the pass
#pragma unroll
  for (int i = 0; i < WM; ++i) {
    unsigned long long t = 0ull;
#pragma unroll
    for (int s = 0; s < 2; ++s)
      if (2 * l + s >= WM && 2 * l + s <= SC4 / 2 - 1 - WM) t = umax64(t, wf_res_word<APX>(tmax[i][s]));
#pragma unroll
    for (int off = 16; off; off >>= 1) t = umax64(t, __shfl_xor_sync(FULL, t, off));
    if (l == 0 && t) atomicMax(&A.rho_bits[A.k + i], APX ? t << 32 : t);  // APX: LB = H << 32
  }
}

template <int WM, int TP, bool APX>
void wf4_prepare() {
  static bool done = false;
  if (!done) {
    cudaFuncSetAttribute(k_sor_wf4<WM, TP, APX>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)wf4_smem<WM>());
    done = true;
  }
}

template <int WM, bool APX>
void wf4_launch_tp(const WfArgs &a, cudaStream_t s) {
  if (a.g.gj0 & 1) {
    wf4_prepare<WM, 1, APX>();
    k_sor_wf4<WM, 1, APX><<<a.items, 32, wf4_smem<WM>(), s>>>(a);
  } else {
    wf4_prepare<WM, 0, APX>();
    k_sor_wf4<WM, 0, APX><<<a.items, 32, wf4_smem<WM>(), s>>>(a);
  }
}

template <int WM, int TP, bool APX>
int wf_blocks_per_sm() {
  static int per = 0;
  if (!per) {
    cudaFuncSetAttribute(k_sor_wf<WM, TP, APX>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)wf_smem<WM>());
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_sor_wf<WM, TP, APX>, WNT, wf_smem<WM>());
    if (per < 1) per = 1;
  }
  return per;
}

template <int WM, bool APX>
void wf_launch_tp(const WfArgs &a, cudaStream_t s) {
  const int grid = (a.items + WNW - 1) / WNW;
  if (a.g.gj0 & 1) {
    wf_blocks_per_sm<WM, 1, APX>();
    k_sor_wf<WM, 1, APX><<<grid, WNT, wf_smem<WM>(), s>>>(a);
  } else {
    wf_blocks_per_sm<WM, 0, APX>();
    k_sor_wf<WM, 0, APX><<<grid, WNT, wf_smem<WM>(), s>>>(a);
  }
}

// approximate residual on every solve: single slab (decision by the pass's last
// CTA) and decomposed (max over ranks of the bounds, k_sor_check with apx = 1);
// the exact instantiation (APX = false) is kept for experiments (WF_EXACT)
template <int WM>
cudaError_t wf_launch(const WfArgs &a, cudaStream_t s) {
#ifdef WF_EXACT
  constexpr bool kApx = false;
#else
  constexpr bool kApx = true;
#endif
  if (wf_cpl() == 4)
    wf4_launch_tp<WM, kApx>(a, s);
  else
    wf_launch_tp<WM, kApx>(a, s);
  return cudaGetLastError();
}

}  // namespace

// columns per lane of the fused pass (2: 64-column strips, 4: 128-column strips),
// fixed per process (the TMA boxes are built at init); IBM_WF_CPL overrides
int wf_cpl() {
  static const int cpl = [] {
    const char *e = std::getenv("IBM_WF_CPL");
    const int v = e ? std::atoi(e) : WF_CPL_DEFAULT;
    return v == 4 ? 4 : 2;
  }();
  return cpl;
}
int wf_box_rows(int m) { return m + 1; }  // half a window (both layouts)
#ifdef WF_EXACT
bool wf_approx() { return false; }
#else
bool wf_approx() { return true; }
#endif
int wf_box_cols() { return wf_cpl() == 4 ? SC4 : SC; }

// Strip / segment plan: segments of L owned rows, L = 64 for m = 2 and 256 for
// m >= 3, halved (down to 32 / 64) while the items would not fill two waves
// (measured on 8192^2, one warp per CTA, over 64..512: short segments
// balance the slower body / edge items over the waves, but every segment
// recomputes 4m halo rows and rounds its 2m+2-row chunks up, which costs more
// for deeper fusion; m = 3: 64 0.139, 128 0.134, 192 0.166, 240 0.143, 256 0.132,
// 512 0.142 ms/iteration -- not monotone, so re-measure for other grids;
// scripts/gpu_wf_rows.sh).  IBM_WF_ROWS overrides L for tuning; it is rounded up
// to even so colours stay compile-time.
namespace {
// SM count of the current device (cached per device ordinal)
int sm_count() {
  static int cache[64] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  int &sms = cache[dev & 63];
  if (!sms) {
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms < 1) sms = 1;
  }
  return sms;
}
// two waves of the 8 resident warps per SM
int wf_items_target() { return 2 * 8 * sm_count(); }
int wf_rows_default(int m) { return m == 2 ? 64 : 256; }
int wf_rows_min(int m) { return m == 2 ? 32 : 64; }
int wf_strips(int ni, int m) {
  const int sc = wf_box_cols();
  return (ni + sc - 4 * m - 1) / (sc - 4 * m);
}
}  // namespace

// The fused pass needs enough work items to fill the GPU at its shortest
// segments; below that (mid-size grids, e.g. the 6-18 lakh production meshes)
// the one-iteration pass with its 60 x 16 tiles is used instead.
bool wf_viable(int ni, int nj, int m) {
  return (long)wf_strips(ni, m) * ((nj + wf_rows_min(m) - 1) / wf_rows_min(m)) >= wf_items_target();
}

static int wf_static_rows(const Geo &g, int m) {
  const int strips = wf_strips(g.ni, m);
  int L = wf_rows_default(m);
  while (L > wf_rows_min(m) && (long)strips * ((g.nj + L - 1) / L) < wf_items_target()) L /= 2;
  return L;
}

// The static choice, half and twice it.  The pass time does not follow a simple
// model in L (8192^2, m = 3: 128 and 256 fast, 160 / 192 / 224 / 240 20-30 %
// slower, although 224 fills the last wave best), so sor_solve
// times the first fused passes of a run with each candidate and keeps the
// fastest; every L gives bit-identical iterates, so the tuning passes are real work.
std::vector<int> wf_candidates(const Geo &g, int m) {
  const int strips = wf_strips(g.ni, m);
  const int L0 = wf_static_rows(g, m);
  std::vector<int> c{L0};
  if (L0 / 2 >= wf_rows_min(m)) c.push_back(L0 / 2);
  if (2 * L0 <= 512 && (long)strips * ((g.nj + 2 * L0 - 1) / (2 * L0)) >= wf_items_target()) c.push_back(2 * L0);
  // (Wave-filling lengths -- L with items / warp slots just below an integer, e.g.
  // 140, 222, 284, 374 at 8192^2 -- were measured slower, 0.123-0.151 vs 0.113 ms per
  // iteration: the DRAM pattern of the concurrently streamed rows favours L = 2^k.)
  return c;
}

void wf_plan(WfArgs &a, int m, int L_force) {
  a.strips = wf_strips(a.g.ni, m);
  int L = L_force > 0 ? L_force : wf_static_rows(a.g, m);
  if (const char *e = std::getenv("IBM_WF_ROWS")) {
    const int v = std::atoi(e);
    if (v > 0) L = v;
  }
  if (L < 2) L = 2;
  L = (L + 1) & ~1;
  a.L = L;
  a.segs = (a.g.nj + L - 1) / L;
  a.items = a.strips * a.segs;
  // edge segments: streamed rows [j0 - 2m, j1 + 2m) leave the owned rows
  a.seg_mode = 0;
  a.e_lo = 0;
  a.e_hi = 0;
  for (int sy = 0; sy < a.segs; ++sy) {
    const int j0 = sy * L, j1 = std::min(j0 + L, a.g.nj);
    const bool edge = j0 - 2 * m < 0 || j1 + 2 * m > a.g.nj;
    if (edge && sy == a.e_lo) ++a.e_lo;
  }
  for (int sy = a.segs - 1; sy >= a.e_lo; --sy) {
    const int j0 = sy * L, j1 = std::min(j0 + L, a.g.nj);
    if (j0 - 2 * m < 0 || j1 + 2 * m > a.g.nj) ++a.e_hi; else break;
  }
  a.order = 2;
  if (const char *e = std::getenv("IBM_WF_ORDER")) a.order = std::atoi(e);
  a.order_g = 8;
  if (const char *e = std::getenv("IBM_WF_GROUP")) a.order_g = std::max(1, std::atoi(e));
  a.order_mul = 1;
  for (int mlt = a.segs / 2 + 1; mlt < a.segs; ++mlt) {  // a multiplier coprime to segs
    int x = mlt, y = a.segs;
    while (y) { const int t = x % y; x = y; y = t; }
    if (x == 1) { a.order_mul = mlt; break; }
  }
}

cudaError_t launch_sor_wf(const WfArgs &a, int m, cudaStream_t s) {
  switch (m) {
    case 2: return wf_launch<2>(a, s);
    case 3: return wf_launch<3>(a, s);
    case 4: return wf_launch<4>(a, s);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace ibm
