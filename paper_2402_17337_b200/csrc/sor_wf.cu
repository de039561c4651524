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
// Rows arrive by TMA in half windows of W/2 rows (x and b, 64 x W/2 boxes; the
// TMA unit zero-fills outside the array, the oracle's "0 outside the family")
// into a per-warp ring of stages armed on mbarriers, issued by an elected lane.
// Chunks whose rows are all inside the family, away from the body box and carry
// the segment's reference row coefficients (host-built WfSeg table) take a
// check-free path with per-column reciprocals; the rest (domain edges, body,
// stretched rows) the predicated one.  One warp per CTA (one work item), 8 per SM.
// Decomposed grids: chunks that store a slab's boundary rows also store them
// into the neighbours' ghost rows (WfArgs::peer_*, device-initiated halo).
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
constexpr int WNT = 32;
// Half-sweep lag.  At step q (row rb + q enters the register window) half-sweep
// h = 0 .. 2WM-1 updates row rb + q - 1 - LAG h.  LAG = 1 is the oracle's sweep
// order restricted to the strip with every half-sweep one row behind the previous
// one: inside a step, half-sweep h reads the row half-sweep h-1 has just updated
// (its north neighbour), a chain of 2WM dependent updates per step.  LAG = 2 keeps
// the same dependences one step apart -- h at row R reads rows R-1 .. R+1, which
// h-1 updated in earlier steps (R+1 at step q-1) and h+1 has not touched yet (it
// reaches R+1 at step q+3) -- so the 2WM updates of a step are independent, at the
// cost of a deeper window (4WM+1 rows instead of 2WM+2) and 2WM-1 more streamed
// rows per item.  Both orders give every update the operands of the oracle's order
// (the same iterate, bit for bit).  Process-wide (the TMA box height depends on
// it): IBM_WF_LAG overrides WF_LAG_DEFAULT.  Measured (8192^2, m = 3, cold): LAG 2
// removes most dependency stalls (ncu "wait" 8.1 k -> 2.8-3.5 k samples) but its
// 84-update chunk bodies miss in the instruction cache (no_instruction 0.5 k ->
// 3.2-6.8 k) and its 3 stages of 7 rows wait longer for TMA data: 0.143-0.148 ms
// per iteration against 0.110 for LAG 1, which stays the default.
#ifndef WF_LAG_DEFAULT
#define WF_LAG_DEFAULT 1
#endif
constexpr int SC = 64;  // stored columns per strip (lane l holds columns 2l, 2l+1)
// Experiment knobs (build variants): WF_EARLYWAIT = 1 waits for both halves of a
// window at its first step (one wait per chunk: the chunk body is one basic block
// between the refills) instead of before its second half; WF_NSTG1 = stages per
// warp at LAG 1 (their lead is NSTG1 - 1 halves minus what EARLYWAIT takes).
#ifndef WF_EARLYWAIT
#define WF_EARLYWAIT 0
#endif
#ifndef WF_NSTG1
#define WF_NSTG1 4
#endif
template <int WM, int LAG>
struct WfGeo {
  static constexpr int DLO = 1 + LAG * (2 * WM - 1);  // last half-sweep's row = entering row - DLO
  static constexpr int W = (DLO + 2 + 1) & ~1;        // window rows (down to its south neighbour; even)
  static constexpr int CR = W / 2;                    // rows per TMA stage (half a window)
  // TMA stages per warp.  Half hc is read by its own steps and -- the b of its
  // last row -- by the first step of half hc+1; right after that step (behind a
  // __syncwarp: every lane has consumed the values it read) its stage is refilled
  // with half hc+NSTG.  So no generic-proxy read of a stage is outstanding when the
  // TMA (async proxy) overwrites it -- no cross-proxy write-after-read race and no
  // proxy fence (MEMBAR.ALL.CTA + FENCE.VIEW.ASYNC.S, which would also drain the
  // warp's stores) -- and NSTG-1 halves are in flight ahead of the one being
  // computed: 11 rows at LAG 1 (4 stages of 4 KB), 13 at LAG 2 (3 of 7 KB).
  static constexpr int NSTG = LAG == 1 ? WF_NSTG1 : 3;
};
template <int CR>
struct __align__(128) WfStage {  // half a window: CR rows of x and b
  double x[CR][SC];
  double b[CR][SC];
};
template <int WM, int LAG>
constexpr size_t wf_smem() {
  using G = WfGeo<WM, LAG>;
  return (size_t)G::NSTG * (sizeof(WfStage<G::CR>) + sizeof(unsigned long long));
}
// 8 resident warps per SM (255 registers per thread), shared memory permitting
template <int WM, int LAG>
constexpr int wf_min_blocks() {
  return (int)((220u * 1024u) / wf_smem<WM, LAG>()) < 8 ? (int)((220u * 1024u) / wf_smem<WM, LAG>()) : 8;
}
constexpr int NS = 1;  // column pairs per lane

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
// refill a stage once it is no longer read (see WfGeo::NSTG).
// H0, H1: the half-sweeps [H0, H1) this warp applies (all 2WM by default; the
// two-warp pipeline k_sor_ws splits them).  SINK 0: the rows leaving the window go
// to global memory; 1: to the next warp through hooks.emit (x and b of the row).
template <int WM, int LAG, int TP, int MODE, bool OWN, bool APX, class Hooks, bool PEER = false, int H0 = 0,
          int H1 = 2 * WM, int SINK = 0>
__device__ __forceinline__ void wf_chunk(double2 (&X)[NS][WfGeo<WM, LAG>::W], double2 (&B)[NS][WfGeo<WM, LAG>::W],
                                         const WfStage<WfGeo<WM, LAG>::CR> &SA, const WfStage<WfGeo<WM, LAG>::CR> &SB,
                                         const WfStage<WfGeo<WM, LAG>::CR> &Sp, const WfCols &C, const WfArgs &A,
                                         int rb, int j0, int j1, int i0, const bool (&lane_own)[NS], bool hasf,
                                         double cN0, double cS0, unsigned long long (&tmax)[WM][NS], Hooks &&hooks) {
  using G = WfGeo<WM, LAG>;
  constexpr int W = G::W, CR = G::CR, DLO = 1 + LAG * (H1 - H0 - 1);
  const int l = threadIdx.x & 31;
  const double omega = A.omega, omc = A.omc;
  const long pitch = A.g.pitch;
  // stored row rb + q - DLO of this lane's pair
  double *const ob = A.xout + (long)(rb - DLO + kGhost) * pitch + (i0 + 2 * l);
  sfor<W>([&](auto qc) {
    constexpr int q = decltype(qc)::value;
    if constexpr (q == (WF_EARLYWAIT ? 0 : CR)) hooks.wait_second();  // second half's stage has landed
    // row rb+q enters the window; the b of row rb+q-1 (first needed in this step)
    // is read now rather than with its x one step earlier (one row less live)
    constexpr int qb = (q + W - 1) % W;
    const WfStage<CR> &Sx = q < CR ? SA : SB;
    const WfStage<CR> &Sb = q == 0 ? Sp : (q - 1 < CR ? SA : SB);
    constexpr int rx = q % CR, rbb = (q + W - 1) % W % CR;
#pragma unroll
    for (int st = 0; st < NS; ++st) {
      X[st][q] = *reinterpret_cast<const double2 *>(&Sx.x[rx][2 * (l + 32 * st)]);
      B[st][qb] = *reinterpret_cast<const double2 *>(&Sb.b[rbb][2 * (l + 32 * st)]);
    }
    sfor<H1 - H0>([&](auto hc) {
      constexpr int h = H0 + decltype(hc)::value;
      constexpr int Q = ((q - 1 - LAG * (h - H0)) % W + W) % W;  // slot of row rb + q - 1 - LAG (h - H0)
      constexpr int E = (TP + Q + h) & 1;                         // red (h even): (i + j) even
      const int r = rb + q - 1 - LAG * (h - H0);
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
    // row rb + q - DLO has received its last half-sweep: store the owned columns
    const int ro = rb + q - DLO;
    const bool rowin = OWN || (ro >= j0 && ro < j1);
    if constexpr (SINK == 1) {
      hooks.emit(q - DLO, X[0][((q - DLO) % W + W) % W], B[0][((q - DLO) % W + W) % W]);
    } else {
#pragma unroll
    for (int st = 0; st < NS; ++st) {
      const double2 v = X[st][((q - DLO) % W + W) % W];
      const bool pair_in = MODE == 2 || i0 + 2 * (l + 32 * st) + 1 < A.g.ni;
      st_pred(rowin && lane_own[st] && pair_in, ob + q * pitch + 64 * st, v);
      if (MODE < 2) st_pred1(rowin && lane_own[st] && !pair_in, ob + q * pitch + 64 * st, v.x);
      if constexpr (PEER) {
        // boundary rows also go straight into the neighbours' ghost rows (f3)
        const long o = (long)(ro + kGhost) * pitch + (i0 + 2 * l) + 64 * st;
        const bool lo = A.peer_lo != nullptr && ro >= 0 && ro < A.peer_rows;
        const bool hi = A.peer_hi != nullptr && ro >= A.g.nj - A.peer_rows && ro < A.g.nj;
        const bool ok = rowin && lane_own[st];
        st_pred(ok && pair_in && lo, A.peer_lo + o, v);
        st_pred1(ok && !pair_in && lo, A.peer_lo + o, v.x);
        st_pred(ok && pair_in && hi, A.peer_hi + o, v);
        st_pred1(ok && !pair_in && hi, A.peer_hi + o, v.x);
      }
    }
    }
    if constexpr (q == 0) hooks.after_first();  // the previous half's stage is no longer read
    if constexpr (q == CR) hooks.after_second();  // this window's first half: no longer read
  });
}

// Work item (strip sx, segment sy) -> its stored columns and streamed rows.
struct WfItem {
  int i0;      // global column of stored column 0
  int j0, j1;  // owned local rows
  int rs;      // first streamed row
  int nch;     // chunks of W rows
  int sy;      // segment index (WfArgs::seg)
};
template <int WM, int LAG>
__device__ __forceinline__ WfItem wf_item(const WfArgs &A, int item) {
  constexpr int W = WfGeo<WM, LAG>::W, DLO = WfGeo<WM, LAG>::DLO, OW = SC - 4 * WM;
  // strip-major item order (consecutive items = the segments of one strip): the
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
  WfItem it;
  it.i0 = sx * OW - 2 * WM;
  it.j0 = sy * A.L;
  it.j1 = min(it.j0 + A.L, A.g.nj);
  it.rs = it.j0 - 2 * WM;
  // rows rs .. j1 - 1 + DLO enter the window (row j1 - 1 is stored when j1 - 1 + DLO enters)
  it.nch = ((it.j1 - it.j0) + 2 * WM + DLO + W - 1) / W;
  it.sy = sy;
  return it;
}

// One warp per CTA; CTA b takes the items b, b + gridDim.x, ... -- one item per
// CTA by default (gridDim.x = items; wf_persist).  The half-window stage ring runs
// on across a CTA's items: the refills near the end of an item already stream the
// first halves of the next one.  The per-item setup is one load of its segment's
// row data (WfArgs::seg, host-built) plus the lane's column coefficients.
template <int WM, int LAG, int TP, bool APX>
__global__ void __launch_bounds__(32, (wf_min_blocks<WM, LAG>())) k_sor_wf(const __grid_constant__ WfArgs A) {
  using Gm = WfGeo<WM, LAG>;
  constexpr int W = Gm::W, NSTG = Gm::NSTG, CR = Gm::CR, DLO = Gm::DLO;
  constexpr unsigned kBytes = 2u * CR * SC * 8;  // one half window of x and b
  extern __shared__ __align__(1024) unsigned char smraw[];
  const int l = threadIdx.x & 31;
  WfStage<CR> *st = reinterpret_cast<WfStage<CR> *>(smraw);
  unsigned long long *bar = reinterpret_cast<unsigned long long *>(smraw + (size_t)NSTG * sizeof(WfStage<CR>));
  unsigned long long tmax[WM][NS];
#pragma unroll
  for (int i = 0; i < WM; ++i)
#pragma unroll
    for (int s = 0; s < NS; ++s) tmax[i][s] = 0ull;
  const Geo &g = A.g;
  const int stride = gridDim.x;
  int item = blockIdx.x;  // (warp-uniform)
  if (l == 0) {
    for (int s = 0; s < NSTG; ++s) mbar_init(&bar[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  WfItem it = wf_item<WM, LAG>(A, item);
  for (int hc = 0; hc < NSTG - 1 && hc < 2 * it.nch; ++hc)  // the first NSTG-1 halves
    tma_load_pair_elect(&bar[hc], kBytes, &st[hc].x[0][0], &A.tmx, &st[hc].b[0][0], &A.tmb, it.i0,
                        it.rs + hc * CR + kGhost);
  // converged at an earlier iteration (host-batched passes): nothing to do.  Tested
  // after the first TMA issue so that the control-word round trip does not delay
  // the item's first chunk; the loads in flight are waited for before leaving.
  if (*(volatile int *)&A.ctl->k_done >= 0) {
    for (int hc = 0; hc < NSTG - 1 && hc < 2 * it.nch; ++hc) mbar_wait_warp(&bar[hc], 0);
    return;
  }
  double2 X[NS][W], B[NS][W];
#pragma unroll
  for (int s = 0; s < NS; ++s)
#pragma unroll
    for (int q = 0; q < W; ++q) X[s][q] = B[s][q] = make_double2(0.0, 0.0);
  int G = 0;  // ring index of the current item's half 0
  for (; item < A.items; item += stride) {
    const bool has_next = item + stride < A.items;
    const WfItem nx = wf_item<WM, LAG>(A, has_next ? item + stride : item);
    const int nh = 2 * it.nch, nhn = has_next ? 2 * nx.nch : 0;
    const int i0 = it.i0, j0 = it.j0, j1 = it.j1, rs = it.rs, nch = it.nch;
    bool lane_own[NS];
#pragma unroll
    for (int s = 0; s < NS; ++s) {
      const int p = l + 32 * s;
      lane_own[s] = p >= WM && p <= 32 * NS - 1 - WM && i0 + 2 * p < g.ni;
    }
    const bool interior = i0 >= A.ui0 && i0 + SC <= A.ui1;
    const bool boxstrip = !A.box.empty() && i0 < A.box.i1 && i0 + SC > A.box.i0;
    // the segment's reference row coefficients and its irregular streamed rows
    // (outside the family or other row coefficients; host-built), plus the body box
    const WfSeg sg = A.seg[it.sy];
    const double cN0 = sg.cN0, cS0 = sg.cS0;
    int irr0 = sg.irr0, irr1 = sg.irr1;
    if (boxstrip) {
      const int lo = max(A.box.j0, rs - DLO), hi = min(A.box.j1 - 1, rs + nch * W - 2);
      if (lo <= hi) {
        irr0 = min(irr0, lo);
        irr1 = max(irr1, hi);
      }
    }
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
    for (int c = 0; c < nch; ++c) {
      const int hA = 2 * c, hB = hA + 1;  // this window's halves
      const int rb = rs + c * W;
      // (rows the chunk updates: rb - DLO .. rb + W - 2)
      const bool fast = rb + W - 2 < irr0 || rb - DLO > irr1;
      const bool hasf = boxstrip && rb + W - 2 >= A.box.j0 && rb - DLO < A.box.j1;
      mbar_wait_warp(&bar[(G + hA) % NSTG], ((G + hA) / NSTG) & 1);
      const bool ownall = rb - DLO >= j0 && rb + W - 2 < j1;
      // refill the stage of half h - 1 with half h + 3 -- of this item, or of the
      // next one near the end of this one -- once the first step of half h has read
      // its last b row (see WfGeo::NSTG)
      auto refill = [&](int h) {
        __syncwarp();
        const int hn = h + NSTG - 1, sr = (G + hn) % NSTG;
        const bool own_h = hn < nh;
        const int hl = own_h ? hn : hn - nh;
        const bool go = own_h || hl < nhn;  // (warp-uniform)
        tma_load_pair_elect_if(go, &bar[sr], kBytes, &st[sr].x[0][0], &A.tmx, &st[sr].b[0][0], &A.tmb,
                               own_h ? i0 : nx.i0, (own_h ? rs : nx.rs) + hl * CR + kGhost);
      };
      struct {
        decltype(refill) &rf;
        unsigned long long *bar;
        int gA, gB;
        __device__ void after_first() { rf(gA); }
        __device__ void wait_second() { mbar_wait_warp(&bar[(gB) % NSTG], ((gB) / NSTG) & 1); }
        __device__ void after_second() { rf(gA + 1); }
      } hooks{refill, bar, hA, G + hB};
      const WfStage<CR> &SA = st[(G + hA) % NSTG], &SB = st[(G + hB) % NSTG],
                        &Sp = st[(G + hA + NSTG - 1) % NSTG];
      // chunks storing slab boundary rows with a neighbour to feed: the predicated
      // path with the peer stores (rows stored here: rb - DLO .. rb + W - 1 - DLO)
      const bool peer = (A.peer_lo != nullptr && rb - DLO < A.peer_rows) ||
                        (A.peer_hi != nullptr && rb + W - 1 - DLO >= g.nj - A.peer_rows);
      if (peer)
        wf_chunk<WM, LAG, TP, 0, false, APX, decltype(hooks) &, true>(X, B, SA, SB, Sp, C, A, rb, j0, j1, i0,
                                                                     lane_own, hasf, cN0, cS0, tmax, hooks);
      else if (fast && interior && ownall)
        wf_chunk<WM, LAG, TP, 2, true, APX>(X, B, SA, SB, Sp, C, A, rb, j0, j1, i0, lane_own, hasf, cN0, cS0, tmax, hooks);
      else if (fast && interior)
        wf_chunk<WM, LAG, TP, 2, false, APX>(X, B, SA, SB, Sp, C, A, rb, j0, j1, i0, lane_own, hasf, cN0, cS0, tmax, hooks);
      else if (fast)
        wf_chunk<WM, LAG, TP, 1, false, APX>(X, B, SA, SB, Sp, C, A, rb, j0, j1, i0, lane_own, hasf, cN0, cS0, tmax, hooks);
      else
        wf_chunk<WM, LAG, TP, 0, false, APX>(X, B, SA, SB, Sp, C, A, rb, j0, j1, i0, lane_own, hasf, cN0, cS0, tmax, hooks);
    }
    G += nh;
    it = nx;
  }
  // residual of each fused iteration over the CTA's items: lanes -> atomicMax on
  // its bit pattern (halo pairs accumulated recomputed cells: dropped here)
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
    // APX: the lower bound LB = H << 32.  The stop decision is k_sor_check's, after
    // the pass (after the cross-slab reduction on decomposed grids): deciding in the
    // pass's last CTA needs a __threadfence per CTA (ncu: ~5 % of the stall samples).
    if (l == 0 && t) atomicMax(&A.rho_bits[A.k + i], APX ? t << 32 : t);
  }
}

// ============================================================================
// Two-warp pipeline (IBM_WF_WS=1, experiment): one work item per CTA of two warps.
// Warp A streams the strip from the TMA stages and applies half-sweeps 0 .. WM-1;
// every row it has finished (x and its b) goes into a shared-memory ring of
// half-window stages; warp B streams the ring and applies half-sweeps WM .. 2WM-1,
// then stores.  Rows flow through A and then B in order, so every update sees the
// operands of the one-warp pass (the oracle's).  Each warp carries half the
// in-step dependency chain and about half the registers, so twice the warps are
// resident.  Ring flow control: full[s] (32 arrivals of A's lanes after they wrote
// the stage's 4 rows), empty[s] (32 arrivals of B's lanes after their last read).
#ifndef WS_NSTG
#define WS_NSTG 3
#endif
#ifndef WS_NR
#define WS_NR 3
#endif
#ifndef WS_MINB
#define WS_MINB 8
#endif
template <int WM>
constexpr size_t ws_smem() {
  using G = WfGeo<WM, 1>;
  return (size_t)(WS_NSTG + WS_NR) * sizeof(WfStage<G::CR>) + (WS_NSTG + 2 * WS_NR) * sizeof(unsigned long long);
}

template <int WM, int TP, bool APX>
__global__ void __launch_bounds__(64, WS_MINB) k_sor_ws(const __grid_constant__ WfArgs A) {
  using Gm = WfGeo<WM, 1>;
  constexpr int W = Gm::W, CR = Gm::CR, NSTG = WS_NSTG, NR = WS_NR, HA = WM;
  constexpr unsigned kBytes = 2u * CR * SC * 8;
  static_assert(CR == 4 && W == 8, "the ring assumes half windows of 4 rows");
  extern __shared__ __align__(1024) unsigned char smraw[];
  const int l = threadIdx.x & 31, warp = threadIdx.x >> 5;
  WfStage<CR> *st = reinterpret_cast<WfStage<CR> *>(smraw);
  WfStage<CR> *ring = st + NSTG;
  unsigned long long *tbar = reinterpret_cast<unsigned long long *>(ring + NR);
  unsigned long long *full = tbar + NSTG, *empty = full + NR;
  unsigned long long tmax[WM][NS];
#pragma unroll
  for (int i = 0; i < WM; ++i) tmax[i][0] = 0ull;
  const int item = blockIdx.x;
  const WfItem it = wf_item<WM, 1>(A, item);
  const Geo &g = A.g;
  if (threadIdx.x == 0) {
    for (int s = 0; s < NSTG; ++s) mbar_init(&tbar[s], 1);
    for (int s = 0; s < NR; ++s) {
      mbar_init(&full[s], 32);
      mbar_init(&empty[s], 32);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (warp == 0)
    for (int hc = 0; hc < NSTG - 1 && hc < 2 * it.nch; ++hc)
      tma_load_pair_elect(&tbar[hc], kBytes, &st[hc].x[0][0], &A.tmx, &st[hc].b[0][0], &A.tmb, it.i0,
                          it.rs + hc * CR + kGhost);
  if (*(volatile int *)&A.ctl->k_done >= 0) {  // converged earlier: drain the loads in flight
    if (warp == 0)
      for (int hc = 0; hc < NSTG - 1 && hc < 2 * it.nch; ++hc) mbar_wait_warp(&tbar[hc], 0);
    return;
  }
  const int i0 = it.i0, j0 = it.j0, j1 = it.j1, rs = it.rs, nch = it.nch;
  bool lane_own[NS];
  lane_own[0] = l >= WM && l <= 31 - WM && i0 + 2 * l < g.ni;
  const bool interior = i0 >= A.ui0 && i0 + SC <= A.ui1;
  const bool boxstrip = !A.box.empty() && i0 < A.box.i1 && i0 + SC > A.box.i0;
  const WfSeg sg = A.seg[it.sy];
  const double cN0 = sg.cN0, cS0 = sg.cS0;
  // rows this warp updates in a chunk at base rb: rb - DLO .. rb + W - 2
  const int DLO = warp == 0 ? HA : 2 * WM - HA;
  int irr0 = sg.irr0, irr1 = sg.irr1;
  if (boxstrip) {
    const int lo = max(A.box.j0, rs - 2 * WM), hi = min(A.box.j1 - 1, rs + nch * W - 2);
    if (lo <= hi) {
      irr0 = min(irr0, lo);
      irr1 = max(irr1, hi);
    }
  }
  WfCols C;
#pragma unroll
  for (int e = 0; e < 2; ++e) {
    const int gi = i0 + 2 * l + e;
    const bool in = gi >= 0 && gi < g.ni;
    const double cE = in ? A.cE[gi] : 0.0, cW = in ? A.cW[gi] : 0.0;
    C.cD[0][e] = in ? A.cD[gi] : 0.0;
    C.aE[0][e] = cE;
    C.aW[0][e] = cW;
    C.sEW[0][e] = cE + cW;
    C.yu[0][e] = __drcp_rn((C.sEW[0][e] + (cN0 + cS0)) + C.cD[0][e]);
    C.inm[0][e] = (gi >= A.ui0 && gi < A.ui1) ? 0xffffffffu : 0u;
  }
  double2 X[NS][W], B[NS][W];
#pragma unroll
  for (int q = 0; q < W; ++q) X[0][q] = B[0][q] = make_double2(0.0, 0.0);
  for (int c = 0; c < nch; ++c) {
    const int hA = 2 * c, hB = hA + 1;
    const int rb = rs + c * W;
    const bool fast = rb + W - 2 < irr0 || rb - DLO > irr1;
    const bool hasf = boxstrip && rb + W - 2 >= A.box.j0 && rb - DLO < A.box.j1;
    const bool ownall = rb - DLO >= j0 && rb + W - 2 < j1;
    if (warp == 0) {
      // ---- warp A: TMA stages in, half-sweeps 0 .. HA-1, finished rows into the ring
      mbar_wait_warp(&tbar[hA % NSTG], (hA / NSTG) & 1);
      auto refill = [&](int h) {
        __syncwarp();
        const int hn = h + NSTG - 1, sr = hn % NSTG;
        tma_load_pair_elect_if(hn < 2 * nch, &tbar[sr], kBytes, &st[sr].x[0][0], &A.tmx, &st[sr].b[0][0], &A.tmb,
                               i0, rs + hn * CR + kGhost);
      };
      // ring stages of the halves this chunk emits into: 2c-1 (tail), 2c, 2c+1 (head)
      struct HooksA {
        decltype(refill) *rf;
        unsigned long long *tbar, *full, *empty;
        double *rl;     // this lane's element of ring stage 0, row 0 (x)
        int sidx[3];    // ring stages of the halves this chunk emits into: 2c-1 (tail), 2c, 2c+1 (head)
        int hA, c, ewait1, ewait2;  // parities of the empty waits due for halves 2c, 2c+1 (< 0: none)
        __device__ __forceinline__ void after_first() { (*rf)(hA); }
        __device__ __forceinline__ void wait_second() {
          mbar_wait_warp(&tbar[(hA + 1) % NSTG], ((hA + 1) / NSTG) & 1);
        }
        __device__ __forceinline__ void after_second() { (*rf)(hA + 1); }
        // row rb + D (D = q - HA, a constant after inlining) leaves A: ring half
        // 2c + floor(D / 4), position D mod 4
        __device__ __forceinline__ void emit(int D, double2 vx, double2 vb) {
          constexpr int kStage = (int)(sizeof(WfStage<CR>) / sizeof(double)), kB = CR * SC;
          const int P = ((D % 4) + 4) % 4, KO = D >= 0 ? D / 4 : -1;
          if (KO < 0 && c == 0) return;  // (rows before the stream: nothing to hand over)
          const int si = sidx[KO + 1];
          if (P == 0 && KO == 0 && ewait1 >= 0) mbar_wait_warp_bounded(&empty[si], ewait1 & 1);
          if (P == 0 && KO == 1 && ewait2 >= 0) mbar_wait_warp_bounded(&empty[si], ewait2 & 1);
          double *px = rl + si * kStage + P * SC;
          *reinterpret_cast<double2 *>(px) = vx;
          *reinterpret_cast<double2 *>(px + kB) = vb;
          if (P == 3) mbar_arrive(&full[si]);
        }
      } hooks;
      hooks.rf = &refill;
      hooks.tbar = tbar;
      hooks.full = full;
      hooks.empty = empty;
      hooks.rl = &ring[0].x[0][2 * l];
      hooks.hA = hA;
      hooks.c = c;
#pragma unroll
      for (int k = 0; k < 3; ++k) hooks.sidx[k] = max(2 * c - 1 + k, 0) % NR;
      // (use u = kh / NR of a stage needs B's release of use u - 1: parity (u - 1) & 1)
      hooks.ewait1 = 2 * c >= NR ? (2 * c) / NR - 1 : -1;
      hooks.ewait2 = 2 * c + 1 >= NR ? (2 * c + 1) / NR - 1 : -1;
      const WfStage<CR> &SA = st[hA % NSTG], &SB = st[hB % NSTG], &Sp = st[(hA + NSTG - 1) % NSTG];
      if (fast && interior && ownall)
        wf_chunk<WM, 1, TP, 2, true, APX, HooksA &, false, 0, HA, 1>(X, B, SA, SB, Sp, C, A, rb, j0, j1, i0, lane_own,
                                                                    hasf, cN0, cS0, tmax, hooks);
      else if (fast && interior)
        wf_chunk<WM, 1, TP, 2, false, APX, HooksA &, false, 0, HA, 1>(X, B, SA, SB, Sp, C, A, rb, j0, j1, i0,
                                                                     lane_own, hasf, cN0, cS0, tmax, hooks);
      else if (fast)
        wf_chunk<WM, 1, TP, 1, false, APX, HooksA &, false, 0, HA, 1>(X, B, SA, SB, Sp, C, A, rb, j0, j1, i0,
                                                                     lane_own, hasf, cN0, cS0, tmax, hooks);
      else
        wf_chunk<WM, 1, TP, 0, false, APX, HooksA &, false, 0, HA, 1>(X, B, SA, SB, Sp, C, A, rb, j0, j1, i0,
                                                                     lane_own, hasf, cN0, cS0, tmax, hooks);
    } else {
      // ---- warp B: ring in, half-sweeps HA .. 2WM-1, rows out to global memory
      mbar_wait_warp_bounded(&full[hA % NR], (hA / NR) & 1);
      struct HooksB {
        unsigned long long *full, *empty;
        int hA;
        __device__ void after_first() {  // the previous half's ring stage is no longer read
          __syncwarp();
          if (hA > 0) mbar_arrive(&empty[(hA - 1) % NR]);
        }
        __device__ void wait_second() { mbar_wait_warp_bounded(&full[(hA + 1) % NR], ((hA + 1) / NR) & 1); }
        __device__ void after_second() {
          __syncwarp();
          mbar_arrive(&empty[hA % NR]);
        }
        __device__ void emit(int, double2, double2) {}
      } hooks{full, empty, hA};
      const WfStage<CR> &SA = ring[hA % NR], &SB = ring[hB % NR], &Sp = ring[(hA + NR - 1) % NR];
      if (fast && interior && ownall)
        wf_chunk<WM, 1, TP, 2, true, APX, HooksB &, false, HA, 2 * WM, 0>(X, B, SA, SB, Sp, C, A, rb, j0, j1, i0,
                                                                          lane_own, hasf, cN0, cS0, tmax, hooks);
      else if (fast && interior)
        wf_chunk<WM, 1, TP, 2, false, APX, HooksB &, false, HA, 2 * WM, 0>(X, B, SA, SB, Sp, C, A, rb, j0, j1, i0,
                                                                           lane_own, hasf, cN0, cS0, tmax, hooks);
      else if (fast)
        wf_chunk<WM, 1, TP, 1, false, APX, HooksB &, false, HA, 2 * WM, 0>(X, B, SA, SB, Sp, C, A, rb, j0, j1, i0,
                                                                           lane_own, hasf, cN0, cS0, tmax, hooks);
      else
        wf_chunk<WM, 1, TP, 0, false, APX, HooksB &, false, HA, 2 * WM, 0>(X, B, SA, SB, Sp, C, A, rb, j0, j1, i0,
                                                                           lane_own, hasf, cN0, cS0, tmax, hooks);
    }
  }
  // A: the last half it partly filled is complete as far as B needs it (the rows it
  // did not write lie past every stored row's dependency cone)
  if (warp == 0) {
    __syncwarp();
    mbar_arrive(&full[(2 * nch - 1) % NR]);
  }
#pragma unroll
  for (int i = 0; i < WM; ++i) {
    unsigned long long t = 0ull;
    if (l >= WM && l <= 31 - WM) t = wf_res_word<APX>(tmax[i][0]);
#pragma unroll
    for (int off = 16; off; off >>= 1) t = umax64(t, __shfl_xor_sync(FULL, t, off));
    if (l == 0 && t) atomicMax(&A.rho_bits[A.k + i], APX ? t << 32 : t);
  }
}

template <int WM, int LAG, int TP, bool APX>
int wf_blocks_per_sm() {
  static int per = 0;
  if (!per) {
    cudaFuncSetAttribute(k_sor_wf<WM, LAG, TP, APX>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)wf_smem<WM, LAG>());
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_sor_wf<WM, LAG, TP, APX>, WNT, wf_smem<WM, LAG>());
    if (per < 1) per = 1;
  }
  return per;
}

int sm_count();
// One CTA per item (default): the hardware hands a freed slot the next item in
// order, so the items streaming at the same time stay a compact range (DRAM
// pattern, L2 reuse of the overlapping strip columns).  IBM_WF_PERSIST=1: one CTA
// per resident slot taking every gridDim-th item, with the next item's first
// halves prefetched across the item boundary -- measured slower (8192^2: 0.156
// ms per iteration at the best L against 0.111): the static assignment lets the
// concurrently streamed items drift apart (27.9 % L2 hits against 32.8 %, and
// 24 % of the stall samples waiting for TMA data against 6 %).
static bool wf_persist() {
  static const bool p = [] {
    const char *e = std::getenv("IBM_WF_PERSIST");
    return e && std::atoi(e) == 1;
  }();
  return p;
}
static bool wf_ws() {
  static const bool p = [] {
    const char *e = std::getenv("IBM_WF_WS");
    return e && std::atoi(e) == 1;
  }();
  return p;
}
template <int WM, int TP, bool APX>
void ws_launch(const WfArgs &a, cudaStream_t s) {
  static bool done = false;
  if (!done) {
    cudaFuncSetAttribute(k_sor_ws<WM, TP, APX>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ws_smem<WM>());
    done = true;
  }
  k_sor_ws<WM, TP, APX><<<a.items, 64, ws_smem<WM>(), s>>>(a);
}
template <int WM, int LAG, bool APX>
void wf_launch_tp(const WfArgs &a, cudaStream_t s) {
  if constexpr (LAG == 1 && WM == 3) {
    if (wf_ws() && !a.peer_lo && !a.peer_hi) {
      if (a.g.gj0 & 1)
        ws_launch<WM, 1, APX>(a, s);
      else
        ws_launch<WM, 0, APX>(a, s);
      return;
    }
  }
  if (a.g.gj0 & 1) {
    const int grid = wf_persist() ? std::min(a.items, wf_blocks_per_sm<WM, LAG, 1, APX>() * sm_count()) : a.items;
    wf_blocks_per_sm<WM, LAG, 1, APX>();
    k_sor_wf<WM, LAG, 1, APX><<<grid, WNT, wf_smem<WM, LAG>(), s>>>(a);
  } else {
    const int grid = wf_persist() ? std::min(a.items, wf_blocks_per_sm<WM, LAG, 0, APX>() * sm_count()) : a.items;
    wf_blocks_per_sm<WM, LAG, 0, APX>();
    k_sor_wf<WM, LAG, 0, APX><<<grid, WNT, wf_smem<WM, LAG>(), s>>>(a);
  }
}

// approximate residual on every solve: single slab and decomposed (max over ranks
// of the bounds, k_sor_check with apx = 1); the exact instantiation (APX = false)
// is kept for experiments (WF_EXACT)
template <int WM>
cudaError_t wf_launch(const WfArgs &a, cudaStream_t s) {
#ifdef WF_EXACT
  constexpr bool kApx = false;
#else
  constexpr bool kApx = true;
#endif
  if (wf_lag() == 2)
    wf_launch_tp<WM, 2, kApx>(a, s);
  else
    wf_launch_tp<WM, 1, kApx>(a, s);
  return cudaGetLastError();
}

}  // namespace

// half-sweep lag of the fused pass (1 or 2), fixed per process (the TMA box height
// is built at init); IBM_WF_LAG overrides
int wf_lag() {
  static const int lag = [] {
    const char *e = std::getenv("IBM_WF_LAG");
    const int v = e ? std::atoi(e) : WF_LAG_DEFAULT;
    return v == 2 ? 2 : 1;
  }();
  return lag;
}
static int wf_dlo(int m) { return 1 + wf_lag() * (2 * m - 1); }
static int wf_w(int m) { return (wf_dlo(m) + 3) & ~1; }
int wf_box_rows(int m) { return wf_w(m) / 2; }  // half a window
#ifdef WF_EXACT
bool wf_approx() { return false; }
#else
bool wf_approx() { return true; }
#endif
int wf_box_cols() { return SC; }

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
int sm_count_impl() {
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
int wf_items_target() { return 2 * 8 * sm_count_impl(); }
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

namespace {
int sm_count() { return sm_count_impl(); }
}  // namespace

std::vector<WfSeg> wf_seg_table(const WfArgs &a, int m, const double *cN, const double *cS) {
  const int W = wf_w(m), DLO = wf_dlo(m), NJ = a.g.NJ;
  std::vector<WfSeg> t(a.segs);
  for (int sy = 0; sy < a.segs; ++sy) {
    const int j0 = sy * a.L, j1 = std::min(j0 + a.L, a.g.nj), rs = j0 - 2 * m;
    const int nch = ((j1 - j0) + 2 * m + DLO + W - 1) / W;
    // the segment's reference row (as the kernel used to pick it)
    const int jr = std::min(std::max(a.g.gj0 + j0 + a.L / 2, 1), NJ - 2);
    WfSeg &e = t[sy];
    e.cN0 = cN[jr];
    e.cS0 = cS[jr];
    e.irr0 = INT_MAX;
    e.irr1 = INT_MIN;
    for (int r = rs - DLO; r <= rs + nch * W - 2; ++r) {  // the rows the item updates
      const int gj = a.g.gj0 + r, gjc = std::min(std::max(gj, 0), NJ - 1);
      const bool reg = gj >= a.uj0 && gj < a.uj1 && cN[gjc] == e.cN0 && cS[gjc] == e.cS0;
      if (!reg) {
        e.irr0 = std::min(e.irr0, r);
        e.irr1 = std::max(e.irr1, r);
      }
    }
  }
  return t;
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
