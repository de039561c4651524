// Device helpers shared by the SOR kernels (sor.cu, sor_wf.cu): mbarrier / TMA
// wrappers, the exact residual max on uint64 bit patterns, element access of a
// column pair.
#pragma once
#include <cstdint>

#include "ibm_internal.h"

namespace ibm {

__device__ __forceinline__ unsigned long long umax64(unsigned long long a, unsigned long long b) {
  return a > b ? a : b;
}
// |d| as its IEEE bit pattern (order-preserving for |d| >= 0; NaN sorts above
// every number).  The sign bit is cleared with an integer AND on the high word:
// written as a plain 64-bit AND, ptxas turns it into DADD |d| on the fp64 pipe.
__device__ __forceinline__ unsigned long long abs_bits(double d) {
  unsigned lo, hi;
  asm("mov.b64 {%0, %1}, %2;" : "=r"(lo), "=r"(hi) : "d"(d));
  asm("and.b32 %0, %0, 0x7fffffff;" : "+r"(hi));
  return ((unsigned long long)hi << 32) | lo;
}
// abs_bits(d) & (m:m): the whole pattern is zeroed where the mask m is 0 (a term
// that is not counted), folded into the sign-clearing AND
__device__ __forceinline__ unsigned long long abs_bits_masked(double d, unsigned m) {
  unsigned lo, hi;
  asm("mov.b64 {%0, %1}, %2;" : "=r"(lo), "=r"(hi) : "d"(d));
  asm("and.b32 %0, %0, 0x7fffffff;" : "+r"(hi));
  hi &= m;
  lo &= m;
  return ((unsigned long long)hi << 32) | lo;
}
__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(unsigned long long *bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long *bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned long long *bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long *bar, uint32_t phase) {
  uint32_t done = 0;
  do {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(phase)
        : "memory");
  } while (!done);
}
// warp-wide wait: the vote keeps the loop exit warp-uniform, so the compiler
// knows the warp is converged afterwards (no divergence checks before shuffles)
__device__ __forceinline__ void mbar_wait_warp(unsigned long long *bar, uint32_t phase) {
  for (;;) {
    uint32_t done;
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(phase)
        : "memory");
    if (__all_sync(0xffffffffu, done)) break;
  }
}
// the same with a watchdog: traps (the launch fails) instead of spinning forever
// when the phase never completes -- for the experimental producer / consumer rings
__device__ __forceinline__ void mbar_wait_warp_bounded(unsigned long long *bar, uint32_t phase) {
  for (unsigned n = 0;; ++n) {
    uint32_t done;
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(phase)
        : "memory");
    if (__all_sync(0xffffffffu, done)) break;
    if (n > (1u << 24)) __trap();
  }
}
__device__ __forceinline__ void tma_load_2d(void *dst, const CUtensorMap *map, int c0, int c1,
                                            unsigned long long *bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}

// One elected lane of the (converged) warp arms bar for `bytes` and issues the two
// 2-D box loads (x and b of the same rows) -- no divergent branch around the
// issue, so the surrounding code stays one basic block; with warp-uniform
// operands ptxas emits plain UTMALDGs (an `if (lane == 0)` region made it wrap
// them in ELECT / BRA.U.ANY loops and split the hot loop at BSSY / BSYNC).
__device__ __forceinline__ void tma_load_pair_elect(unsigned long long *bar, uint32_t bytes, void *dx,
                                                    const CUtensorMap *mx, void *db, const CUtensorMap *mb, int c0,
                                                    int c1) {
  asm volatile(
      "{\n .reg .pred p;\n elect.sync _|p, 0xffffffff;\n"
      "@p mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n"
      "@p cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%2], [%3, {%6, %7}], [%0];\n"
      "@p cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%4], [%5, {%6, %7}], [%0];\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(bytes), "r"(smem_u32(dx)), "l"(reinterpret_cast<uint64_t>(mx)), "r"(smem_u32(db)),
      "l"(reinterpret_cast<uint64_t>(mb)), "r"(c0), "r"(c1)
      : "memory");
}

// Same, issued only if `go` (warp-uniform): the predicate is folded into the
// elected lane's, so there is no branch either.
__device__ __forceinline__ void tma_load_pair_elect_if(bool go, unsigned long long *bar, uint32_t bytes, void *dx,
                                                       const CUtensorMap *mx, void *db, const CUtensorMap *mb, int c0,
                                                       int c1) {
  asm volatile(
      "{\n .reg .pred p, q;\n elect.sync _|p, 0xffffffff;\n setp.ne.b32 q, %8, 0;\n and.pred p, p, q;\n"
      "@p mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n"
      "@p cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%2], [%3, {%6, %7}], [%0];\n"
      "@p cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%4], [%5, {%6, %7}], [%0];\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(bytes), "r"(smem_u32(dx)), "l"(reinterpret_cast<uint64_t>(mx)), "r"(smem_u32(db)),
      "l"(reinterpret_cast<uint64_t>(mb)), "r"(c0), "r"(c1), "r"((int)go)
      : "memory");
}

__device__ __forceinline__ void tma_load_1d(void *dst, const CUtensorMap *map, int c0, unsigned long long *bar) {
  tma_load_2d(dst, map, c0, 0, bar);  // one-row 2-D map
}

__device__ __forceinline__ double rd(const double2 &v, int e) { return e ? v.y : v.x; }
__device__ __forceinline__ void wr(double2 &v, int e, double x) {
  if (e)
    v.y = x;
  else
    v.x = x;
}

}  // namespace ibm
