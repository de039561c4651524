// Dependent-chain latency of DFMA / DADD / DMUL / SHFL on this GPU (one warp).
#include <cstdio>
__global__ void k(double *o, long long *t, double a, double b) {
  double x = a + threadIdx.x;
  long long t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 256; ++i) {
#pragma unroll
    for (int j = 0; j < 16; ++j) x = __fma_rn(x, b, a);
  }
  long long t1 = clock64();
  double y = x;
#pragma unroll 1
  for (int i = 0; i < 256; ++i) {
#pragma unroll
    for (int j = 0; j < 16; ++j) y = __dadd_rn(y, b);
  }
  long long t2 = clock64();
  double z = y;
#pragma unroll 1
  for (int i = 0; i < 256; ++i) {
#pragma unroll
    for (int j = 0; j < 16; ++j) z = __shfl_sync(0xffffffffu, z, (threadIdx.x + 1) & 31);
  }
  long long t3 = clock64();
  o[threadIdx.x] = z;
  if (threadIdx.x == 0) { t[0] = t1 - t0; t[1] = t2 - t1; t[2] = t3 - t2; }
}
// throughput: many independent chains per warp, many warps
__global__ void thr(double *o, double a, double b, int iters) {
  double x0 = a + threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
  for (int i = 0; i < iters; ++i) {
    x0 = __fma_rn(x0, b, a); x1 = __fma_rn(x1, b, a); x2 = __fma_rn(x2, b, a); x3 = __fma_rn(x3, b, a);
    x4 = __fma_rn(x4, b, a); x5 = __fma_rn(x5, b, a); x6 = __fma_rn(x6, b, a); x7 = __fma_rn(x7, b, a);
  }
  o[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}
int main() {
  double *o; long long *t, h[3];
  cudaMalloc(&o, 1 << 26); cudaMalloc(&t, 64);
  k<<<1, 32>>>(o, t, 0.5, 0.999);
  cudaMemcpy(h, t, 24, cudaMemcpyDeviceToHost);
  printf("latency cycles: dfma %.2f dadd %.2f shfl(64-bit, 2 SHFL) %.2f\n", h[0] / 4096.0, h[1] / 4096.0, h[2] / 4096.0);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int iters = 4096;
  thr<<<sms * 8, 256>>>(o, 0.5, 0.999, iters);
  cudaEventRecord(e0);
  thr<<<sms * 8, 256>>>(o, 0.5, 0.999, iters);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double fmas = (double)sms * 8 * 256 * iters * 8;
  printf("DFMA throughput %.2f TFMA/s = %.1f TFLOP/s\n", fmas / ms / 1e9, 2 * fmas / ms / 1e9);
  return 0;
}
