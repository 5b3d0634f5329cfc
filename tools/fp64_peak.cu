// FP64 DFMA peak microbenchmark (B200 has no FP64 entry in MEASURED_PEAKS.json).
// Each thread runs 8 independent DFMA chains; FLOPs = 2 per DFMA.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void dfma_chain(double* out, int iters, double a, double b) {
  double x0 = threadIdx.x * 1e-3, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3;
  double x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
      x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
    }
  }
  double s = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
  if (s == 12345.678) out[0] = s;
}
int main() {
  int dev = 0; cudaDeviceProp p; cudaGetDeviceProperties(&p, dev);
  int l2 = 0; cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, dev);
  int clk = 0; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  printf("name=%s sms=%d l2_bytes=%d clock_khz=%d smem_optin=%zu regs_per_sm=%d\n", p.name,
         p.multiProcessorCount, l2, clk, p.sharedMemPerBlockOptin, p.regsPerMultiprocessor);
  double* d; cudaMalloc(&d, 8);
  int iters = 4096;
  for (int tpb : {128, 256, 512, 1024}) {
    for (int bps : {1, 2, 4, 8}) {
      int blocks = p.multiProcessorCount * bps;
      if (tpb * bps > 2048) continue;
      cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
      dfma_chain<<<blocks, tpb>>>(d, 16, 0.999999, 1e-7);
      cudaEventRecord(e0);
      for (int r = 0; r < 5; ++r) dfma_chain<<<blocks, tpb>>>(d, iters, 0.999999, 1e-7);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double flops = 5.0 * blocks * tpb * (double)iters * 16 * 8 * 2;
      printf("tpb=%d blocks=%d  %.3f ms  %.2f TFLOP/s\n", tpb, blocks, ms, flops / (ms * 1e-3) / 1e12);
    }
  }
  cudaError_t e = cudaGetLastError(); printf("err=%s\n", cudaGetErrorString(e));
  return 0;
}
