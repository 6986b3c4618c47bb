// Dev probe: do DMMA (mma.sync f64) and DFMA share the FP64 datapath on B200?
// mode 0: DMMA warps only, 1: DFMA warps only, 2: both kinds in one CTA.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}

__global__ void k(int mode, int iters, double* out) {
  const int warp = threadIdx.x >> 5;
  const bool mma_warp = (mode == 0) || (mode == 2 && warp < 4);
  const bool fma_warp = (mode == 1) || (mode == 2 && warp >= 4);
  double s = 0;
  if (mma_warp) {
    double acc[4][2] = {};
    const double a = 1.0 + threadIdx.x * 1e-9, b = 0.5;
    for (int it = 0; it < iters; ++it)
#pragma unroll
      for (int q = 0; q < 4; ++q) dmma(acc[q][0], acc[q][1], a, b);
    for (int q = 0; q < 4; ++q) s += acc[q][0] + acc[q][1];
  }
  if (fma_warp) {
    double x[8];
    for (int q = 0; q < 8; ++q) x[q] = threadIdx.x * 1e-9 + q;
    for (int it = 0; it < iters; ++it)
#pragma unroll
      for (int q = 0; q < 8; ++q) x[q] = fma(x[q], 0.999999, 1e-7);
    for (int q = 0; q < 8; ++q) s += x[q];
  }
  if (s == 12345.678) out[0] = s;
}

int main() {
  double* out;
  cudaMalloc(&out, 8);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int blocks = 148 * 4;
  struct { int mode, threads, iters; const char* name; } cfg[] = {
      {0, 128, 20000, "DMMA 4 warps/CTA"}, {1, 128, 40000, "DFMA 4 warps/CTA"},
      {2, 256, 20000, "DMMA 4 + DFMA 4 warps/CTA (DFMA iters = DMMA iters)"},
      {0, 256, 20000, "DMMA 8 warps/CTA"}};
  for (auto& c : cfg) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(a);
      k<<<blocks, c.threads>>>(c.mode, c.iters, out);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
    }
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    const double mma_warps = (c.mode == 0 ? c.threads / 32 : c.mode == 2 ? 4 : 0) * (double)blocks;
    const double fma_warps = (c.mode == 1 ? c.threads / 32 : c.mode == 2 ? 4 : 0) * (double)blocks;
    const double mma_tf = mma_warps * c.iters * 4 * 512 / (ms * 1e-3) / 1e12;
    const double fma_tf = fma_warps * 32 * c.iters * 8 * 2 / (ms * 1e-3) / 1e12;
    printf("%-55s %8.3f ms  DMMA %6.2f TF  DFMA %6.2f TF  sum %6.2f\n", c.name, ms, mma_tf, fma_tf, mma_tf + fma_tf);
  }
  return 0;
}
