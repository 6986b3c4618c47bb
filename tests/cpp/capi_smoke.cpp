// C++ consumer of the C-ABI exactly as the reference would bind it
// (INTEGRATION.md): no Python, no torch.  Checks the equal-biaxial closed
// form of test_material.cpp:151-163 through podecm_material_batch and one
// assembly of a 16x16 cell through podecm_assemble_batch.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <vector>

#include "../../include/podecm_cuda.h"

#define CHECK(x)                                                   \
  do {                                                             \
    int rc_ = (x);                                                 \
    if (rc_) {                                                     \
      std::printf("FAIL %s -> %d (%s)\n", #x, rc_, podecm_last_error(ctx)); \
      return 1;                                                    \
    }                                                              \
  } while (0)

int main(int argc, char** argv) {
  podecm_ctx* ctx = nullptr;
  if (podecm_ctx_create(0, &ctx)) {
    std::printf("FAIL ctx\n");
    return 1;
  }
  // --- material: equal biaxial stretch, elastic (sigma_y0 = 1e12) ---------
  const podecm_params p{10.0, 0.3, 1e12, 5.0};
  const double c = 1.05;
  std::vector<double> hF = {c, 0, 0, c}, hS = {1, 0, 0, 1, 1, 0};  // n = 1: planes of length 1
  double *dF, *dS, *dP, *dA, *dS1;
  cudaMalloc(&dF, 32);
  cudaMalloc(&dS, 48);
  cudaMalloc(&dP, 32);
  cudaMalloc(&dA, 128);
  cudaMalloc(&dS1, 48);
  cudaMemcpy(dF, hF.data(), 32, cudaMemcpyHostToDevice);
  cudaMemcpy(dS, hS.data(), 48, cudaMemcpyHostToDevice);
  CHECK(podecm_material_batch(ctx, nullptr, 1, &p, 1, nullptr, dF, dS, dP, dA, dS1, nullptr, 1e-7));
  CHECK(podecm_check(ctx, nullptr));
  double hP[4];
  cudaMemcpy(hP, dP, 32, cudaMemcpyDeviceToHost);
  const double la = p.E * p.nu / ((1 + p.nu) * (1 - 2 * p.nu)), mu = p.E / (2 * (1 + p.nu));
  const double sig = la * 2 * std::log(c) + 2 * mu * std::log(c);
  const bool ok1 = std::fabs(hP[0] - sig / c) <= 1e-12 && std::fabs(hP[3] - sig / c) <= 1e-12 &&
                   std::fabs(hP[1]) <= 1e-13 && std::fabs(hP[2]) <= 1e-13;
  std::printf("material closed form: P00 = %.17g (expect %.17g) %s\n", hP[0], sig / c, ok1 ? "ok" : "FAIL");

  // --- assembly: 16x16 cell, one instance, zero fluctuation, virgin history
  const podecm_params mats[2] = {{1.0, 0.3, 0.01, 0.1}, {10.0, 0.3, 1e300, 0.0}};
  podecm_rve* rve = nullptr;
  CHECK(podecm_rve_create_q4(ctx, 16, 0.25, mats, 2, &rve));
  int64_t info[6];
  podecm_rve_info(rve, info);
  const int64_t nq = info[2], nr = info[3], nnz = info[4];
  std::vector<double> geom = {0.3, 0.2}, fbar = {1.02, 0.01, 0.0, 0.99};
  std::vector<double> st0(6 * nq);
  for (int64_t q = 0; q < nq; ++q) {
    st0[q] = 1.0;
    st0[3 * nq + q] = 1.0;
    st0[4 * nq + q] = 1.0;
  }
  double *dg, *dfb, *dw, *dst0, *df, *dK;
  cudaMalloc(&dg, 16);
  cudaMalloc(&dfb, 32);
  cudaMalloc(&dw, nr * 8);
  cudaMalloc(&dst0, 6 * nq * 8);
  cudaMalloc(&df, nr * 8);
  cudaMalloc(&dK, nnz * 8);
  cudaMemcpy(dg, geom.data(), 16, cudaMemcpyHostToDevice);
  cudaMemcpy(dfb, fbar.data(), 32, cudaMemcpyHostToDevice);
  cudaMemset(dw, 0, nr * 8);
  cudaMemcpy(dst0, st0.data(), 6 * nq * 8, cudaMemcpyHostToDevice);
  CHECK(podecm_assemble_batch(ctx, nullptr, rve, 1, dg, nullptr, dfb, dw, dst0, nullptr, df, dK, nullptr,
                              nullptr));
  CHECK(podecm_check(ctx, nullptr));
  std::vector<double> hf(nr), hK(nnz);
  cudaMemcpy(hf.data(), df, nr * 8, cudaMemcpyDeviceToHost);
  cudaMemcpy(hK.data(), dK, nnz * 8, cudaMemcpyDeviceToHost);
  double fn = 0, kn = 0;
  bool finite = true;
  for (double v : hf) fn += v * v, finite &= std::isfinite(v);
  for (double v : hK) kn += v * v, finite &= std::isfinite(v);
  const bool ok2 = finite && kn > 0 && fn > 0;  // heterogeneous cell: nonzero residual
  std::printf("assembly: n_red %lld nnz %lld |f| %.6e |K| %.6e %s\n", (long long)nr, (long long)nnz,
              std::sqrt(fn), std::sqrt(kn), ok2 ? "ok" : "FAIL");
  if (argc > 1) {  // the caller (tests/test_gpu_capi_cpp.py) checks f and K against the oracle
    if (FILE* fo = std::fopen(argv[1], "wb")) {
      const int64_t hdr[2] = {nr, nnz};
      std::fwrite(hdr, sizeof(int64_t), 2, fo);
      std::fwrite(hf.data(), sizeof(double), hf.size(), fo);
      std::fwrite(hK.data(), sizeof(double), hK.size(), fo);
      std::fclose(fo);
    }
  }
  std::printf("launches: %lld\n", (long long)podecm_launch_count(ctx));
  podecm_rve_destroy(rve);
  podecm_ctx_destroy(ctx);
  return ok1 && ok2 ? 0 : 1;
}
