// K4a — offline POD by the method of snapshots (BASELINE config 4).
//
// Replaces pod_impl / mgs_pass / pod_diag (/root/reference/proj/src/
// podkit.cpp:43-86, 117-127):
//   1. corr = S^T diag(g) S — symmetric DMMA GEMM (only the upper tile
//      triangle is computed and mirrored; exactly symmetric, so the
//      reference's 0.5 (corr + corr^T) is the identity on it);
//   2. the dense symmetric eigendecomposition — cuSOLVER syevd (library
//      call), eigenvalues reordered descending;
//   3. keep while lambda > tol^2 lambda_0 and lambda > 0, <= max_modes;
//      mode_i = S v_i / sqrt(lambda_i) — DMMA GEMM + column division;
//   4. one modified Gram-Schmidt pass in the diag(g) metric, one CTA with
//      fixed-tree block reductions (deterministic).
#include <cusolverDn.h>

#include <algorithm>
#include <cmath>
#include <vector>

#include "common.cuh"
#include "dmma_gemm.cuh"

using namespace podecm_dev;
using namespace podecm_impl;

namespace {

__device__ double block_sum(double v, double* red) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  __syncthreads();
  if (lane == 0) red[w] = v;
  __syncthreads();
  double s = 0.0;
  for (int k = 0; k < nw; ++k) s += red[k];  // same order in every thread
  return s;
}

// mode_i = (S v_i) / sqrt(lambda_i): column scaling after the GEMM
__global__ void k_scale_cols(double* M, int64_t rows, int cols, const double* lam) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= rows * cols) return;
  const int c = (int)(t / rows);
  M[t] = M[t] / sqrt(lam[c]);
}

// mgs_pass (podkit.cpp:75-86) with gram images gm = diag(g) m (g == null: identity).
__global__ void __launch_bounds__(1024) k_mgs(double* m, double* gm, int64_t rows, int cols,
                                              const double* g) {
  __shared__ double red[32];
  if (g)
    for (int c = 0; c < cols; ++c)
      for (int64_t r = threadIdx.x; r < rows; r += blockDim.x) gm[c * rows + r] = g[r] * m[c * rows + r];
  __syncthreads();
  const double* G = g ? gm : m;
  for (int i = 0; i < cols; ++i) {
    double* mi = m + (int64_t)i * rows;
    double* gi = g ? gm + (int64_t)i * rows : mi;
    for (int j = 0; j < i; ++j) {
      const double* mj = m + (int64_t)j * rows;
      const double* gj = G + (int64_t)j * rows;
      double p = 0.0;
      for (int64_t r = threadIdx.x; r < rows; r += blockDim.x) p = fma(gj[r], mi[r], p);
      const double c = block_sum(p, red);
      for (int64_t r = threadIdx.x; r < rows; r += blockDim.x) {
        mi[r] -= c * mj[r];
        if (g) gi[r] -= c * gj[r];
      }
      __syncthreads();
    }
    double p = 0.0;
    for (int64_t r = threadIdx.x; r < rows; r += blockDim.x) p = fma(gi[r], mi[r], p);
    const double nrm = sqrt(block_sum(p, red));
    for (int64_t r = threadIdx.x; r < rows; r += blockDim.x) {
      mi[r] /= nrm;
      if (g) gi[r] /= nrm;
    }
    __syncthreads();
  }
}

int gemm(podecm_ctx* ctx, cudaStream_t s, const GemmArgs& a) {
  dim3 grid((unsigned)((a.N + kGBN - 1) / kGBN), (unsigned)((a.M + kGBM - 1) / kGBM));
  {
    KTimer kt(ctx, s, "k_gemm_dmma");
    k_gemm_dmma<<<grid, 128, 0, s>>>(a);
  }
  PODECM_LAUNCHED(ctx, 1);
  return PODECM_OK;
}

}  // namespace

extern "C" {

int podecm_pod_gram(podecm_ctx* ctx, void* stream, const double* S, int64_t n_dof, int n_snap,
                    const double* gram_diag, double* C) {
  if (!ctx || !S || !C) return PODECM_ECONFIG;
  if (n_dof <= 0 || n_snap <= 0) return set_err(ctx, PODECM_ECONFIG, "pod_gram: empty snapshot matrix");
  GemmArgs a{};
  a.M = n_snap;
  a.N = n_snap;
  a.K = n_dof;
  a.A = S;  // A(i,k) = S(k,i): column i of the column-major S
  a.a_rs = n_dof;
  a.a_cs = 1;
  a.B = S;  // B(k,j) = S(k,j)
  a.b_rs = 1;
  a.b_cs = n_dof;
  a.C = C;
  a.c_rs = n_snap;  // symmetric: row/column-major identical
  a.c_cs = 1;
  a.diag = gram_diag;
  a.sym = 1;
  return gemm(ctx, static_cast<cudaStream_t>(stream), a);
}

// C (n_snap x n_snap, overwritten by eigenvectors).  Outputs modes
// [max_modes][n_dof] (column-major n_dof x keep), evals [n_snap]
// descending (device), *n_kept (host).  Synchronises the stream.
int podecm_pod_modes(podecm_ctx* ctx, void* stream, const double* S, int64_t n_dof, int n_snap,
                     double* C, const double* gram_diag, int max_modes, double tol_rel,
                     double* modes, double* evals, int* n_kept) {
  return podecm_pod_modes_ex(ctx, stream, S, n_dof, n_snap, C, gram_diag, max_modes, tol_rel, modes, evals,
                             n_kept, 1);
}

int podecm_pod_mgs(podecm_ctx* ctx, void* stream, double* modes, int64_t n_dof, int k, const double* gram_diag) {
  if (!ctx || !modes || k < 0 || n_dof <= 0) return PODECM_ECONFIG;
  if (k == 0) return PODECM_OK;
  auto s = static_cast<cudaStream_t>(stream);
  double* gm = nullptr;
  if (gram_diag) PODECM_CUDA_TRY(ctx, cudaMalloc(&gm, sizeof(double) * n_dof * k));
  {
    KTimer kt(ctx, s, "k_mgs");
    k_mgs<<<1, 1024, 0, s>>>(modes, gm, n_dof, k, gram_diag);
  }
  PODECM_LAUNCHED(ctx, 1);
  cudaStreamSynchronize(s);
  cudaFree(gm);
  return PODECM_OK;
}

int podecm_pod_modes_ex(podecm_ctx* ctx, void* stream, const double* S, int64_t n_dof, int n_snap,
                        double* C, const double* gram_diag, int max_modes, double tol_rel,
                        double* modes, double* evals, int* n_kept, int mgs) {
  if (!ctx || !S || !C || !modes || !evals || !n_kept) return PODECM_ECONFIG;
  auto s = static_cast<cudaStream_t>(stream);
  cusolverDnHandle_t h = nullptr;
  if (cusolverDnCreate(&h) != CUSOLVER_STATUS_SUCCESS)
    return set_err(ctx, PODECM_ECUDA, "cusolverDnCreate failed");
  cusolverDnSetStream(h, s);
  double* w = nullptr;
  int* info = nullptr;
  double* work = nullptr;
  int lwork = 0;
  int rc = PODECM_OK;
  PODECM_CUDA_TRY(ctx, cudaMalloc(&w, sizeof(double) * n_snap));
  PODECM_CUDA_TRY(ctx, cudaMalloc(&info, sizeof(int)));
  if (cusolverDnDsyevd_bufferSize(h, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_UPPER, n_snap, C,
                                  n_snap, w, &lwork) != CUSOLVER_STATUS_SUCCESS)
    rc = set_err(ctx, PODECM_ECUDA, "syevd buffer query failed");
  if (!rc && cudaMalloc(&work, sizeof(double) * std::max(lwork, 1)) != cudaSuccess)
    rc = set_err(ctx, PODECM_ECUDA, "syevd workspace");
  if (!rc) {
    KTimer kt(ctx, s, "cusolver_syevd");
    if (cusolverDnDsyevd(h, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_UPPER, n_snap, C, n_snap, w,
                         work, lwork, info) != CUSOLVER_STATUS_SUCCESS)
      rc = set_err(ctx, PODECM_ECUDA, "syevd failed");
  }
  int hinfo = 0;
  std::vector<double> lam(n_snap);
  if (!rc) {
    cudaMemcpyAsync(&hinfo, info, sizeof(int), cudaMemcpyDeviceToHost, s);
    cudaMemcpyAsync(lam.data(), w, sizeof(double) * n_snap, cudaMemcpyDeviceToHost, s);
    cudaStreamSynchronize(s);
    if (hinfo != 0) rc = set_err(ctx, PODECM_ESOLVE, "snapshot eigenproblem failed to converge");
  }
  int keep = 0;
  if (!rc) {
    std::vector<double> desc(n_snap);
    for (int i = 0; i < n_snap; ++i) desc[i] = lam[n_snap - 1 - i];
    const double lead = std::max(desc[0], 0.0);
    const double cut = tol_rel * tol_rel * lead;
    while (keep < n_snap && keep < max_modes && desc[keep] > cut && desc[keep] > 0.0) ++keep;
    cudaMemcpyAsync(evals, desc.data(), sizeof(double) * n_snap, cudaMemcpyHostToDevice, s);
    if (keep > 0) {
      // modes = S * V_desc, V_desc(:, i) = C(:, n_snap-1-i)
      GemmArgs a{};
      a.M = n_dof;
      a.N = keep;
      a.K = n_snap;
      a.A = S;
      a.a_rs = 1;
      a.a_cs = n_dof;
      a.B = C + (int64_t)(n_snap - 1) * n_snap;
      a.b_rs = 1;
      a.b_cs = -(int64_t)n_snap;
      a.C = modes;
      a.c_rs = 1;
      a.c_cs = n_dof;
      rc = gemm(ctx, s, a);
      if (!rc) {
        k_scale_cols<<<grid_for(n_dof * keep, 256), 256, 0, s>>>(modes, n_dof, keep, evals);
        PODECM_LAUNCHED(ctx, 1);
        if (mgs) rc = podecm_pod_mgs(ctx, s, modes, n_dof, keep, gram_diag);
        cudaStreamSynchronize(s);
      }
    }
  }
  *n_kept = keep;
  cudaFree(w);
  cudaFree(info);
  cudaFree(work);
  cusolverDnDestroy(h);
  return rc;
}

}  // extern "C"
