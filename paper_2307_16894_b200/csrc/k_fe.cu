// §8(f) item 3 — full-order Newton on the GPU: solve_rve with
// solve_step_adaptive (/root/reference/proj/src/microfem.cpp:142-238) for a
// batch of independent RVE instances around the K2 assembly.
//
// One "global iteration" assembles every instance (K2: residual, CSR
// tangent, trial history, stress field), takes the residual norms to the host
// where each instance runs the reference's Newton / bisection logic, then
// solves K dw = -f for the whole batch with one batched sparse LU
// refactorisation.  All instances share the CSR pattern, so the symbolic
// work (symmetric AMD ordering, L/U pattern, level schedule) is done once on
// the host (cuSOLVER csrlu*Host) and every later factorisation is a device
// refactorisation of new values (cuSOLVER Rf, batched) — the GPU analogue of
// Eigen::SparseLU's analyzePattern-once / factorize-per-iteration use in
// solve_step (microfem.cpp:179-183).  The refactorisation keeps the first
// factorisation's (diagonal) pivot sequence; a zero pivot fails that
// instance's attempt like the reference's "cell tangent factorization failed"
// (microfem.cpp:182).
#include <cusolverRf.h>
#include <cusolverSp.h>
#include <cusolverSp_LOWLEVEL_PREVIEW.h>
#include <cusparse.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "rve.cuh"

using namespace podecm_impl;

namespace {

constexpr int kFeMaxStack = 8;

bool fe_debug() {
  static const bool v = [] {
    const char* e = getenv("PODECM_FE_DEBUG");
    return e && atoi(e) != 0;
  }();
  return v;
}
#define FE_DBG(...)                   \
  do {                                \
    if (fe_debug()) {                 \
      fprintf(stderr, "[fe] " __VA_ARGS__); \
      fflush(stderr);                 \
    }                                 \
  } while (0)

// per-instance residual norm (one CTA per instance, fixed-order tree)
__global__ void __launch_bounds__(256) k_fe_norm(int n_red, const double* f, double* norm) {
  __shared__ double red[256];
  const double* fs = f + (size_t)blockIdx.x * n_red;
  double s = 0.0;
  for (int i = threadIdx.x; i < n_red; i += blockDim.x) s = fma(fs[i], fs[i], s);
  red[threadIdx.x] = s;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) norm[blockIdx.x] = sqrt(red[0]);
}

// effective_stress (microfem.cpp:132-140): pbar = sum_q w_q det_q P_q / vol
__global__ void __launch_bounds__(256) k_fe_pbar(int nq, const double* w, const double* det, const double* pf,
                                                 double* pbar) {
  __shared__ double red[4][256];
  const int s = blockIdx.x;
  double acc[4] = {0.0, 0.0, 0.0, 0.0};
  for (int q = threadIdx.x; q < nq; q += blockDim.x) {
    const double wq = w[q] * det[(size_t)s * nq + q];
    for (int k = 0; k < 4; ++k) acc[k] = fma(wq, pf[((size_t)s * 4 + k) * nq + q], acc[k]);
  }
  for (int k = 0; k < 4; ++k) red[k][threadIdx.x] = acc[k];
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if (threadIdx.x < o)
      for (int k = 0; k < 4; ++k) red[k][threadIdx.x] += red[k][threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x < 4) pbar[4 * s + threadIdx.x] = red[threadIdx.x][0] / 1.0;  // cell_volume
}

// masked per-instance copies: dst[s] = src[s] for mask[s] (len doubles each)
__global__ void k_fe_copy(int64_t n, int64_t len, const int32_t* mask, const double* src, double* dst) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n * len) return;
  if (mask[t / len]) dst[t] = src[t];
}

// x = -f (all instances), the right-hand sides of the batched solve
__global__ void k_fe_negate(int64_t m, const double* f, double* x) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t < m) x[t] = -f[t];
}

// w += dw for mask[s]
__global__ void k_fe_update(int64_t n, int n_red, const int32_t* mask, const double* dw, double* w) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n * n_red) return;
  if (mask[t / n_red]) w[t] += dw[t];
}

__global__ void k_fe_addfail(unsigned int* fail, unsigned int n) { atomicAdd(fail, n); }

__global__ void k_fe_virgin(int64_t n, int nq, double* S) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n * nq) return;
  const int64_t s = t / nq;
  const int q = (int)(t - s * nq);
  const double v[6] = {1.0, 0.0, 0.0, 1.0, 1.0, 0.0};
  for (int k = 0; k < 6; ++k) S[(s * 6 + k) * nq + q] = v[k];
}


// effective_stiffness (microfem.cpp:283-308): for each unit perturbation
// E_kl (column c = k + 2l) with fluctuation response x_c,
//   Abar(:, c) = sum_q wq A_q (grad(x_c) Fmu^-1 + E_kl)
// one CTA per instance, fixed-order block tree over the qps.
__global__ void __launch_bounds__(256) k_fe_abar(int nq, int n_red, int64_t n, const int32_t* elems,
                                                 const int32_t* node_dof, const double* grad, const double* w,
                                                 const double* fmi, const double* det, const double* af,
                                                 const double* x, double* abar) {
  __shared__ double red[16][256];
  const int64_t s = blockIdx.x;
  double acc[16];
#pragma unroll
  for (int t = 0; t < 16; ++t) acc[t] = 0.0;
  for (int q = threadIdx.x; q < nq; q += blockDim.x) {
    const int e = q >> 2;
    double g[8], m[4], A[16];
#pragma unroll
    for (int t = 0; t < 8; ++t) g[t] = grad[(size_t)q * 8 + t];
#pragma unroll
    for (int t = 0; t < 4; ++t) m[t] = fmi[((size_t)s * 4 + t) * nq + q];
#pragma unroll
    for (int t = 0; t < 16; ++t) A[t] = af[((size_t)s * 16 + t) * nq + q];
    const double wq = w[q] * det[(size_t)s * nq + q];
    int dof[4];
#pragma unroll
    for (int a = 0; a < 4; ++a) dof[a] = node_dof[elems[4 * e + a]];
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const double* xs = x + ((size_t)c * n + s) * n_red;
      double gq[4];  // (i + 2j)
#pragma unroll
      for (int j = 0; j < 2; ++j)
#pragma unroll
        for (int i = 0; i < 2; ++i) {
          double v = 0.0;
#pragma unroll
          for (int a = 0; a < 4; ++a) v = v + (dof[a] >= 0 ? xs[dof[a] + i] : 0.0) * g[2 * a + j];
          gq[i + 2 * j] = v;
        }
      double df[4];
#pragma unroll
      for (int j = 0; j < 2; ++j)
#pragma unroll
        for (int i = 0; i < 2; ++i) df[i + 2 * j] = gq[i] * m[2 * j] + gq[i + 2] * m[1 + 2 * j];
      df[c] = df[c] + 1.0;  // E_kl, k + 2l = c
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        double cr = 0.0;
#pragma unroll
        for (int t = 0; t < 4; ++t) cr = cr + A[r + 4 * t] * df[t];
        acc[r + 4 * c] = acc[r + 4 * c] + wq * cr;
      }
    }
  }
#pragma unroll
  for (int t = 0; t < 16; ++t) red[t][threadIdx.x] = acc[t];
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if (threadIdx.x < o)
#pragma unroll
      for (int t = 0; t < 16; ++t) red[t][threadIdx.x] += red[t][threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x < 16) abar[s * 16 + threadIdx.x] = red[threadIdx.x][0] / 1.0;  // cell_volume
}


// weighted_stress_field (ecm.cpp:10-18): W_q = P_q Fmu_q^-T det_q, [n][nq][4]
__global__ void k_fe_wstress(int64_t n, int nq, const double* fmi, const double* det, const double* pf,
                             double* W) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n * nq) return;
  const int64_t s = t / nq;
  const int q = (int)(t - s * nq);
  double P[4], m[4];
  for (int k = 0; k < 4; ++k) {
    P[k] = pf[(s * 4 + k) * nq + q];
    m[k] = fmi[(s * 4 + k) * nq + q];
  }
  const double d = det[s * nq + q];
  for (int j = 0; j < 2; ++j)
    for (int i = 0; i < 2; ++i)  // (P Fmi^T)(i,j) = P(i,0) Fmi(j,0) + P(i,1) Fmi(j,1)
      W[(s * nq + q) * 4 + i + 2 * j] = (P[i] * m[j] + P[i + 2] * m[j + 2]) * d;
}

struct Frame {
  double fp[4], ft[4];
  int depth;
};

struct Inst {
  std::vector<Frame> stack;
  int k = 0, it = 0, iters_acc = 0;
  double tol = 0, r0 = 0;
  bool active = true;
  int status = 0;
};

}  // namespace

struct podecm_fe {
  podecm_ctx* ctx = nullptr;
  podecm_rve* rve = nullptr;
  int64_t cap = 0;  // instances the buffers (and the Rf batch) hold
  // one Rf handle per instance (the batched Rf entry points crash in
  // cusolverRfBatchAnalyze on this stack; tools/dev/rf_probe.cu reproduces it)
  std::vector<cusolverRfHandle_t> rf;
  int *d_row = nullptr, *d_col = nullptr, *d_P = nullptr, *d_Q = nullptr;
  double *d_w = nullptr, *d_w0 = nullptr, *d_Sc = nullptr, *d_St = nullptr, *d_f = nullptr, *d_K = nullptr,
         *d_pf = nullptr, *d_fb = nullptr, *d_fmi = nullptr, *d_det = nullptr, *d_x = nullptr, *d_tmp = nullptr,
         *d_norm = nullptr, *d_pb = nullptr;
  int32_t *d_astat = nullptr, *d_mask = nullptr, *d_mstat = nullptr;
  double* h_pin = nullptr;  // pinned: norms, pbar, fbar, masks
  int64_t global_iters = 0;
  double *d_af = nullptr, *d_rhs = nullptr;  // effective stiffness: tangent field, 4 right-hand sides
  int64_t af_cap = 0;
};

namespace {

void fe_free(podecm_fe* e) {
  for (double* p : {e->d_w, e->d_w0, e->d_Sc, e->d_St, e->d_f, e->d_K, e->d_pf, e->d_fb, e->d_fmi, e->d_det,
                    e->d_x, e->d_tmp, e->d_norm, e->d_pb})
    cudaFree(p);
  for (int32_t* p : {e->d_astat, e->d_mask, e->d_mstat}) cudaFree(p);
  if (e->h_pin) cudaFreeHost(e->h_pin);
  e->d_w = e->d_w0 = e->d_Sc = e->d_St = e->d_f = e->d_K = e->d_pf = e->d_fb = e->d_fmi = e->d_det = e->d_x =
      e->d_tmp = e->d_norm = e->d_pb = nullptr;
  e->d_astat = e->d_mask = e->d_mstat = nullptr;
  e->h_pin = nullptr;
  e->cap = 0;
}

int fe_alloc(podecm_fe* e, int64_t n) {
  if (e->cap >= n) return PODECM_OK;
  fe_free(e);
  podecm_rve* r = e->rve;
  const size_t nr = r->n_red, nq = r->n_qp, nnz = r->nnz;
  auto A = [&](double** p, size_t cnt) { return cudaMalloc(p, std::max<size_t>(cnt, 1) * sizeof(double)); };
  auto Ai = [&](int32_t** p, size_t cnt) { return cudaMalloc(p, std::max<size_t>(cnt, 1) * sizeof(int32_t)); };
  cudaError_t c = cudaSuccess;
  if (!c) c = A(&e->d_w, n * nr);
  if (!c) c = A(&e->d_w0, n * nr);
  if (!c) c = A(&e->d_Sc, n * 6 * nq);
  if (!c) c = A(&e->d_St, n * 6 * nq);
  if (!c) c = A(&e->d_f, n * nr);
  if (!c) c = A(&e->d_K, n * nnz);
  if (!c) c = A(&e->d_pf, n * 4 * nq);
  if (!c) c = A(&e->d_fb, n * 4);
  if (!c) c = A(&e->d_fmi, n * 4 * nq);
  if (!c) c = A(&e->d_det, n * nq);
  if (!c) c = A(&e->d_x, n * nr);
  if (!c) c = A(&e->d_tmp, 2 * n * nr);
  if (!c) c = A(&e->d_norm, n);
  if (!c) c = A(&e->d_pb, n * 4);
  if (!c) c = Ai(&e->d_astat, n);
  if (!c) c = Ai(&e->d_mask, n);
  if (!c) c = Ai(&e->d_mstat, n);
  if (!c) c = cudaMallocHost(&e->h_pin, sizeof(double) * (size_t)n * 12);
  if (c) {
    fe_free(e);
    return cuda_err(e->ctx, c, "fe: allocation");
  }
  e->cap = n;
  return PODECM_OK;
}

#define FE_SP(call, what)                                                          \
  do {                                                                             \
    const int st_ = (int)(call);                                                   \
    if (st_ != (int)CUSOLVER_STATUS_SUCCESS) {                                     \
      ok = false;                                                                  \
      msg = std::string(what) + " (cusolver status " + std::to_string(st_) + ")";  \
    }                                                                              \
  } while (0)

// Symbolic + first numeric LU on the host (symmetric AMD ordering, diagonal
// pivots), then the batched Rf handle for `batch` matrices of this pattern.
int rf_setup(podecm_fe* e, cudaStream_t s, int64_t batch) {
  podecm_rve* r = e->rve;
  const int n = r->n_red, nnz = (int)r->nnz;
  if ((int64_t)e->rf.size() >= batch) return PODECM_OK;
  std::vector<double> val(nnz);
  PODECM_CUDA_TRY(e->ctx, cudaMemcpyAsync(val.data(), e->d_K, sizeof(double) * nnz, cudaMemcpyDeviceToHost, s));
  PODECM_CUDA_TRY(e->ctx, cudaStreamSynchronize(s));
  bool ok = true;
  std::string msg;
  cusolverSpHandle_t sp = nullptr;
  cusparseMatDescr_t dA = nullptr;
  csrluInfoHost_t info = nullptr;
  FE_SP(cusolverSpCreate(&sp), "cusolverSpCreate");
  if (ok && cusparseCreateMatDescr(&dA) != CUSPARSE_STATUS_SUCCESS) ok = false, msg = "cusparseCreateMatDescr";
  if (ok) {
    cusparseSetMatType(dA, CUSPARSE_MATRIX_TYPE_GENERAL);
    cusparseSetMatIndexBase(dA, CUSPARSE_INDEX_BASE_ZERO);
  }
  std::vector<int> row(r->row_ptr.begin(), r->row_ptr.end()), col(r->col_idx.begin(), r->col_idx.end());
  std::vector<int> qre(n), rowB = row, colB = col, map(nnz);
  if (ok) FE_SP(cusolverSpXcsrsymamdHost(sp, n, nnz, dA, row.data(), col.data(), qre.data()), "symamd");
  size_t bsz = 0;
  if (ok)
    FE_SP(cusolverSpXcsrperm_bufferSizeHost(sp, n, n, nnz, dA, rowB.data(), colB.data(), qre.data(), qre.data(),
                                            &bsz),
          "csrperm buffer");
  std::vector<char> pbuf(std::max<size_t>(bsz, 1));
  for (int j = 0; j < nnz; ++j) map[j] = j;
  if (ok)
    FE_SP(cusolverSpXcsrpermHost(sp, n, n, nnz, dA, rowB.data(), colB.data(), qre.data(), qre.data(), map.data(),
                                 pbuf.data()),
          "csrperm");
  std::vector<double> valB(nnz);
  for (int j = 0; j < nnz; ++j) valB[j] = val[map[j]];
  if (ok) FE_SP(cusolverSpCreateCsrluInfoHost(&info), "csrluInfo");
  if (ok) FE_SP(cusolverSpXcsrluAnalysisHost(sp, n, nnz, dA, rowB.data(), colB.data(), info), "csrlu analysis");
  size_t internal = 0, work = 0;
  if (ok)
    FE_SP(cusolverSpDcsrluBufferInfoHost(sp, n, nnz, dA, valB.data(), rowB.data(), colB.data(), info, &internal,
                                         &work),
          "csrlu buffer");
  std::vector<char> lbuf(std::max<size_t>(work, 1));
  if (ok)
    FE_SP(cusolverSpDcsrluFactorHost(sp, n, nnz, dA, valB.data(), rowB.data(), colB.data(), info, 0.0,
                                     lbuf.data()),
          "csrlu factor");
  int sing = -1;
  if (ok) FE_SP(cusolverSpDcsrluZeroPivotHost(sp, info, 0.0, &sing), "csrlu zero pivot");
  if (ok && sing >= 0) ok = false, msg = "first tangent is structurally singular";
  int nnzL = 0, nnzU = 0;
  if (ok) FE_SP(cusolverSpXcsrluNnzHost(sp, &nnzL, &nnzU, info), "csrlu nnz");
  std::vector<int> Plu(n), Qlu(n), rowL(n + 1), colL(std::max(nnzL, 1)), rowU(n + 1), colU(std::max(nnzU, 1));
  std::vector<double> valL(std::max(nnzL, 1)), valU(std::max(nnzU, 1));
  if (ok)
    FE_SP(cusolverSpDcsrluExtractHost(sp, Plu.data(), Qlu.data(), dA, valL.data(), rowL.data(), colL.data(), dA,
                                      valU.data(), rowU.data(), colU.data(), info, lbuf.data()),
          "csrlu extract");
  int ldiag = 0;
  for (int i = 0; ok && i < n; ++i)
    for (int k = rowL[i]; k < rowL[i + 1]; ++k) ldiag += colL[k] == i;
  const std::string lu_info = " [n " + std::to_string(n) + ", nnzA " + std::to_string(nnz) + ", nnzL " +
                              std::to_string(nnzL) + " (diag stored " + std::to_string(ldiag) + "), nnzU " +
                              std::to_string(nnzU) + "]";
  std::vector<int> P(n), Q(n);
  for (int j = 0; j < n; ++j) {
    P[j] = qre[Plu[j]];
    Q[j] = qre[Qlu[j]];
  }
  if (info) cusolverSpDestroyCsrluInfoHost(info);
  if (dA) cusparseDestroyMatDescr(dA);
  if (sp) cusolverSpDestroy(sp);
  if (!ok) return set_err(e->ctx, PODECM_ESOLVE, std::string("fe: host LU setup failed: ") + msg);

  if (!e->d_row) {
    PODECM_CUDA_TRY(e->ctx, cudaMalloc(&e->d_row, sizeof(int) * (n + 1)));
    PODECM_CUDA_TRY(e->ctx, cudaMalloc(&e->d_col, sizeof(int) * nnz));
    PODECM_CUDA_TRY(e->ctx, cudaMalloc(&e->d_P, sizeof(int) * n));
    PODECM_CUDA_TRY(e->ctx, cudaMalloc(&e->d_Q, sizeof(int) * n));
    PODECM_CUDA_TRY(e->ctx, cudaMemcpy(e->d_row, row.data(), sizeof(int) * (n + 1), cudaMemcpyHostToDevice));
    PODECM_CUDA_TRY(e->ctx, cudaMemcpy(e->d_col, col.data(), sizeof(int) * nnz, cudaMemcpyHostToDevice));
  }
  PODECM_CUDA_TRY(e->ctx, cudaMemcpy(e->d_P, P.data(), sizeof(int) * n, cudaMemcpyHostToDevice));
  PODECM_CUDA_TRY(e->ctx, cudaMemcpy(e->d_Q, Q.data(), sizeof(int) * n, cudaMemcpyHostToDevice));
  // csrluExtractHost returns L without its unit diagonal
  for (int64_t i = (int64_t)e->rf.size(); ok && i < batch; ++i) {
    cusolverRfHandle_t h = nullptr;
    FE_SP(cusolverRfCreate(&h), "cusolverRfCreate");
    if (!ok) break;
    e->rf.push_back(h);
    FE_SP(cusolverRfSetNumericProperties(h, 0.0, 0.0), "Rf numeric properties");
    // Refactorisation ALG1 + triangular solve ALG3: bitwise run-to-run
    // deterministic (tools/dev/rf_det_probe.sh).  The default ALG0 is not: its
    // ulp-level jitter flips Newton convergence decisions on ill-conditioned
    // increments, and a flipped bisection changes the plastic load path
    // (2.7 % in P-bar on the exact-limit case).  PODECM_RF_ALGS = 10 * factor
    // alg + solve alg overrides it.
    static const int rf_algs = [] {
      const char* v = getenv("PODECM_RF_ALGS");
      return v ? atoi(v) : 13;
    }();
    if (ok)
      FE_SP(cusolverRfSetAlgs(h, (cusolverRfFactorization_t)(rf_algs / 10),
                              (cusolverRfTriangularSolve_t)(rf_algs % 10)),
            "Rf algs");
    if (ok)
      FE_SP(cusolverRfSetMatrixFormat(h, CUSOLVERRF_MATRIX_FORMAT_CSR, CUSOLVERRF_UNIT_DIAGONAL_ASSUMED_L),
            "Rf format");
    if (ok) FE_SP(cusolverRfSetResetValuesFastMode(h, CUSOLVERRF_RESET_VALUES_FAST_MODE_ON), "Rf fast mode");
    if (ok)
      FE_SP(cusolverRfSetupHost(n, nnz, row.data(), col.data(), val.data(), nnzL, rowL.data(), colL.data(),
                                valL.data(), nnzU, rowU.data(), colU.data(), valU.data(), P.data(), Q.data(), h),
            "Rf setup");
    if (ok) FE_SP(cusolverRfAnalyze(h), "Rf analyze");
  }
  FE_DBG("rf setup handles=%zu ok=%d\n", e->rf.size(), (int)ok);
  if (!ok) return set_err(e->ctx, PODECM_ESOLVE, std::string("fe: ") + msg + lu_info);
  return PODECM_OK;
}

}  // namespace

extern "C" {

int podecm_fe_create(podecm_ctx* ctx, podecm_rve* rve, podecm_fe** out) {
  if (!ctx || !rve || !out) return PODECM_ECONFIG;
  auto* e = new podecm_fe;
  e->ctx = ctx;
  e->rve = rve;
  *out = e;
  return PODECM_OK;
}

void podecm_fe_destroy(podecm_fe* e) {
  if (!e) return;
  for (cusolverRfHandle_t h : e->rf) cusolverRfDestroy(h);
  fe_free(e);
  cudaFree(e->d_af);
  cudaFree(e->d_rhs);
  cudaFree(e->d_row);
  cudaFree(e->d_col);
  cudaFree(e->d_P);
  cudaFree(e->d_Q);
  delete e;
}

int64_t podecm_fe_global_iterations(const podecm_fe* e) { return e ? e->global_iters : 0; }

int podecm_fe_solve_batch_ex(podecm_ctx* ctx, void* stream, podecm_fe* e, int64_t n, const double* geom,
                             const double* sched, int K, const podecm_newton* opts, double* pbar,
                             int32_t* iters, double* resid, double* w_final, int32_t* status, double* w_hist,
                             double* p_hist) {
  if (!ctx || !e || !opts) return PODECM_ECONFIG;
  if (n < 0 || K < 0) return set_err(ctx, PODECM_ECONFIG, "negative batch or schedule size");
  if (n == 0 || K == 0) return PODECM_OK;
  if (!geom || !sched || !pbar) return set_err(ctx, PODECM_ECONFIG, "geom, sched, pbar required");
  if (opts->max_bisect < 0 || opts->max_bisect + 1 > kFeMaxStack)
    return set_err(ctx, PODECM_ECONFIG, "max_bisect must lie in [0, 7]");
  if (opts->max_iter < 0) return set_err(ctx, PODECM_ECONFIG, "max_iter must be >= 0");
  if (int rc = fe_alloc(e, n)) return rc;
  auto s = static_cast<cudaStream_t>(stream);
  podecm_rve* r = e->rve;
  const int nr = r->n_red, nq = r->n_qp;
  const int64_t nnz = r->nnz;
  // host copies of the schedule, pinned staging
  std::vector<double> hs((size_t)n * K * 4);
  PODECM_CUDA_TRY(ctx, cudaMemcpyAsync(hs.data(), sched, sizeof(double) * hs.size(), cudaMemcpyDeviceToHost, s));
  double* h_norm = e->h_pin;
  double* h_pb = h_norm + n;
  double* h_fb = h_pb + 4 * n;
  int32_t* h_mask = reinterpret_cast<int32_t*>(h_fb + 4 * n);  // n ints
  int32_t* h_astat = h_mask + n;                                // n ints (fits in 1 double per 2)
  // the failed-attempt and Newton-update masks go to the device by async
  // copies within one global iteration, without a host sync in between: each
  // needs its own pinned buffer (reusing h_mask raced with the pending copy)
  int32_t* h_mask_fail = h_astat + n;
  int32_t* h_mask_solve = h_mask_fail + n;
  // morph (det per qp) and virgin history, w = 0
  if (int rc = podecm_rve_morph(ctx, stream, r, n, geom, e->d_fmi, e->d_det, e->d_mstat)) return rc;
  k_fe_virgin<<<grid_for(n * nq, 256), 256, 0, s>>>(n, nq, e->d_Sc);
  PODECM_CUDA_TRY(ctx, cudaMemsetAsync(e->d_w, 0, sizeof(double) * n * nr, s));
  PODECM_CUDA_TRY(ctx, cudaMemsetAsync(e->d_w0, 0, sizeof(double) * n * nr, s));
  PODECM_LAUNCHED(ctx, 1);
  std::vector<int32_t> mstat(n);
  PODECM_CUDA_TRY(ctx, cudaMemcpyAsync(mstat.data(), e->d_mstat, sizeof(int32_t) * n, cudaMemcpyDeviceToHost, s));
  PODECM_CUDA_TRY(ctx, cudaStreamSynchronize(s));
  std::vector<Inst> in(n);
  std::vector<double> hpbar((size_t)n * K * 4, 0.0), hres((size_t)n * K, 0.0);
  std::vector<int32_t> hit((size_t)n * K, 0), hst(n, 0);
  for (int64_t i = 0; i < n; ++i) {
    Frame f;
    for (int t = 0; t < 4; ++t) {
      f.fp[t] = t == 0 || t == 3 ? 1.0 : 0.0;
      f.ft[t] = hs[((size_t)i * K) * 4 + t];
    }
    f.depth = opts->max_bisect;
    in[i].stack.push_back(f);
    if (mstat[i]) {  // folding morph: SolveError (morph.cpp:116-119)
      in[i].active = false;
      in[i].status = PODECM_ESOLVE;
    }
  }
  const int64_t max_global = (int64_t)K * (opts->max_iter + 1) * (2ll << opts->max_bisect) + 8;
  e->global_iters = 0;
  std::vector<double*> kp(n), xp(n);
  for (int64_t i = 0; i < n; ++i) {
    kp[i] = e->d_K + (size_t)i * nnz;
    xp[i] = e->d_x + (size_t)i * nr;
  }
  for (int64_t git = 0; git < max_global; ++git) {
    bool any = false;
    for (int64_t i = 0; i < n; ++i) any = any || in[i].active;
    if (!any) break;
    ++e->global_iters;
    for (int64_t i = 0; i < n; ++i) {
      const Frame& f = in[i].stack.back();
      for (int t = 0; t < 4; ++t) h_fb[4 * i + t] = f.ft[t];
    }
    PODECM_CUDA_TRY(ctx, cudaMemcpyAsync(e->d_fb, h_fb, sizeof(double) * 4 * n, cudaMemcpyHostToDevice, s));
    // K2: residual, tangent, trial history and stress field of every instance
    if (int rc = podecm_assemble_batch(ctx, stream, r, n, geom, nullptr, e->d_fb, e->d_w, e->d_Sc, e->d_St,
                                       e->d_f, e->d_K, e->d_pf, e->d_astat))
      return rc;
    k_fe_norm<<<(unsigned)n, 256, 0, s>>>(nr, e->d_f, e->d_norm);
    PODECM_LAUNCHED(ctx, 1);
    PODECM_CUDA_TRY(ctx, cudaMemcpyAsync(h_norm, e->d_norm, sizeof(double) * n, cudaMemcpyDeviceToHost, s));
    PODECM_CUDA_TRY(ctx, cudaMemcpyAsync(h_astat, e->d_astat, sizeof(int32_t) * n, cudaMemcpyDeviceToHost, s));
    PODECM_CUDA_TRY(ctx, cudaStreamSynchronize(s));
    // Newton logic per instance (microfem.cpp:157-186)
    enum { kNone = 0, kSolve = 1, kConv = 2, kFail = 3, kZeroPivot = 4 };
    std::vector<int> act(n, kNone);
    for (int64_t i = 0; i < n; ++i) {
      Inst& c = in[i];
      if (!c.active) continue;
      if (h_astat[i] != 0) {  // material SolveError inside assemble
        act[i] = kFail;
        continue;
      }
      const double rn = h_norm[i];
      if (c.it == 0) {
        c.r0 = rn;
        c.tol = std::max(opts->eps_rel * std::max(rn, opts->force_ref), opts->eps_abs);
      }
      if (rn <= c.tol)
        act[i] = kConv;
      else if (c.it == opts->max_iter)
        act[i] = kFail;
      else
        act[i] = kSolve;
    }
    // converged attempts: commit the trial history, pbar on the last sub-step
    bool any_conv = false, any_fail = false, any_solve = false;
    for (int64_t i = 0; i < n; ++i) {
      h_mask[i] = act[i] == kConv;
      any_conv |= act[i] == kConv;
      any_fail |= act[i] == kFail;
      any_solve |= act[i] == kSolve;
    }
    if (any_conv) {
      PODECM_CUDA_TRY(ctx, cudaMemcpyAsync(e->d_mask, h_mask, sizeof(int32_t) * n, cudaMemcpyHostToDevice, s));
      k_fe_copy<<<grid_for(n * 6 * nq, 256), 256, 0, s>>>(n, 6 * (int64_t)nq, e->d_mask, e->d_St, e->d_Sc);
      k_fe_copy<<<grid_for(n * nr, 256), 256, 0, s>>>(n, nr, e->d_mask, e->d_w, e->d_w0);
      k_fe_pbar<<<(unsigned)n, 256, 0, s>>>(nq, r->d_w, e->d_det, e->d_pf, e->d_pb);
      PODECM_LAUNCHED(ctx, 3);
      PODECM_CUDA_TRY(ctx, cudaMemcpyAsync(h_pb, e->d_pb, sizeof(double) * 4 * n, cudaMemcpyDeviceToHost, s));
      PODECM_CUDA_TRY(ctx, cudaStreamSynchronize(s));
      for (int64_t i = 0; i < n; ++i) {
        if (act[i] != kConv) continue;
        Inst& c = in[i];
        c.iters_acc += c.it;
        c.stack.pop_back();
        c.it = 0;
        if (c.stack.empty()) {  // increment done (solve_rve, microfem.cpp:221-236)
          for (int t = 0; t < 4; ++t) hpbar[((size_t)i * K + c.k) * 4 + t] = h_pb[4 * i + t];
          if (w_hist)  // RveSolution::Step::w_red (snapshot collection, pipeline.cpp:167-175)
            PODECM_CUDA_TRY(ctx, cudaMemcpyAsync(w_hist + ((size_t)i * K + c.k) * nr, e->d_w + (size_t)i * nr,
                                                 sizeof(double) * nr, cudaMemcpyDeviceToDevice, s));
          if (p_hist)  // RveSolution::Step::p_field
            PODECM_CUDA_TRY(ctx, cudaMemcpyAsync(p_hist + ((size_t)i * K + c.k) * 4 * nq,
                                                 e->d_pf + (size_t)i * 4 * nq, sizeof(double) * 4 * nq,
                                                 cudaMemcpyDeviceToDevice, s));
          hit[(size_t)i * K + c.k] = c.iters_acc;
          hres[(size_t)i * K + c.k] = h_norm[i];
          c.iters_acc = 0;
          c.k += 1;
          if (c.k == K) {
            c.active = false;
          } else {
            Frame f;
            for (int t = 0; t < 4; ++t) {
              f.fp[t] = hs[((size_t)i * K + c.k - 1) * 4 + t];
              f.ft[t] = hs[((size_t)i * K + c.k) * 4 + t];
            }
            f.depth = opts->max_bisect;
            c.stack.push_back(f);
          }
        }
      }
    }
    // failed attempts: restore w, bisect (solve_step_adaptive, microfem.cpp:190-211)
    if (any_fail) {
      for (int64_t i = 0; i < n; ++i) h_mask_fail[i] = act[i] == kFail;
      PODECM_CUDA_TRY(ctx, cudaMemcpyAsync(e->d_mask, h_mask_fail, sizeof(int32_t) * n, cudaMemcpyHostToDevice, s));
      k_fe_copy<<<grid_for(n * nr, 256), 256, 0, s>>>(n, nr, e->d_mask, e->d_w0, e->d_w);
      PODECM_LAUNCHED(ctx, 1);
      for (int64_t i = 0; i < n; ++i) {
        if (act[i] != kFail) continue;
        Inst& c = in[i];
        c.it = 0;
        Frame top = c.stack.back();
        if (top.depth <= 0 || (int)c.stack.size() + 1 > kFeMaxStack) {
          c.active = false;
          c.status = PODECM_ESOLVE;
          continue;
        }
        c.stack.pop_back();
        Frame second = top, first = top;
        for (int t = 0; t < 4; ++t) {
          const double mid = 0.5 * (top.fp[t] + top.ft[t]);
          first.ft[t] = mid;
          second.fp[t] = mid;
        }
        first.depth = second.depth = top.depth - 1;
        c.stack.push_back(second);
        c.stack.push_back(first);
      }
    }
    // Newton updates: one batched refactorisation + solve for the whole batch
    if (any_solve) {
      if (int rc = rf_setup(e, s, n)) return rc;
      for (int64_t i = 0; i < n; ++i) h_mask_solve[i] = act[i] == kSolve;
      PODECM_CUDA_TRY(ctx, cudaMemcpyAsync(e->d_mask, h_mask_solve, sizeof(int32_t) * n, cudaMemcpyHostToDevice, s));
      k_fe_negate<<<grid_for(n * nr, 256), 256, 0, s>>>(n * nr, e->d_f, e->d_x);
      PODECM_LAUNCHED(ctx, 1);
      PODECM_CUDA_TRY(ctx, cudaStreamSynchronize(s));  // Rf runs on the legacy stream
      bool ok = true;
      std::string msg;
      {
        KTimer kt(ctx, s, "rf_refactor_solve");
        for (int64_t i = 0; ok && i < n; ++i) {
          if (act[i] != kSolve) continue;
          cusolverRfHandle_t h = e->rf[i];
          FE_SP(cusolverRfResetValues(nr, (int)nnz, e->d_row, e->d_col, kp[i], e->d_P, e->d_Q, h), "Rf reset values");
          if (!ok) break;
          const cusolverStatus_t rs = cusolverRfRefactor(h);
          if (rs == CUSOLVER_STATUS_ZERO_PIVOT) {  // factorization failed
            h_mask_solve[i] = 0;
            act[i] = kZeroPivot;
            continue;
          }
          FE_SP(rs, "Rf refactor");
          if (ok) FE_SP(cusolverRfSolve(h, e->d_P, e->d_Q, 1, e->d_tmp, nr, xp[i], nr), "Rf solve");
        }
        cudaDeviceSynchronize();
        FE_DBG("solve ok=%d err=%s\n", (int)ok, cudaGetErrorString(cudaGetLastError()));
      }
      if (!ok) return set_err(ctx, PODECM_ESOLVE, std::string("fe: ") + msg);
      PODECM_CUDA_TRY(ctx, cudaMemcpyAsync(e->d_mask, h_mask_solve, sizeof(int32_t) * n, cudaMemcpyHostToDevice, s));
      k_fe_update<<<grid_for(n * nr, 256), 256, 0, s>>>(n, nr, e->d_mask, e->d_x, e->d_w);
      PODECM_LAUNCHED(ctx, 1);
      for (int64_t i = 0; i < n; ++i) {
        if (act[i] == kSolve) in[i].it += 1;
        // zero pivot ("cell tangent factorization failed", microfem.cpp:182):
        // w is left unchanged and the next assembly fails the attempt
        if (act[i] == kZeroPivot) in[i].it = opts->max_iter;
      }
    }
  }
  for (int64_t i = 0; i < n; ++i)
    if (in[i].active) in[i].status = PODECM_ESOLVE, in[i].active = false;  // global budget exhausted
  unsigned int nfail = 0;
  for (int64_t i = 0; i < n; ++i) {
    hst[i] = in[i].status;
    nfail += in[i].status != 0;
  }
  PODECM_CUDA_TRY(ctx, cudaMemcpyAsync(pbar, hpbar.data(), sizeof(double) * hpbar.size(), cudaMemcpyHostToDevice, s));
  if (iters)
    PODECM_CUDA_TRY(ctx, cudaMemcpyAsync(iters, hit.data(), sizeof(int32_t) * hit.size(), cudaMemcpyHostToDevice, s));
  if (resid)
    PODECM_CUDA_TRY(ctx, cudaMemcpyAsync(resid, hres.data(), sizeof(double) * hres.size(), cudaMemcpyHostToDevice, s));
  if (status)
    PODECM_CUDA_TRY(ctx, cudaMemcpyAsync(status, hst.data(), sizeof(int32_t) * n, cudaMemcpyHostToDevice, s));
  if (w_final)
    PODECM_CUDA_TRY(ctx, cudaMemcpyAsync(w_final, e->d_w, sizeof(double) * n * nr, cudaMemcpyDeviceToDevice, s));
  if (nfail) {  // context-wide failure count (podecm_check reports SolveError)
    k_fe_addfail<<<1, 1, 0, s>>>(ctx->d_fail, nfail);
    PODECM_LAUNCHED(ctx, 1);
  }
  PODECM_CUDA_TRY(ctx, cudaStreamSynchronize(s));
  return PODECM_OK;
}


int podecm_fe_effective_stiffness_batch(podecm_ctx* ctx, void* stream, podecm_fe* e, int64_t n,
                                        const double* geom, const double* st0, const double* fbar,
                                        const double* w, double* abar, int32_t* status) {
  if (!ctx || !e) return PODECM_ECONFIG;
  if (n < 0) return set_err(ctx, PODECM_ECONFIG, "negative batch size");
  if (n == 0) return PODECM_OK;
  if (!geom || !st0 || !fbar || !w || !abar)
    return set_err(ctx, PODECM_ECONFIG, "geom, st0, fbar, w, abar required");
  if (int rc = fe_alloc(e, n)) return rc;
  podecm_rve* r = e->rve;
  const int nr = r->n_red, nq = r->n_qp;
  const int64_t nnz = r->nnz;
  auto s = static_cast<cudaStream_t>(stream);
  if (e->af_cap < n) {
    cudaFree(e->d_af);
    cudaFree(e->d_rhs);
    e->d_af = e->d_rhs = nullptr;
    e->af_cap = 0;
    PODECM_CUDA_TRY(ctx, cudaMalloc(&e->d_af, sizeof(double) * (size_t)n * 16 * nq));
    PODECM_CUDA_TRY(ctx, cudaMalloc(&e->d_rhs, sizeof(double) * (size_t)n * 4 * nr));
    e->af_cap = n;
  }
  if (int rc = podecm_rve_morph(ctx, stream, r, n, geom, e->d_fmi, e->d_det, e->d_mstat)) return rc;
  // tangent assembly with the tangent field (microfem.cpp:247-251)
  if (int rc = podecm_assemble_batch_ex(ctx, stream, r, n, geom, nullptr, fbar, w, st0, nullptr, e->d_f, e->d_K,
                                        nullptr, e->d_astat, e->d_af))
    return rc;
  // right-hand sides (microfem.cpp:262-281): rhs_c = -(row sums of A(:, :, c))
  for (int c = 0; c < 4; ++c)
    if (int rc = assemble_field_rows(ctx, s, r, n, geom, nullptr, e->d_af, c, e->d_rhs + (size_t)c * n * nr))
      return rc;
  k_fe_negate<<<grid_for(4 * n * nr, 256), 256, 0, s>>>(4 * n * nr, e->d_rhs, e->d_rhs);
  PODECM_LAUNCHED(ctx, 1);
  if (int rc = rf_setup(e, s, n)) return rc;
  std::vector<int32_t> ast(n), mst(n);
  PODECM_CUDA_TRY(ctx, cudaMemcpyAsync(ast.data(), e->d_astat, sizeof(int32_t) * n, cudaMemcpyDeviceToHost, s));
  PODECM_CUDA_TRY(ctx, cudaMemcpyAsync(mst.data(), e->d_mstat, sizeof(int32_t) * n, cudaMemcpyDeviceToHost, s));
  PODECM_CUDA_TRY(ctx, cudaStreamSynchronize(s));  // Rf runs on the legacy stream
  std::vector<int32_t> hst(n, 0);
  bool ok = true;
  std::string msg;
  {
    KTimer kt(ctx, s, "rf_refactor_solve");
    for (int64_t i = 0; ok && i < n; ++i) {
      if (ast[i] || mst[i]) {  // material or morph SolveError
        hst[i] = PODECM_ESOLVE;
        continue;
      }
      cusolverRfHandle_t h = e->rf[i];
      FE_SP(cusolverRfResetValues(nr, (int)nnz, e->d_row, e->d_col, e->d_K + (size_t)i * nnz, e->d_P, e->d_Q, h),
            "Rf reset values");
      if (!ok) break;
      const cusolverStatus_t rs = cusolverRfRefactor(h);
      if (rs == CUSOLVER_STATUS_ZERO_PIVOT) {  // "tangent factorization failed" (microfem.cpp:254-255)
        hst[i] = PODECM_ESOLVE;
        continue;
      }
      FE_SP(rs, "Rf refactor");
      for (int c = 0; ok && c < 4; ++c)
        FE_SP(cusolverRfSolve(h, e->d_P, e->d_Q, 1, e->d_tmp, nr, e->d_rhs + ((size_t)c * n + i) * nr, nr),
              "Rf solve");
    }
    cudaDeviceSynchronize();
  }
  if (!ok) return set_err(ctx, PODECM_ESOLVE, std::string("fe: ") + msg);
  k_fe_abar<<<(unsigned)n, 256, 0, s>>>(nq, nr, n, r->d_elems, r->d_node_dof, r->d_grad, r->d_w, e->d_fmi, e->d_det,
                                        e->d_af, e->d_rhs, abar);
  PODECM_LAUNCHED(ctx, 1);
  unsigned int nfail = 0;
  for (int64_t i = 0; i < n; ++i) nfail += hst[i] != 0;
  if (status)
    PODECM_CUDA_TRY(ctx, cudaMemcpyAsync(status, hst.data(), sizeof(int32_t) * n, cudaMemcpyHostToDevice, s));
  if (nfail) {
    k_fe_addfail<<<1, 1, 0, s>>>(ctx->d_fail, nfail);
    PODECM_LAUNCHED(ctx, 1);
  }
  PODECM_CUDA_TRY(ctx, cudaStreamSynchronize(s));
  return PODECM_OK;
}


int podecm_fe_solve_batch(podecm_ctx* ctx, void* stream, podecm_fe* e, int64_t n, const double* geom,
                          const double* sched, int K, const podecm_newton* opts, double* pbar, int32_t* iters,
                          double* resid, double* w_final, int32_t* status) {
  return podecm_fe_solve_batch_ex(ctx, stream, e, n, geom, sched, K, opts, pbar, iters, resid, w_final, status,
                                  nullptr, nullptr);
}

int podecm_weighted_stress_field(podecm_ctx* ctx, void* stream, podecm_rve* r, int64_t n, const double* geom,
                                 const double* p_field, double* W) {
  if (!ctx || !r || !geom || !p_field || !W) return PODECM_ECONFIG;
  if (n <= 0) return PODECM_OK;
  auto s = static_cast<cudaStream_t>(stream);
  const int nq = r->n_qp;
  double *fmi = nullptr, *det = nullptr;
  cudaError_t ce = cudaMallocAsync(&fmi, sizeof(double) * (size_t)n * 4 * nq, s);
  if (ce == cudaSuccess) ce = cudaMallocAsync(&det, sizeof(double) * (size_t)n * nq, s);
  int rc = ce == cudaSuccess ? podecm_rve_morph(ctx, stream, r, n, geom, fmi, det, nullptr)
                             : cuda_err(ctx, ce, "weighted_stress_field: allocation");
  if (!rc) {
    k_fe_wstress<<<grid_for(n * nq, 256), 256, 0, s>>>(n, nq, fmi, det, p_field, W);
    rc = cudaGetLastError() == cudaSuccess ? PODECM_OK : set_err(ctx, PODECM_ECUDA, "launch");
    if (!rc) ctx->launches += 1;
  }
  if (fmi) cudaFreeAsync(fmi, s);
  if (det) cudaFreeAsync(det, s);
  return rc;
}

}  // extern "C"
