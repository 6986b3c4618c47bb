// Dev probe of the cuSOLVER Rf call sequence on a small nonsymmetric sparse
// matrix (not part of the library): host csrlu + Rf (single / batched).
#include <cusolverRf.h>
#include <cusolverSp.h>
#include <cusolverSp_LOWLEVEL_PREVIEW.h>
#include <cusparse.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <vector>
#define CK(x) do { int s_ = (int)(x); printf("%-40s -> %d\n", #x, s_); fflush(stdout); if (s_) return 1; } while (0)
int main(int argc, char** argv) {
  const int batched = argc > 1 ? atoi(argv[1]) : 1, stored = argc > 2 ? atoi(argv[2]) : 1;
  const int fast = argc > 3 ? atoi(argv[3]) : 1, falg = argc > 4 ? atoi(argv[4]) : 0, salg = argc > 5 ? atoi(argv[5]) : 1;
  const int n = 10;
  std::vector<int> row(n + 1), col;
  std::vector<double> val;
  for (int i = 0; i < n; ++i) {
    for (int j = i - 1; j <= i + 1; ++j)
      if (j >= 0 && j < n) { col.push_back(j); val.push_back(j == i ? 4.0 : (j < i ? -1.0 : -1.5)); }
    row[i + 1] = (int)col.size();
  }
  const int nnz = (int)col.size();
  cusolverSpHandle_t sp; CK(cusolverSpCreate(&sp));
  cusparseMatDescr_t d; cusparseCreateMatDescr(&d);
  cusparseSetMatType(d, CUSPARSE_MATRIX_TYPE_GENERAL); cusparseSetMatIndexBase(d, CUSPARSE_INDEX_BASE_ZERO);
  csrluInfoHost_t info; CK(cusolverSpCreateCsrluInfoHost(&info));
  CK(cusolverSpXcsrluAnalysisHost(sp, n, nnz, d, row.data(), col.data(), info));
  size_t in_b = 0, wk = 0;
  CK(cusolverSpDcsrluBufferInfoHost(sp, n, nnz, d, val.data(), row.data(), col.data(), info, &in_b, &wk));
  std::vector<char> buf(wk + 1);
  CK(cusolverSpDcsrluFactorHost(sp, n, nnz, d, val.data(), row.data(), col.data(), info, 1.0, buf.data()));
  int nL, nU; CK(cusolverSpXcsrluNnzHost(sp, &nL, &nU, info));
  std::vector<int> P(n), Q(n), rL(n + 1), cL(nL), rU(n + 1), cU(nU);
  std::vector<double> vL(nL), vU(nU);
  CK(cusolverSpDcsrluExtractHost(sp, P.data(), Q.data(), d, vL.data(), rL.data(), cL.data(), d, vU.data(), rU.data(), cU.data(), info, buf.data()));
  printf("nnzL %d nnzU %d, L row0 cols:", nL, nU);
  for (int k = rL[0]; k < rL[2]; ++k) printf(" %d", cL[k]);
  printf("\n");
  cusolverRfHandle_t rf; CK(cusolverRfCreate(&rf));
  CK(cusolverRfSetNumericProperties(rf, 0.0, 0.0));
  CK(cusolverRfSetAlgs(rf, (cusolverRfFactorization_t)falg, (cusolverRfTriangularSolve_t)salg));
  CK(cusolverRfSetMatrixFormat(rf, CUSOLVERRF_MATRIX_FORMAT_CSR, stored ? CUSOLVERRF_UNIT_DIAGONAL_STORED_L : CUSOLVERRF_UNIT_DIAGONAL_ASSUMED_L));
  CK(cusolverRfSetResetValuesFastMode(rf, fast ? CUSOLVERRF_RESET_VALUES_FAST_MODE_ON : CUSOLVERRF_RESET_VALUES_FAST_MODE_OFF));
  int *dr, *dc, *dP, *dQ; double *dv, *dx, *dt;
  cudaMalloc(&dr, 4 * (n + 1)); cudaMalloc(&dc, 4 * nnz); cudaMalloc(&dP, 4 * n); cudaMalloc(&dQ, 4 * n);
  cudaMalloc(&dv, 8 * nnz); cudaMalloc(&dx, 8 * n * 2); cudaMalloc(&dt, 8 * n * 4);
  cudaMemcpy(dr, row.data(), 4 * (n + 1), cudaMemcpyHostToDevice); cudaMemcpy(dc, col.data(), 4 * nnz, cudaMemcpyHostToDevice);
  cudaMemcpy(dP, P.data(), 4 * n, cudaMemcpyHostToDevice); cudaMemcpy(dQ, Q.data(), 4 * n, cudaMemcpyHostToDevice);
  cudaMemcpy(dv, val.data(), 8 * nnz, cudaMemcpyHostToDevice);
  std::vector<double> b(n, 1.0);
  cudaMemcpy(dx, b.data(), 8 * n, cudaMemcpyHostToDevice); cudaMemcpy(dx + n, b.data(), 8 * n, cudaMemcpyHostToDevice);
  if (batched) {
    std::vector<double*> hv = {val.data(), val.data()};
    CK(cusolverRfBatchSetupHost(2, n, nnz, row.data(), col.data(), hv.data(), nL, rL.data(), cL.data(), vL.data(), nU, rU.data(), cU.data(), vU.data(), P.data(), Q.data(), rf));
    CK(cusolverRfBatchAnalyze(rf));
    std::vector<double*> dvv = {dv, dv};
    CK(cusolverRfBatchResetValues(2, n, nnz, dr, dc, dvv.data(), dP, dQ, rf));
    CK(cusolverRfBatchRefactor(rf));
    std::vector<double*> xx = {dx, dx + n};
    CK(cusolverRfBatchSolve(rf, dP, dQ, 1, dt, n, xx.data(), n));
  } else {
    CK(cusolverRfSetupHost(n, nnz, row.data(), col.data(), val.data(), nL, rL.data(), cL.data(), vL.data(), nU, rU.data(), cU.data(), vU.data(), P.data(), Q.data(), rf));
    CK(cusolverRfAnalyze(rf));
    CK(cusolverRfResetValues(n, nnz, dr, dc, dv, dP, dQ, rf));
    CK(cusolverRfRefactor(rf));
    CK(cusolverRfSolve(rf, dP, dQ, 1, dt, n, dx, n));
  }
  cudaDeviceSynchronize();
  std::vector<double> x(n);
  cudaMemcpy(x.data(), dx, 8 * n, cudaMemcpyDeviceToHost);
  double rmax = 0;
  for (int i = 0; i < n; ++i) {
    double s = 0;
    for (int k = row[i]; k < row[i + 1]; ++k) s += val[k] * x[col[k]];
    rmax = fmax(rmax, fabs(s - 1.0));
  }
  printf("residual max %.3e  x0 %.6f\n", rmax, x[0]);
  return 0;
}
