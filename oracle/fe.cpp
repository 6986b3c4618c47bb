// ORACLE — TEST INFRASTRUCTURE ONLY (see oracle.hpp).
// Restates /root/reference/proj/src/microfem.cpp:132-238: effective_stress,
// solve_step (full-order Newton), solve_step_adaptive (bisection) and
// solve_rve, around the restated assemble.  Eigen::SparseLU is replaced by a
// dense partial-pivot LU of the assembled CSR tangent (the tests use small
// cells); both are direct solves, and the stated parity is 1e-8 on the
// homogenised stress history.
#include "oracle.hpp"

#include <algorithm>
#include <cmath>

namespace orc {

namespace {

// A(i, j, k, l) of a Tensor4 stored as m[r + 4c], r = i + 2j, c = k + 2l
inline double A4(const double* m, int i, int j, int k, int l) { return m[(i + 2 * j) + 4 * (k + 2 * l)]; }

struct FeStep {
  std::vector<double> w, pf;  // pf: converged p_field [q][4]
  std::vector<PlasticState> states;
  Mat2 pbar;
  int iters = 0;
  double residual = 0, initial_residual = 0;
};

// microfem.cpp:132-140 (p_field flattened [q][4])
Mat2 effective_stress(const RveProblem& prob, const std::vector<double>& pf, const Morph& mo) {
  Mat2 pbar;
  for (int q = 0; q < prob.cache.n_qp(); ++q) {
    const double wq = prob.cache.w[q] * mo.det[q];
    for (int k = 0; k < 4; ++k) pbar.a[k] += wq * pf[4 * (size_t)q + k];
  }
  for (int k = 0; k < 4; ++k) pbar.a[k] /= prob.cell_volume;
  return pbar;
}

// microfem.cpp:142-188
FeStep solve_step(const RveProblem& prob, const Morph& mo, const std::vector<PlasticState>& s0,
                  const Mat2& fbar, const std::vector<double>& w_init, const NewtonOpts& o) {
  FeStep res;
  res.w = w_init;
  const int n = prob.dofs.n_red;
  double f0 = 0.0;
  for (int it = 0; it <= o.max_iter; ++it) {
    std::vector<double> f, pf;
    Csr K;
    res.states.clear();
    assemble(prob, mo, s0, &res.states, fbar, res.w, true, f, &K, &pf);
    double ss = 0.0;
    for (double v : f) ss += v * v;
    const double rn = std::sqrt(ss);
    if (it == 0) {
      f0 = rn;
      res.initial_residual = rn;
    }
    const double tol = std::max(o.eps_rel * std::max(f0, o.force_ref), o.eps_abs);
    if (rn <= tol) {
      res.iters = it;
      res.residual = rn;
      res.pbar = effective_stress(prob, pf, mo);
      res.pf = std::move(pf);
      return res;
    }
    if (it == o.max_iter) break;
    std::vector<double> dense((size_t)n * n, 0.0);  // column-major
    for (int r = 0; r < n; ++r)
      for (int k = K.row_ptr[r]; k < K.row_ptr[r + 1]; ++k) dense[(size_t)K.col[k] * n + r] = K.val[k];
    std::vector<double> neg(n);
    for (int i = 0; i < n; ++i) neg[i] = -f[i];
    const std::vector<double> dw = lu_solve(std::move(dense), n, neg);
    for (int i = 0; i < n; ++i) res.w[i] += dw[i];
  }
  throw SolveError("cell Newton did not converge");
}

// microfem.cpp:190-211
FeStep solve_step_adaptive(const RveProblem& prob, const Morph& mo, const std::vector<PlasticState>& s0,
                           const Mat2& fprev, const Mat2& fbar, const std::vector<double>& w_init,
                           const NewtonOpts& o, int max_bisect) {
  try {
    return solve_step(prob, mo, s0, fbar, w_init, o);
  } catch (const SolveError&) {
    if (max_bisect <= 0) throw;
  }
  Mat2 mid;
  for (int k = 0; k < 4; ++k) mid.a[k] = 0.5 * (fprev.a[k] + fbar.a[k]);
  FeStep half = solve_step_adaptive(prob, mo, s0, fprev, mid, w_init, o, max_bisect - 1);
  FeStep full = solve_step_adaptive(prob, mo, half.states, mid, fbar, half.w, o, max_bisect - 1);
  full.iters += half.iters;
  full.initial_residual = std::max(full.initial_residual, half.initial_residual);
  return full;
}

}  // namespace

// microfem.cpp:213-238 (solve_rve)
std::vector<RomStepRecord> fe_solve(const RveProblem& prob, const Morph& mo, const std::vector<Mat2>& schedule,
                                    const NewtonOpts& o, int max_bisect, std::vector<double>* w_final,
                                    std::vector<double>* w_hist, std::vector<double>* p_hist) {
  std::vector<PlasticState> committed(prob.cache.n_qp());
  std::vector<double> w(prob.dofs.n_red, 0.0);
  Mat2 fprev = Mat2::identity();
  std::vector<RomStepRecord> recs;
  for (const Mat2& fbar : schedule) {
    FeStep st = solve_step_adaptive(prob, mo, committed, fprev, fbar, w, o, max_bisect);
    fprev = fbar;
    committed = st.states;
    w = st.w;
    if (w_hist) w_hist->insert(w_hist->end(), st.w.begin(), st.w.end());
    if (p_hist) p_hist->insert(p_hist->end(), st.pf.begin(), st.pf.end());
    RomStepRecord r;
    r.pbar = st.pbar;
    r.iters = st.iters;
    r.residual = st.residual;
    recs.push_back(r);
  }
  if (w_final) *w_final = w;
  return recs;
}

// microfem.cpp:240-313: tangent assembly with the tangent field, one
// factorisation, four unit macro perturbations E_kl (k outer, l inner).
void fe_effective_stiffness(const RveProblem& prob, const Morph& mo, const std::vector<PlasticState>& s0,
                            const Mat2& fbar, const std::vector<double>& w, double out[16]) {
  const Mesh& mesh = prob.mesh;
  const QuadCache& cache = prob.cache;
  const int nqp = cache.n_qp(), n = prob.dofs.n_red;
  std::vector<double> f, pf, af;
  Csr K;
  assemble(prob, mo, s0, nullptr, fbar, w, true, f, &K, nullptr, &af);
  std::vector<double> dense((size_t)n * n, 0.0);
  for (int r = 0; r < n; ++r)
    for (int k = K.row_ptr[r]; k < K.row_ptr[r + 1]; ++k) dense[(size_t)K.col[k] * n + r] = K.val[k];
  std::vector<double> rhs((size_t)n * 4, 0.0);  // column-major n x 4
  for (int q = 0; q < nqp; ++q) {
    const int e = cache.elem_of[q];
    const double* g = &cache.grad[(size_t)q * 8];
    const Mat2& fmi = mo.fmu_inv[q];
    const double wq = cache.w[q] * mo.det[q];
    double gt[4][2];
    for (int a = 0; a < 4; ++a)
      for (int j = 0; j < 2; ++j) gt[a][j] = g[2 * a] * fmi(0, j) + g[2 * a + 1] * fmi(1, j);
    const double* a4 = &af[16 * (size_t)q];
    for (int a = 0; a < 4; ++a) {
      const int ra = prob.dofs.node_dof[mesh.elems[4 * e + a]];
      if (ra < 0) continue;
      for (int k = 0; k < 2; ++k)
        for (int l = 0; l < 2; ++l) {
          const int col = k + 2 * l;
          for (int i = 0; i < 2; ++i)
            rhs[(size_t)col * n + ra + i] -= wq * (A4(a4, i, 0, k, l) * gt[a][0] + A4(a4, i, 1, k, l) * gt[a][1]);
        }
    }
  }
  double abar[16] = {0};
  for (int k = 0; k < 2; ++k)
    for (int l = 0; l < 2; ++l) {
      const int col = k + 2 * l;
      const std::vector<double> qk = lu_solve(dense, n, std::vector<double>(rhs.begin() + (size_t)col * n,
                                                                          rhs.begin() + (size_t)(col + 1) * n));
      std::vector<double> qf(2 * (size_t)mesh.n_nodes, 0.0);  // DofMap::expand
      for (int i = 0; i < mesh.n_nodes; ++i) {
        const int d = prob.dofs.node_dof[i];
        if (d < 0) continue;
        qf[2 * i] = qk[d];
        qf[2 * i + 1] = qk[d + 1];
      }
      for (int q = 0; q < nqp; ++q) {
        const int e = cache.elem_of[q];
        const double* g = &cache.grad[(size_t)q * 8];
        const Mat2& fmi = mo.fmu_inv[q];
        const double wq = cache.w[q] * mo.det[q];
        const double* a4 = &af[16 * (size_t)q];
        Mat2 gq;
        for (int a = 0; a < 4; ++a) {
          const int node = mesh.elems[4 * e + a];
          for (int i = 0; i < 2; ++i)
            for (int j = 0; j < 2; ++j) gq(i, j) += qf[2 * node + i] * g[2 * a + j];
        }
        Mat2 df = mul(gq, fmi);
        df(k, l) += 1.0;
        for (int r = 0; r < 4; ++r) {  // contract: m * flatten(df)
          double c = 0.0;
          for (int t = 0; t < 4; ++t) c += a4[r + 4 * t] * df.a[t];
          abar[r + 4 * col] += wq * c;
        }
      }
    }
  for (int t = 0; t < 16; ++t) out[t] = abar[t] / prob.cell_volume;
}

}  // namespace orc
