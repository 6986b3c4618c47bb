// ORACLE — TEST INFRASTRUCTURE ONLY (see oracle.hpp).
// Restates /root/reference/proj/src/rom.cpp:16-241: right_mult_op,
// rom_assemble, rom_effective_stress, rom_solve_step (Newton with a dense
// partial-pivot LU, Eigen::PartialPivLU semantics), the adaptive bisection,
// rom_solve and rom_effective_stiffness.
#include "oracle.hpp"

#include <algorithm>

namespace orc {

namespace {

struct RomAsm {
  std::vector<double> f;  // N
  std::vector<double> k;  // N x N column-major
  std::vector<Mat2> p;
};

// rom.cpp:34-66.  mapped = mode_grads_p * R(Fmu^-1) (rom.cpp:16-26: only the
// two nonzeros k(i+2j, i+2l) = m(j,l) contribute to each coefficient).
RomAsm rom_assemble(const RveProblem& prob, const RomModel& model, const std::vector<Mat2>& fmi,
                    const std::vector<double>& det, const std::vector<PlasticState>& s0,
                    std::vector<PlasticState>& s1, const Mat2& fbar, const std::vector<double>& a) {
  const int n = model.N, np = (int)model.ids.size();
  RomAsm out;
  out.f.assign(n, 0.0);
  out.k.assign((size_t)n * n, 0.0);
  out.p.resize(np);
  std::vector<double> mapped((size_t)n * 4), ma((size_t)n * 4);
  for (int p = 0; p < np; ++p) {
    const double* mg = &model.mode_grads[(size_t)p * n * 4];
    const Mat2& m = fmi[p];
    for (int i = 0; i < n; ++i)
      for (int ii = 0; ii < 2; ++ii)
        for (int l = 0; l < 2; ++l)
          mapped[(size_t)i * 4 + ii + 2 * l] =
              mg[(size_t)i * 4 + ii] * m(0, l) + mg[(size_t)i * 4 + ii + 2] * m(1, l);
    double fl[4] = {0, 0, 0, 0};
    for (int c = 0; c < 4; ++c)
      for (int i = 0; i < n; ++i) fl[c] += mapped[(size_t)i * 4 + c] * a[i];
    Mat2 F;
    for (int c = 0; c < 4; ++c) F.a[c] = fbar.a[c] + fl[c];
    const PlasticityParams& mat = prob.material_at(model.ids[p]);
    const LargeResult res = large_strain_update(mat, s0[p], F, &s1[p]);
    const double c = model.weights[p] * det[p];
    out.p[p] = res.P;
    for (int i = 0; i < n; ++i) {
      double acc = 0;
      for (int r = 0; r < 4; ++r) acc += mapped[(size_t)i * 4 + r] * res.P.a[r];
      out.f[i] += c * acc;
    }
    double A[16];
    large_strain_tangent(mat, s0[p], F, 1e-7, A);
    for (int i = 0; i < n; ++i)
      for (int s = 0; s < 4; ++s) {
        double acc = 0;
        for (int r = 0; r < 4; ++r) acc += mapped[(size_t)i * 4 + r] * A[r + 4 * s];
        ma[(size_t)i * 4 + s] = acc;
      }
    for (int j = 0; j < n; ++j)
      for (int i = 0; i < n; ++i) {
        double acc = 0;
        for (int s = 0; s < 4; ++s) acc += ma[(size_t)i * 4 + s] * mapped[(size_t)j * 4 + s];
        out.k[(size_t)j * n + i] += c * acc;
      }
  }
  return out;
}

// rom.cpp:68-76
Mat2 rom_effective_stress(const RveProblem& prob, const RomModel& model,
                          const std::vector<double>& det, const std::vector<Mat2>& pp) {
  Mat2 pbar;
  for (size_t p = 0; p < model.ids.size(); ++p) {
    const double c = model.weights[p] * det[p];
    for (int k = 0; k < 4; ++k) pbar.a[k] += c * pp[p].a[k];
  }
  for (int k = 0; k < 4; ++k) pbar.a[k] /= prob.cell_volume;
  return pbar;
}

double norm2(const std::vector<double>& v) {
  double s = 0;
  for (double x : v) s += x * x;
  return std::sqrt(s);
}

struct StepOut {
  std::vector<double> a;
  std::vector<PlasticState> states;
  Mat2 pbar;
  int iters = 0;
  double residual = 0, initial_residual = 0;
};

// rom.cpp:122-150
StepOut rom_solve_step(const RveProblem& prob, const RomModel& model, const std::vector<Mat2>& fmi,
                       const std::vector<double>& det, const std::vector<PlasticState>& s0,
                       const Mat2& fbar, const std::vector<double>& a_init, const NewtonOpts& o) {
  StepOut out;
  out.a = a_init;
  out.states = s0;
  double tol = o.eps_abs;
  for (int it = 0; it <= o.max_iter; ++it) {
    RomAsm as = rom_assemble(prob, model, fmi, det, s0, out.states, fbar, out.a);
    out.residual = norm2(as.f);
    if (it == 0) {
      out.initial_residual = out.residual;
      tol = std::max(o.eps_rel * std::max(out.residual, o.force_ref), o.eps_abs);
    }
    if (out.residual <= tol) {
      out.iters = it;
      out.pbar = rom_effective_stress(prob, model, det, as.p);
      return out;
    }
    if (it == o.max_iter) break;
    std::vector<double> neg(as.f.size());
    for (size_t i = 0; i < neg.size(); ++i) neg[i] = -as.f[i];
    const std::vector<double> da = lu_solve(as.k, model.N, neg);
    for (int i = 0; i < model.N; ++i) out.a[i] += da[i];
  }
  throw SolveError("reduced cell Newton did not converge");
}

// rom.cpp:152-175
StepOut rom_step_adaptive(const RveProblem& prob, const RomModel& model,
                          const std::vector<Mat2>& fmi, const std::vector<double>& det,
                          const std::vector<PlasticState>& s0, const Mat2& fprev, const Mat2& fbar,
                          const std::vector<double>& a_init, const NewtonOpts& o, int max_bisect) {
  try {
    return rom_solve_step(prob, model, fmi, det, s0, fbar, a_init, o);
  } catch (const SolveError&) {
    if (max_bisect <= 0) throw;
  }
  Mat2 mid;
  for (int k = 0; k < 4; ++k) mid.a[k] = 0.5 * (fprev.a[k] + fbar.a[k]);
  StepOut half = rom_step_adaptive(prob, model, fmi, det, s0, fprev, mid, a_init, o, max_bisect - 1);
  StepOut full =
      rom_step_adaptive(prob, model, fmi, det, half.states, mid, fbar, half.a, o, max_bisect - 1);
  full.iters += half.iters;
  full.initial_residual = std::max(full.initial_residual, half.initial_residual);
  return full;
}

}  // namespace

// Eigen PartialPivLU (unblocked restatement): pivot = first row of maximal
// |a_ik|, rows swapped whole, unit-lower L, then forward/back substitution.
std::vector<double> lu_solve(std::vector<double> k, int n, std::vector<double> rhs) {
  std::vector<int> perm(n);
  for (int c = 0; c < n; ++c) {
    int piv = c;
    double best = std::abs(k[(size_t)c * n + c]);
    for (int r = c + 1; r < n; ++r)
      if (std::abs(k[(size_t)c * n + r]) > best) {
        best = std::abs(k[(size_t)c * n + r]);
        piv = r;
      }
    perm[c] = piv;
    if (piv != c)
      for (int j = 0; j < n; ++j) std::swap(k[(size_t)j * n + c], k[(size_t)j * n + piv]);
    if (best != 0.0) {
      const double d = k[(size_t)c * n + c];
      for (int r = c + 1; r < n; ++r) k[(size_t)c * n + r] /= d;
    }
    for (int j = c + 1; j < n; ++j) {
      const double u = k[(size_t)j * n + c];
      for (int r = c + 1; r < n; ++r) k[(size_t)j * n + r] -= k[(size_t)c * n + r] * u;
    }
  }
  for (int c = 0; c < n; ++c) std::swap(rhs[c], rhs[perm[c]]);
  for (int c = 0; c < n; ++c)
    for (int r = c + 1; r < n; ++r) rhs[r] -= k[(size_t)c * n + r] * rhs[c];
  for (int c = n - 1; c >= 0; --c) {
    rhs[c] /= k[(size_t)c * n + c];
    for (int r = 0; r < c; ++r) rhs[r] -= k[(size_t)c * n + r] * rhs[c];
  }
  return rhs;
}

// rom.cpp:177-200.  prev_states (nullable): the history committed at the
// start of the last increment (run_online's prev_states, pipeline.cpp:456-468).
std::vector<RomStepRecord> rom_solve(const RveProblem& prob, const RomModel& model,
                                     const std::vector<Mat2>& fmu_inv,
                                     const std::vector<double>& det,
                                     const std::vector<Mat2>& schedule, const NewtonOpts& opts,
                                     int max_bisect, std::vector<double>* a_final,
                                     std::vector<PlasticState>* prev_states) {
  std::vector<PlasticState> states(model.ids.size());
  std::vector<double> a(model.N, 0.0);
  Mat2 fprev = Mat2::identity();
  std::vector<RomStepRecord> recs;
  for (const Mat2& fbar : schedule) {
    if (prev_states) *prev_states = states;
    StepOut st = rom_step_adaptive(prob, model, fmu_inv, det, states, fprev, fbar, a, opts, max_bisect);
    fprev = fbar;
    states = st.states;
    a = st.a;
    RomStepRecord r;
    r.pbar = st.pbar;
    r.iters = st.iters;
    r.residual = st.residual;
    r.initial_residual = st.initial_residual;
    recs.push_back(r);
  }
  if (a_final) *a_final = a;
  return recs;
}

// rom.cpp:202-241: one reduced assembly at (states0, fbar, a) with the
// tangent, one PartialPivLU of K and, per unit macro perturbation e_kl, the
// condensed column  Abar(:, kl) = sum_p c A_p (e_kl + mapped_p^T q),
// q = K^-1 rhs,  rhs = -sum_p c mapped_p (A_p e_kl).  out[r + 4c] (Tensor4
// storage, r = i + 2j, c = k + 2l).
void rom_effective_stiffness(const RveProblem& prob, const RomModel& model,
                             const std::vector<Mat2>& fmi, const std::vector<double>& det,
                             const std::vector<PlasticState>& s0, const Mat2& fbar,
                             const std::vector<double>& a, double out[16]) {
  const int n = model.N, np = (int)model.ids.size();
  std::vector<PlasticState> s1(s0.size());
  const RomAsm as = rom_assemble(prob, model, fmi, det, s0, s1, fbar, a);
  // a_field: the tangent at every point (rom_assemble's a_field, rom.cpp:58-61)
  std::vector<double> af((size_t)np * 16), mapped((size_t)np * n * 4);
  for (int p = 0; p < np; ++p) {
    const double* mg = &model.mode_grads[(size_t)p * n * 4];
    const Mat2& m = fmi[p];
    double* mp = &mapped[(size_t)p * n * 4];
    for (int i = 0; i < n; ++i)
      for (int ii = 0; ii < 2; ++ii)
        for (int l = 0; l < 2; ++l)
          mp[(size_t)i * 4 + ii + 2 * l] = mg[(size_t)i * 4 + ii] * m(0, l) + mg[(size_t)i * 4 + ii + 2] * m(1, l);
    double fl[4] = {0, 0, 0, 0};
    for (int c = 0; c < 4; ++c)
      for (int i = 0; i < n; ++i) fl[c] += mp[(size_t)i * 4 + c] * a[i];
    Mat2 F;
    for (int c = 0; c < 4; ++c) F.a[c] = fbar.a[c] + fl[c];
    large_strain_tangent(prob.material_at(model.ids[p]), s0[p], F, 1e-7, &af[(size_t)p * 16]);
  }
  for (int kl = 0; kl < 4; ++kl) {  // kl = k + 2l, k outer / l inner order is immaterial
    std::vector<double> rhs(n, 0.0);
    for (int p = 0; p < np; ++p) {
      const double c = model.weights[p] * det[p];
      const double* A = &af[(size_t)p * 16];
      const double* mp = &mapped[(size_t)p * n * 4];
      for (int i = 0; i < n; ++i) {
        double acc = 0;
        for (int r = 0; r < 4; ++r) acc += mp[(size_t)i * 4 + r] * A[r + 4 * kl];
        rhs[i] -= c * acc;
      }
    }
    const std::vector<double> q = lu_solve(as.k, n, rhs);
    double col[4] = {0, 0, 0, 0};
    for (int p = 0; p < np; ++p) {
      const double c = model.weights[p] * det[p];
      const double* A = &af[(size_t)p * 16];
      const double* mp = &mapped[(size_t)p * n * 4];
      double df[4];
      for (int t = 0; t < 4; ++t) {
        double acc = 0;
        for (int i = 0; i < n; ++i) acc += mp[(size_t)i * 4 + t] * q[i];
        df[t] = (t == kl ? 1.0 : 0.0) + acc;
      }
      for (int r = 0; r < 4; ++r) {
        double acc = 0;
        for (int t = 0; t < 4; ++t) acc += A[r + 4 * t] * df[t];
        col[r] += c * acc;
      }
    }
    for (int r = 0; r < 4; ++r) out[r + 4 * kl] = col[r] / prob.cell_volume;
  }
}

// twoscale.cpp:53-96
void RomMicroEngine::respond(const Mat2& fbar, Mat2* pbar, double* abar, int* iters) {
  if (bounds.size() == 6) {
    const double comp[3] = {fbar(0, 0), fbar(1, 1), fbar(0, 1)};
    for (int k = 0; k < 3; ++k)
      if (comp[k] < bounds[2 * k] || comp[k] > bounds[2 * k + 1]) {
        ++out_of_range;
        break;
      }
  }
  NewtonOpts o = opts;
  o.force_ref = std::max(o.force_ref, force_ref);
  StepOut step = rom_step_adaptive(*prob, *model, fmi, det, states, fbar_committed, fbar, a, o, max_bisect);
  force_ref = std::max(force_ref, step.initial_residual);
  states_trial = std::move(step.states);
  a_trial = step.a;
  fbar_trial = fbar;
  *pbar = step.pbar;
  if (iters) *iters = step.iters;
  if (abar) rom_effective_stiffness(*prob, *model, fmi, det, states, fbar, a_trial, abar);
}

void RomMicroEngine::commit() {
  if (!states_trial.empty()) {
    states = states_trial;
    a = a_trial;
    fbar_committed = fbar_trial;
  }
}

}  // namespace orc
