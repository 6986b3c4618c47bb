// ORACLE — TEST INFRASTRUCTURE ONLY.
//
// CPU restatement of the hot path of the reference (POD + ECM reduced-order
// model, /root/reference/proj).  Only tests/, __graft_entry__.smoke() and the
// cpu_baseline / --impl reference legs of bench.py may load this library; the
// product path (paper_2307_16894_b200/) never links or calls it.
//
// Parity status: the reference cannot be compiled here (Eigen 3.4, GTest and
// the vendored json/CLI11 headers are absent), and it ships no
// golden vectors.  This restatement is pinned by the reference's own
// closed-form and property tests (ported in tests/test_oracle_*.py) — value
// parity against reference *outputs* is therefore unpinned.
//
// Arithmetic contract: compiled without FMA contraction (-ffp-contract=off,
// baseline x86-64 like the reference's Release build), so every expression
// below evaluates in the order written, which follows the reference's
// source order (Eigen's 2x2 products are two-term sums).
#pragma once

#include <cmath>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <array>
#include <functional>
#include <vector>

namespace orc {

// Column-major 2x2, same storage as Eigen::Matrix2d (types.hpp:13-15):
// a[0]=A00, a[1]=A10, a[2]=A01, a[3]=A11 == flatten() order (types.hpp:40-42).
struct Mat2 {
  double a[4] = {0, 0, 0, 0};
  double& operator()(int i, int j) { return a[i + 2 * j]; }
  double operator()(int i, int j) const { return a[i + 2 * j]; }
  static Mat2 identity() {
    Mat2 m;
    m.a[0] = 1;
    m.a[3] = 1;
    return m;
  }
};

// Eigen fixed 2x2 lazy product: each coefficient is a two-term sum.
inline Mat2 mul(const Mat2& x, const Mat2& y) {
  Mat2 r;
  for (int j = 0; j < 2; ++j)
    for (int i = 0; i < 2; ++i) r(i, j) = x(i, 0) * y(0, j) + x(i, 1) * y(1, j);
  return r;
}
inline Mat2 transpose(const Mat2& x) {
  Mat2 r;
  r(0, 0) = x(0, 0);
  r(1, 0) = x(0, 1);
  r(0, 1) = x(1, 0);
  r(1, 1) = x(1, 1);
  return r;
}
// Eigen determinant_impl<2>: m00*m11 - m10*m01.
inline double det(const Mat2& m) { return m(0, 0) * m(1, 1) - m(1, 0) * m(0, 1); }
// Eigen compute_inverse<2>: invdet = 1/det, cofactors times invdet.
inline Mat2 inverse(const Mat2& m) {
  const double invdet = 1.0 / det(m);
  Mat2 r;
  r(0, 0) = m(1, 1) * invdet;
  r(1, 0) = -m(1, 0) * invdet;
  r(0, 1) = -m(0, 1) * invdet;
  r(1, 1) = m(0, 0) * invdet;
  return r;
}
// Eigen squaredNorm on a 4-vector with SSE2 packets: (a0^2+a2^2)+(a1^2+a3^2).
inline double frob_norm(const Mat2& m) {
  const double s = (m.a[0] * m.a[0] + m.a[2] * m.a[2]) + (m.a[1] * m.a[1] + m.a[3] * m.a[3]);
  return std::sqrt(s);
}

struct SolveError : std::runtime_error {
  explicit SolveError(const std::string& w) : std::runtime_error(w) {}
};
struct ConfigError : std::runtime_error {
  explicit ConfigError(const std::string& w) : std::runtime_error(w) {}
};

// material.hpp:9-17
struct PlasticityParams {
  double E = 1.0, nu = 0.3, sigma_y0 = 1e300, H = 0.0;
  double lambda() const { return E * nu / ((1 + nu) * (1 - 2 * nu)); }
  double mu() const { return E / (2 * (1 + nu)); }
};

// material.hpp:55-59
struct PlasticState {
  Mat2 Fp = Mat2::identity();
  double Fp_zz = 1.0;
  double xi = 0.0;
};

// material.hpp:61-67
struct LargeResult {
  Mat2 P;
  double dgamma = 0, f_trial = 0, q_trial = 0, mises = 0;
};

struct SmallResult {
  double sigma[4] = {0, 0, 0, 0};
  double dgamma = 0, f_trial = 0, q_trial = 0, mises = 0;
};

SmallResult small_strain_update(const PlasticityParams& p, const double eps_p0[4], double xi0,
                                const double eps[4], double eps_p1[4], double* xi1);
LargeResult large_strain_update(const PlasticityParams& p, const PlasticState& s0, const Mat2& F,
                                PlasticState* s1);
// Tangent as Eigen::Matrix4d storage: out[r + 4c], r = idx(i,j), c = idx(k,l).
void large_strain_tangent(const PlasticityParams& p, const PlasticState& s0, const Mat2& F,
                          double h_rel, double out[16]);

// ---------------------------------------------------------------- mesh ----
// Structured Q4 grid of the unit square (numbering after meshgen.cpp:72-113).
struct Mesh {
  int n_nodes = 0, n_elems = 0;
  std::vector<double> nodes;  // n_nodes x 2 row-major (x, y)
  std::vector<int> elems;     // n_elems x 4 (CCW corners)
  std::vector<int> regions;   // n_elems
};
Mesh structured_q4(int n, double r0);

struct QuadCache {
  int n_per_elem = 4;
  std::vector<double> grad;  // n_qp x 4 x 2 : grad[(q*4+a)*2+j]
  std::vector<double> w;
  std::vector<int> elem_of;
  int n_qp() const { return (int)w.size(); }
};
QuadCache build_quad_cache(const Mesh& m);

struct DofMap {
  std::vector<int> node_dof;
  int n_red = 0;
  int anchor = -1;
};
DofMap periodic_dof_map(const Mesh& m, double tol = 1e-8);

struct Morph {
  std::vector<Mat2> fmu_inv;
  std::vector<double> det;
  double volume = 0, min_det = 0;
};
std::vector<double> analytic_morph_d(const Mesh& m, double a, double b, double r0);
Morph derive(const Mesh& m, const QuadCache& c, const std::vector<double>& d);

// CSR of the assembled tangent: Eigen setFromTriplets semantics.
struct Csr {
  int n = 0;
  std::vector<int> row_ptr, col;
  std::vector<double> val;
};

struct RveProblem {
  Mesh mesh;
  QuadCache cache;
  DofMap dofs;
  std::vector<PlasticityParams> materials;
  double cell_volume = 1.0;
  const PlasticityParams& material_at(int q) const {
    return materials[mesh.regions[cache.elem_of[q]]];
  }
};

// microfem.cpp:56-130.  states1 may be null; p_field (4*nqp) may be null;
// tangent=false skips K.
void assemble(const RveProblem& prob, const Morph& morph, const std::vector<PlasticState>& s0,
              std::vector<PlasticState>* s1, const Mat2& fbar, const std::vector<double>& w_red,
              bool tangent, std::vector<double>& f, Csr* K, std::vector<double>* p_field,
              std::vector<double>* a_field = nullptr);

// ------------------------------------------------------------------ rom ----
struct RomModel {
  int N = 0;
  std::vector<int> ids;             // ascending
  std::vector<double> weights;      // per point
  std::vector<double> mode_grads;   // [p][i][4]
};
struct NewtonOpts {
  double eps_rel = 1e-8, eps_abs = 1e-12;
  int max_iter = 25;
  double force_ref = 0.0;
};
struct RomStepRecord {
  Mat2 pbar;
  int iters = 0;
  double residual = 0;
  double initial_residual = 0;  // RomStepResult::initial_residual (sets the increment's tolerance)
};
// rom.cpp:177-200 with rom_solve_step_adaptive (rom.cpp:152-175).
// fmu_inv/det are the morph slice at the ECM ids.  Throws SolveError.
std::vector<RomStepRecord> rom_solve(const RveProblem& prob, const RomModel& model,
                                     const std::vector<Mat2>& fmu_inv,
                                     const std::vector<double>& det,
                                     const std::vector<Mat2>& schedule, const NewtonOpts& opts,
                                     int max_bisect, std::vector<double>* a_final,
                                     std::vector<PlasticState>* prev_states = nullptr);
// microfem.cpp:213-238 (solve_rve) with solve_step_adaptive (:190-211);
// dense LU in place of Eigen::SparseLU.  Throws SolveError.
std::vector<RomStepRecord> fe_solve(const RveProblem& prob, const Morph& mo, const std::vector<Mat2>& schedule,
                                    const NewtonOpts& o, int max_bisect, std::vector<double>* w_final,
                                    std::vector<double>* w_hist = nullptr, std::vector<double>* p_hist = nullptr);
// microfem.cpp:240-313 (effective_stiffness); out[r + 4c] Tensor4 storage.
void fe_effective_stiffness(const RveProblem& prob, const Morph& mo, const std::vector<PlasticState>& s0,
                            const Mat2& fbar, const std::vector<double>& w, double out[16]);
// Eigen PartialPivLU restated (dense, column-major k n x n); returns k^-1 rhs.
std::vector<double> lu_solve(std::vector<double> k, int n, std::vector<double> rhs);
// rom.cpp:202-241; out[r + 4c] (Tensor4 storage).  Throws SolveError.
void rom_effective_stiffness(const RveProblem& prob, const RomModel& model,
                             const std::vector<Mat2>& fmi, const std::vector<double>& det,
                             const std::vector<PlasticState>& s0, const Mat2& fbar,
                             const std::vector<double>& a, double out[16]);

// twoscale.hpp:82-118 (MacroConfig / TwoscaleResult) and run_twoscale
// (twoscale.cpp:131-242) over caller-supplied MicroEngine callbacks.
struct MacroCfg {
  int nx = 5, ny = 3;
  double width = 2.0, height = 1.0, peak = 0.2;
  int steps = 50;
  double eps_rel = 1e-8, eps_abs = 1e-12;
  int max_iter = 25;
};
struct TwoscaleResult {
  std::vector<double> load_factor, compliance, u_final;
  std::vector<int> iters;
  double residual_norm = 0;
};
std::vector<std::array<double, 2>> macro_qp_positions(int nx, int ny, double w, double h);
TwoscaleResult twoscale(const MacroCfg& cfg,
                        const std::function<void(int, const double*, double*, double*)>& respond,
                        const std::function<void()>& commit);

// twoscale.hpp:55-80 (RomMicroEngine): per-engine committed history,
// reduced coordinates, macro gradient and force_ref.
struct RomMicroEngine {
  const RveProblem* prob = nullptr;
  const RomModel* model = nullptr;
  std::vector<Mat2> fmi;
  std::vector<double> det;
  NewtonOpts opts;
  int max_bisect = 5;
  std::vector<double> bounds;  // empty or (lo, hi) x 3 for (F00, F11, F01)
  std::vector<PlasticState> states, states_trial;
  std::vector<double> a, a_trial;
  Mat2 fbar_committed = Mat2::identity(), fbar_trial = Mat2::identity();
  double force_ref = 0.0;
  int out_of_range = 0;
  void respond(const Mat2& fbar, Mat2* pbar, double* abar, int* iters);
  void commit();
};

}  // namespace orc
