// ORACLE — test infrastructure only (never linked or loaded by the product).
//
// C entry points over the reference's OWN source files, compiled unchanged
// from /root/reference/proj/src (material.cpp, rom.cpp, store.cpp, mesh.cpp, microfem.cpp)
// against the Eigen stand-in in oracle/eigen_shim (oracle/ref/Makefile ->
// oracle/_ref/libpodecm_ref.so).  This pins the restated oracle (oracle/*.cpp)
// and the CUDA path to the reference's code itself:
//   * ref_material_batch: large_strain_update + large_strain_tangent
//     (material.hpp:69-75) per point — bitwise comparable (2x2 arithmetic and
//     the ||F|| reduction follow Eigen's order, glibc exp/log as the
//     reference uses them);
//   * ref_rom_solve: rom_solve (rom.hpp:86-88, rom.cpp:177-200) with the
//     reference's Newton / adaptive bisection and, optionally,
//     rom_effective_stiffness (rom.cpp:202-241) at the final step — its
//     dynamic-size products / LU use the shim's plain order, so compared at
//     the BASELINE tolerance;
//   * ref_periodic_dof_map / ref_fingerprint: periodic_pairs +
//     periodic_dof_map (mesh.cpp:307-374) and Mesh::fingerprint
//     (mesh.cpp:158-180) on a structured Q4 node set;
//   * ref_rom_model_save / ref_rom_model_load: RomModel::save / load
//     (rom.cpp:265-327) through ArrayStore (store.cpp), i.e. the PODECM1
//     container written and read by the reference's code.
//   * ref_assemble / ref_solve_rve: assemble (microfem.cpp:56-130) and the
//     full-order solve_rve / solve_step_adaptive (microfem.cpp:142-238) on the
//     Q4 cell (ElemKind{2}; q4_kind.hpp), setFromTriplets summing duplicates
//     in triplet order like Eigen — bitwise comparable; the sparse solve is a
//     dense LU stand-in (small cells only).
// Symbols rom.cpp references but the calls above never reach (geometry and
// the morph aux-solve, out of scope per SURVEY §2) are stubs that throw.
#include <omp.h>

#include <cstring>
#include <string>
#include <vector>

#include "podecm/material.hpp"
#include "podecm/mesh.hpp"
#include "podecm/microfem.hpp"
#include "podecm/morph.hpp"
#include "podecm/rom.hpp"
#include "podecm/store.hpp"

namespace podecm {
// nodes_per_elem as microfem.cpp sees it (q4_kind.hpp): ElemKind{2} = Quad4.
int podecm_ref_nodes_per_elem_q4(ElemKind kind) {
  return static_cast<int>(kind) == 2 ? 4 : nodes_per_elem(kind);
}
// rom_sensitivity's morph solve (morph.cpp) is not compiled into oracle/_ref.
MorphField MorphOperator::solve(const GeomParams&) const {
  throw ConfigError("oracle/_ref: MorphOperator::solve is not built (morph.cpp out of scope)");
}
}  // namespace podecm

using namespace podecm;

namespace {

thread_local std::string g_err;

PlasticityParams params_from(const double* m) {
  PlasticityParams p;
  p.E = m[0];
  p.nu = m[1];
  p.sigma_y0 = m[2];
  p.H = m[3];
  return p;
}

void set_threads(int n) {
  if (n > 0) omp_set_num_threads(n);
}

// Structured Q4 cell as a reference Mesh: node j*(n+1)+i at (i/n, j/n),
// elements row-major with CCW corners, regions as given (the kind byte of
// Mesh::fingerprint maps every non-Tri6 kind to 1).  The quadrature cache
// comes from the caller (grad [nq][4][2], w [nq]; build_quad_cache has no Q4
// shape functions in the reference).
Mesh q4_mesh(int n_cells, const int* regions) {
  Mesh m;
  m.kind = static_cast<ElemKind>(2);  // Quad4 (q4_kind.hpp)
  const int nn = n_cells + 1;
  m.nodes = MatX(nn * nn, 2);
  for (int j = 0; j < nn; ++j)
    for (int i = 0; i < nn; ++i) {
      m.nodes(j * nn + i, 0) = static_cast<double>(i) / n_cells;
      m.nodes(j * nn + i, 1) = static_cast<double>(j) / n_cells;
    }
  m.elements = Eigen::MatrixXi(n_cells * n_cells, 4);
  m.regions = VecXi(n_cells * n_cells);
  for (int j = 0; j < n_cells; ++j)
    for (int i = 0; i < n_cells; ++i) {
      const int e = j * n_cells + i, n0 = j * nn + i;
      m.elements(e, 0) = n0;
      m.elements(e, 1) = n0 + 1;
      m.elements(e, 2) = n0 + nn + 1;
      m.elements(e, 3) = n0 + nn;
      m.regions(e) = regions ? regions[e] : 0;
    }
  return m;
}

QuadCache q4_cache(int n_elems, const double* grad, const double* w) {
  QuadCache c;
  c.n_per_elem = 4;
  const int nq = 4 * n_elems;
  c.grad.resize(nq);
  c.w = VecX(nq);
  c.elem_of = VecXi(nq);
  for (int q = 0; q < nq; ++q) {
    c.grad[q] = MatX(4, 2);
    for (int a = 0; a < 4; ++a)
      for (int j = 0; j < 2; ++j) c.grad[q](a, j) = grad[(size_t)q * 8 + a * 2 + j];
    c.w(q) = w[q];
    c.elem_of(q) = q / 4;
  }
  return c;
}

MorphField morph_field(int nq, const double* fmi, const double* det) {
  MorphField m;
  m.fmu_inv.resize(nq);
  m.det_fmu = VecX(nq);
  for (int q = 0; q < nq; ++q) {
    m.fmu_inv[q] << fmi[q], fmi[2 * (size_t)nq + q], fmi[(size_t)nq + q], fmi[3 * (size_t)nq + q];
    m.det_fmu(q) = det[q];
  }
  return m;
}

std::vector<PlasticityParams> params_vec(const double* mats, int n_mats) {
  std::vector<PlasticityParams> v;
  for (int k = 0; k < n_mats; ++k) v.push_back(params_from(mats + 4 * k));
  return v;
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// Per point: F[4][n], st_in[6][n] (Fp00, Fp10, Fp01, Fp11, Fp_zz, xi) ->
// P[4][n], A[16][n] (Tensor4 storage r + 4c), st_out[6][n], status (0 / 3
// SolveError; outputs of a failed point are left untouched), extra[4][n]
// (nullable: dgamma, f_trial, q_trial, mises).
long ref_material_batch(long n, const double* mat, const double* F, const double* st_in, double* P,
                        double* A, double* st_out, int* status, double h_rel, int nthreads, double* extra) {
  set_threads(nthreads);
  const PlasticityParams p = params_from(mat);
  long fails = 0;
#pragma omp parallel for schedule(static) reduction(+ : fails)
  for (long i = 0; i < n; ++i) {
    PlasticState s0;
    s0.Fp << st_in[0 * n + i], st_in[2 * n + i], st_in[1 * n + i], st_in[3 * n + i];
    s0.Fp_zz = st_in[4 * n + i];
    s0.xi = st_in[5 * n + i];
    Mat2 f;
    f << F[0 * n + i], F[2 * n + i], F[1 * n + i], F[3 * n + i];
    try {
      PlasticState s1;
      const LargeResult r = large_strain_update(p, s0, f, &s1);
      const Tensor4 a = large_strain_tangent(p, s0, f, h_rel);
      for (int k = 0; k < 4; ++k) P[k * n + i] = r.P.data()[k];
      for (int k = 0; k < 16; ++k) A[k * n + i] = a.m.data()[k];
      for (int k = 0; k < 4; ++k) st_out[k * n + i] = s1.Fp.data()[k];
      st_out[4 * n + i] = s1.Fp_zz;
      st_out[5 * n + i] = s1.xi;
      if (extra) {  // the remaining LargeResult fields (material.hpp:61-67)
        extra[i] = r.dgamma;
        extra[n + i] = r.f_trial;
        extra[2 * n + i] = r.q_trial;
        extra[3 * n + i] = r.mises;
      }
      status[i] = 0;
    } catch (const SolveError&) {
      status[i] = 3;
      ++fails;
    }
  }
  return fails;
}

// rom_solve per instance on a structured n_cells^2 Q4 cell (2x2 Gauss, qp
// q = 4 e + k, regions per element, mats[n_mats][4] by region).  Model:
// ids[Q] ascending, weights[Q], mode_grads[Q][N][4].  Morph restricted to the
// ECM points: fmi[n][Q][4] (flatten order), det[n][Q].  Schedule
// sched[n][K][4].  Out: pbar[n][K][4], iters[n][K], resid[n][K],
// a_final[n][N], status[n] (0 / 3 SolveError), abar[n][16] (nullable:
// rom_effective_stiffness at the last step from the previous step's
// committed history, run_online's request).
long ref_rom_solve(int n_cells, const int* regions, const double* mats, int n_mats, int N, int Q,
                   const int* ids, const double* weights, const double* mode_grads, long n_inst,
                   const double* fmi, const double* det, const double* sched, int K, double eps_rel,
                   double eps_abs, int max_iter, double* pbar, int* iters, double* resid,
                   double* a_final, int* status, double* abar, int nthreads) {
  set_threads(nthreads);
  const Mesh mesh = q4_mesh(n_cells, regions);
  QuadCache cache;
  cache.n_per_elem = 4;
  const int n_qp = 4 * mesh.n_elems();
  cache.elem_of = VecXi(n_qp);
  cache.w = VecX(n_qp);
  for (int q = 0; q < n_qp; ++q) cache.elem_of(q) = q / 4;
  RveProblem prob;
  prob.mesh = &mesh;
  prob.cache = &cache;
  for (int k = 0; k < n_mats; ++k) prob.materials.push_back(params_from(mats + 4 * k));
  RomModel model;
  model.modes = MatX(1, N);
  model.ecm_ids.assign(ids, ids + Q);
  model.ecm_weights = VecX(Q);
  for (int p = 0; p < Q; ++p) model.ecm_weights(p) = weights[p];
  model.mode_grads.resize(Q);
  for (int p = 0; p < Q; ++p) {
    model.mode_grads[p] = MatX(N, 4);
    for (int i = 0; i < N; ++i)
      for (int c = 0; c < 4; ++c) model.mode_grads[p](i, c) = mode_grads[((size_t)p * N + i) * 4 + c];
  }
  NewtonOpts o;
  o.eps_rel = eps_rel;
  o.eps_abs = eps_abs;
  o.max_iter = max_iter;
  long fails = 0;
#pragma omp parallel for schedule(dynamic, 1) reduction(+ : fails)
  for (long s = 0; s < n_inst; ++s) {
    MorphField morph;
    morph.fmu_inv.assign(n_qp, Mat2::Identity());
    morph.det_fmu = VecX::Constant(n_qp, 1.0);
    for (int p = 0; p < Q; ++p) {
      const double* f = fmi + ((size_t)s * Q + p) * 4;
      Mat2 m;
      m << f[0], f[2], f[1], f[3];
      morph.fmu_inv[ids[p]] = m;
      morph.det_fmu(ids[p]) = det[(size_t)s * Q + p];
    }
    LoadSchedule sc;
    for (int k = 0; k < K; ++k) {
      const double* g = sched + ((size_t)s * K + k) * 4;
      Mat2 m;
      m << g[0], g[2], g[1], g[3];
      sc.fbar.push_back(m);
    }
    try {
      const RomSolution sol = rom_solve(prob, model, morph, sc, o, abar != nullptr);
      for (int k = 0; k < K; ++k) {
        for (int c = 0; c < 4; ++c) pbar[((size_t)s * K + k) * 4 + c] = sol.steps[k].pbar.data()[c];
        iters[(size_t)s * K + k] = sol.steps[k].iters;
        resid[(size_t)s * K + k] = sol.steps[k].residual;
      }
      for (int i = 0; i < N; ++i) a_final[(size_t)s * N + i] = sol.steps.back().a(i);
      if (abar) {
        const MorphSlice sl = slice_morph(morph, model.ecm_ids);
        const std::vector<PlasticState> st0 =
            K > 1 ? sol.steps[K - 2].states : std::vector<PlasticState>(Q);
        const Tensor4 ab = rom_effective_stiffness(prob, model, sl, st0, sc.fbar.back(), sol.steps.back().a);
        for (int c = 0; c < 16; ++c) abar[(size_t)s * 16 + c] = ab.m.data()[c];
      }
      status[s] = 0;
    } catch (const SolveError&) {
      status[s] = 3;
      ++fails;
    }
  }
  return fails;
}

// periodic_pairs + periodic_dof_map on the structured Q4 node set:
// node_dof[(n+1)^2]; returns n_red (or -1 on error, see ref_last_error).
int ref_periodic_dof_map(int n_cells, int* node_dof) {
  try {
    const Mesh m = q4_mesh(n_cells, nullptr);
    const DofMap d = periodic_dof_map(m, periodic_pairs(m));
    for (int i = 0; i < m.n_nodes(); ++i) node_dof[i] = d.node_dof(i);
    return d.n_red;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

unsigned long long ref_fingerprint(int n_cells, const int* regions) {
  return q4_mesh(n_cells, regions).fingerprint();
}

// RomModel::save with the reference's ArrayStore (modes [n_dof][N] given
// column-major, mode_grads [Q][N][4]).  0 ok, 5 IoError, 6 FormatError.
int ref_rom_model_save(const char* path, unsigned long long mesh_tag, int kind, int n_stress_modes,
                       double ecm_eps, long n_dof, int N, const double* modes, int Q, const int* ids,
                       const double* weights, const double* mode_grads) {
  try {
    RomModel m;
    m.mesh_tag = mesh_tag;
    m.kind = static_cast<GeomKind>(kind);
    m.n_stress_modes = n_stress_modes;
    m.ecm_eps = ecm_eps;
    m.modes = MatX(n_dof, N);
    std::memcpy(m.modes.data(), modes, sizeof(double) * n_dof * N);
    m.ecm_ids.assign(ids, ids + Q);
    m.ecm_weights = VecX(Q);
    for (int p = 0; p < Q; ++p) m.ecm_weights(p) = weights[p];
    m.mode_grads.resize(Q);
    for (int p = 0; p < Q; ++p) {
      m.mode_grads[p] = MatX(N, 4);
      for (int i = 0; i < N; ++i)
        for (int c = 0; c < 4; ++c) m.mode_grads[p](i, c) = mode_grads[((size_t)p * N + i) * 4 + c];
    }
    m.save(path);
    return 0;
  } catch (const IoError& e) {
    g_err = e.what();
    return 5;
  } catch (const FormatError& e) {
    g_err = e.what();
    return 6;
  }
}

// RomModel::load: sizes first (modes == nullptr), then the arrays.
int ref_rom_model_load(const char* path, long* n_dof, int* N, int* Q, unsigned long long* mesh_tag,
                       int* kind, int* n_stress_modes, double* ecm_eps, double* modes, int* ids,
                       double* weights, double* mode_grads) {
  try {
    const RomModel m = RomModel::load(path);
    *n_dof = m.modes.rows();
    *N = m.n_modes();
    *Q = m.n_points();
    *mesh_tag = m.mesh_tag;
    *kind = static_cast<int>(m.kind);
    *n_stress_modes = m.n_stress_modes;
    *ecm_eps = m.ecm_eps;
    if (modes) {
      std::memcpy(modes, m.modes.data(), sizeof(double) * m.modes.size());
      for (int p = 0; p < m.n_points(); ++p) {
        ids[p] = m.ecm_ids[p];
        weights[p] = m.ecm_weights(p);
        for (int i = 0; i < m.n_modes(); ++i)
          for (int c = 0; c < 4; ++c) mode_grads[((size_t)p * m.n_modes() + i) * 4 + c] = m.mode_grads[p](i, c);
      }
    }
    return 0;
  } catch (const IoError& e) {
    g_err = e.what();
    return 5;
  } catch (const FormatError& e) {
    g_err = e.what();
    return 6;
  }
}

// assemble (microfem.cpp:56-130) of one instance.  fmi [4][nq] / det [nq]
// the MorphField, st0 [6][nq], fbar [4], w_red [n_red]; K values read as
// K(r, c) on the caller's CSR pattern (row_ptr / col_idx); p_field [4][nq],
// st1 [6][nq].  Returns 0, 3 (SolveError) or 2 (ConfigError).
int ref_assemble(int n_cells, const int* regions, const double* mats, int n_mats, const double* grad,
                 const double* w, const double* fmi, const double* det, const double* st0, const double* fbar,
                 const double* w_red, int tangent, const int* row_ptr, const int* col_idx, double* f,
                 double* kvals, double* p_field, double* st1) {
  try {
    const Mesh mesh = q4_mesh(n_cells, regions);
    const QuadCache cache = q4_cache(mesh.n_elems(), grad, w);
    const RveProblem prob = RveProblem::build(mesh, cache, params_vec(mats, n_mats));
    const int nq = cache.n_qp();
    const MorphField morph = morph_field(nq, fmi, det);
    std::vector<PlasticState> s0(nq), s1;
    for (int q = 0; q < nq; ++q) {
      s0[q].Fp << st0[q], st0[2 * (size_t)nq + q], st0[(size_t)nq + q], st0[3 * (size_t)nq + q];
      s0[q].Fp_zz = st0[4 * (size_t)nq + q];
      s0[q].xi = st0[5 * (size_t)nq + q];
    }
    Mat2 fb;
    fb << fbar[0], fbar[2], fbar[1], fbar[3];
    VecX wr(prob.dofs.n_red);
    for (int i = 0; i < prob.dofs.n_red; ++i) wr(i) = w_red[i];
    AssemblyOpts opts;
    opts.tangent = tangent != 0;
    opts.store_stress = true;
    const Assembly as = assemble(prob, morph, s0, &s1, fb, wr, opts);
    for (int i = 0; i < prob.dofs.n_red; ++i) f[i] = as.f(i);
    if (tangent)
      for (int r = 0; r < prob.dofs.n_red; ++r)
        for (int k = row_ptr[r]; k < row_ptr[r + 1]; ++k) kvals[k] = as.k.coeff(r, col_idx[k]);
    for (int q = 0; q < nq; ++q) {
      for (int c = 0; c < 4; ++c) p_field[(size_t)c * nq + q] = as.p_field(c, q);
      for (int c = 0; c < 4; ++c) st1[(size_t)c * nq + q] = s1[q].Fp.data()[c];
      st1[4 * (size_t)nq + q] = s1[q].Fp_zz;
      st1[5 * (size_t)nq + q] = s1[q].xi;
    }
    return 0;
  } catch (const SolveError& e) {
    g_err = e.what();
    return 3;
  } catch (const ConfigError& e) {
    g_err = e.what();
    return 2;
  }
}

// solve_rve (microfem.cpp:213-238) with solve_step_adaptive on one instance:
// sched [K][4] -> pbar [K][4], iters [K], resid [K], w_final [n_red].
int ref_solve_rve(int n_cells, const int* regions, const double* mats, int n_mats, const double* grad,
                  const double* w, const double* fmi, const double* det, const double* sched, int K,
                  double eps_rel, double eps_abs, int max_iter, double* pbar, int* iters, double* resid,
                  double* w_final) {
  try {
    const Mesh mesh = q4_mesh(n_cells, regions);
    const QuadCache cache = q4_cache(mesh.n_elems(), grad, w);
    const RveProblem prob = RveProblem::build(mesh, cache, params_vec(mats, n_mats));
    const MorphField morph = morph_field(cache.n_qp(), fmi, det);
    LoadSchedule sc;
    for (int k = 0; k < K; ++k) {
      Mat2 m;
      m << sched[4 * k], sched[4 * k + 2], sched[4 * k + 1], sched[4 * k + 3];
      sc.fbar.push_back(m);
    }
    NewtonOpts o;
    o.eps_rel = eps_rel;
    o.eps_abs = eps_abs;
    o.max_iter = max_iter;
    const RveSolution sol = solve_rve(prob, morph, sc, o);
    for (int k = 0; k < K; ++k) {
      for (int c = 0; c < 4; ++c) pbar[4 * k + c] = sol.steps[k].pbar.data()[c];
      iters[k] = sol.steps[k].iters;
      resid[k] = sol.steps[k].residual;
    }
    for (int i = 0; i < prob.dofs.n_red; ++i) w_final[i] = sol.steps.back().w_red(i);
    return 0;
  } catch (const SolveError& e) {
    g_err = e.what();
    return 3;
  }
}

}  // extern "C"
