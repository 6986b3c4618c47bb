// ORACLE — test infrastructure only.  C entry points that drive the
// reference-signature drop-in (paper_2307_16894_b200/dropin/podecm_dropin.cpp)
// with reference types built from plain arrays, for tests/test_gpu_dropin.py:
// the drop-in is compiled against the reference's own headers
// (/root/reference/proj/include) with oracle/eigen_shim standing in for
// Eigen, and linked with the reference's mesh.cpp / store.cpp (periodic dof
// map, fingerprint) — never with its material.cpp / microfem.cpp / rom.cpp,
// whose functions the drop-in defines.  oracle/ref/Makefile ->
// oracle/_ref/libpodecm_dropin.so.
#include <cstring>
#include <vector>

#include "../../paper_2307_16894_b200/dropin/podecm_dropin.hpp"

using namespace podecm;

namespace {

PlasticityParams params_from(const double* m) {
  PlasticityParams p;
  p.E = m[0];
  p.nu = m[1];
  p.sigma_y0 = m[2];
  p.H = m[3];
  return p;
}

Mat2 mat2(const double* planes, size_t stride, size_t i) {
  Mat2 m;
  m << planes[i], planes[2 * stride + i], planes[stride + i], planes[3 * stride + i];
  return m;
}

struct Cell {
  Mesh mesh;
  QuadCache cache;
  RveProblem prob;
};

// The structured Q4 cell as a reference Mesh / QuadCache / RveProblem (what a
// reference caller with a Quad4 ElemKind would build; the quadrature cache is
// given, grad [nq][4][2], w [nq]).
void build_cell(Cell& c, int n_cells, const int* regions, const double* mats, int n_mats, const double* grad,
                const double* w) {
  Mesh& m = c.mesh;
  m.kind = static_cast<ElemKind>(2);
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
      m.regions(e) = regions[e];
    }
  const int nq = 4 * m.n_elems();
  c.cache.n_per_elem = 4;
  c.cache.grad.resize(nq);
  c.cache.w = VecX(nq);
  c.cache.elem_of = VecXi(nq);
  for (int q = 0; q < nq; ++q) {
    c.cache.grad[q] = MatX(4, 2);
    for (int a = 0; a < 4; ++a)
      for (int j = 0; j < 2; ++j) c.cache.grad[q](a, j) = grad[(size_t)q * 8 + a * 2 + j];
    c.cache.w(q) = w[q];
    c.cache.elem_of(q) = q / 4;
  }
  c.prob.mesh = &c.mesh;
  c.prob.cache = &c.cache;
  c.prob.pairing = periodic_pairs(c.mesh);  // RveProblem::build (microfem.cpp:9-23)
  c.prob.dofs = periodic_dof_map(c.mesh, c.prob.pairing);
  for (int k = 0; k < n_mats; ++k) c.prob.materials.push_back(params_from(mats + 4 * k));
}

}  // namespace

extern "C" {

// Drop-in material on n points: per_call = 1 runs the reference signatures
// (large_strain_update then large_strain_tangent per point; status 3 where
// either throws SolveError), 0 the batch entry point.
void dropin_material(long n, const double* mat, const double* F, const double* st_in, double* P, double* A,
                     double* st_out, double* extra, int* status, int per_call) {
  const PlasticityParams p = params_from(mat);
  std::vector<PlasticState> s0(n);
  std::vector<Mat2> f(n);
  for (long i = 0; i < n; ++i) {
    s0[i].Fp = mat2(st_in, n, i);
    s0[i].Fp_zz = st_in[4 * n + i];
    s0[i].xi = st_in[5 * n + i];
    f[i] = mat2(F, n, i);
  }
  std::vector<LargeResult> r(n);
  std::vector<PlasticState> s1(n);
  std::vector<Tensor4> a(n);
  std::vector<int> st(n, 0);
  if (per_call) {
    for (long i = 0; i < n; ++i) {
      try {
        r[i] = large_strain_update(p, s0[i], f[i], &s1[i]);
        a[i] = large_strain_tangent(p, s0[i], f[i]);
      } catch (const SolveError&) {
        st[i] = 3;
      }
    }
  } else {
    large_strain_batch(p, s0, f, &r, &s1, &a, &st);
  }
  for (long i = 0; i < n; ++i) {
    status[i] = st[i];
    if (st[i]) continue;
    for (int k = 0; k < 4; ++k) P[k * n + i] = r[i].P.data()[k];
    for (int k = 0; k < 16; ++k) A[k * n + i] = a[i].m.data()[k];
    for (int k = 0; k < 4; ++k) st_out[k * n + i] = s1[i].Fp.data()[k];
    st_out[4 * n + i] = s1[i].Fp_zz;
    st_out[5 * n + i] = s1[i].xi;
    extra[i] = r[i].dgamma;
    extra[n + i] = r[i].f_trial;
    extra[2 * n + i] = r[i].q_trial;
    extra[3 * n + i] = r[i].mises;
  }
}

// Drop-in assemble of one instance (ref_assemble's layouts).  Returns 0, 2
// (ConfigError) or 3 (SolveError).
int dropin_assemble(int n_cells, const int* regions, const double* mats, int n_mats, const double* grad,
                    const double* w, const double* fmi, const double* det, const double* st0, const double* fbar,
                    const double* w_red, const int* row_ptr, const int* col_idx, double* f, double* kvals,
                    double* p_field, double* st1) {
  try {
    Cell c;
    build_cell(c, n_cells, regions, mats, n_mats, grad, w);
    const int nq = c.cache.n_qp();
    MorphField morph;
    morph.fmu_inv.resize(nq);
    morph.det_fmu = VecX(nq);
    std::vector<PlasticState> s0(nq), s1;
    for (int q = 0; q < nq; ++q) {
      morph.fmu_inv[q] = mat2(fmi, nq, q);
      morph.det_fmu(q) = det[q];
      s0[q].Fp = mat2(st0, nq, q);
      s0[q].Fp_zz = st0[4 * (size_t)nq + q];
      s0[q].xi = st0[5 * (size_t)nq + q];
    }
    VecX wr(c.prob.dofs.n_red);
    for (int i = 0; i < c.prob.dofs.n_red; ++i) wr(i) = w_red[i];
    AssemblyOpts opts;
    opts.store_stress = true;
    const Assembly as = assemble(c.prob, morph, s0, &s1, mat2(fbar, 1, 0), wr, opts);
    for (int i = 0; i < c.prob.dofs.n_red; ++i) f[i] = as.f(i);
    for (int r = 0; r < c.prob.dofs.n_red; ++r)
      for (int k = row_ptr[r]; k < row_ptr[r + 1]; ++k) kvals[k] = as.k.coeff(r, col_idx[k]);
    for (int q = 0; q < nq; ++q) {
      for (int k = 0; k < 4; ++k) p_field[(size_t)k * nq + q] = as.p_field(k, q);
      for (int k = 0; k < 4; ++k) st1[(size_t)k * nq + q] = s1[q].Fp.data()[k];
      st1[4 * (size_t)nq + q] = s1[q].Fp_zz;
      st1[5 * (size_t)nq + q] = s1[q].xi;
    }
    return 0;
  } catch (const ConfigError&) {
    return 2;
  } catch (const SolveError&) {
    return 3;
  }
}

// Drop-in rom_solve (per_call = 1: one reference-signature call per instance;
// 0: rom_solve_batch).  Layouts as ref_rom_solve plus a_hist [n][K][N].
void dropin_rom_solve(int n_cells, const int* regions, const double* mats, int n_mats, const double* grad,
                      const double* w, int N, int Q, const int* ids, const double* weights,
                      const double* mode_grads, long n_inst, const double* fmi_q, const double* det_q,
                      const double* sched, int K, double eps_rel, double eps_abs, int max_iter, double* pbar,
                      int* iters, double* resid, double* a_hist, int* status, int per_call) {
  Cell c;
  build_cell(c, n_cells, regions, mats, n_mats, grad, w);
  const int nq = c.cache.n_qp();
  RomModel model;
  model.modes = MatX(1, N);
  model.ecm_ids.assign(ids, ids + Q);
  model.ecm_weights = VecX(Q);
  model.mode_grads.resize(Q);
  for (int p = 0; p < Q; ++p) {
    model.ecm_weights(p) = weights[p];
    model.mode_grads[p] = MatX(N, 4);
    for (int i = 0; i < N; ++i)
      for (int k = 0; k < 4; ++k) model.mode_grads[p](i, k) = mode_grads[((size_t)p * N + i) * 4 + k];
  }
  std::vector<MorphField> morphs(n_inst);
  std::vector<LoadSchedule> scheds(n_inst);
  for (long s = 0; s < n_inst; ++s) {
    morphs[s].fmu_inv.assign(nq, Mat2::Identity());
    morphs[s].det_fmu = VecX::Constant(nq, 1.0);
    for (int p = 0; p < Q; ++p) {
      const double* f = fmi_q + ((size_t)s * Q + p) * 4;
      morphs[s].fmu_inv[ids[p]] << f[0], f[2], f[1], f[3];
      morphs[s].det_fmu(ids[p]) = det_q[(size_t)s * Q + p];
    }
    for (int k = 0; k < K; ++k) scheds[s].fbar.push_back(mat2(sched + ((size_t)s * K + k) * 4, 1, 0));
  }
  NewtonOpts o;
  o.eps_rel = eps_rel;
  o.eps_abs = eps_abs;
  o.max_iter = max_iter;
  std::vector<RomSolution> sols(n_inst);
  std::vector<int> st(n_inst, 0);
  if (per_call) {
    for (long s = 0; s < n_inst; ++s) {
      try {
        sols[s] = rom_solve(c.prob, model, morphs[s], scheds[s], o);
      } catch (const SolveError&) {
        st[s] = 3;
      }
    }
  } else {
    sols = rom_solve_batch(c.prob, model, morphs, scheds, o, &st);
  }
  for (long s = 0; s < n_inst; ++s) {
    status[s] = st[s];
    if (st[s]) continue;
    for (int k = 0; k < K; ++k) {
      const auto& rec = sols[s].steps[k];
      for (int m = 0; m < 4; ++m) pbar[((size_t)s * K + k) * 4 + m] = rec.pbar.data()[m];
      iters[(size_t)s * K + k] = rec.iters;
      resid[(size_t)s * K + k] = rec.residual;
      for (int i = 0; i < N; ++i) a_hist[((size_t)s * K + k) * N + i] = rec.a(i);
    }
  }
}

}  // extern "C"
