// ORACLE — TEST INFRASTRUCTURE ONLY (see oracle.hpp).
// Flat extern "C" surface for the checker (ctypes from tests/ and bench.py's
// cpu_baseline leg).  Layouts mirror include/podecm_cuda.h so the same host
// buffers feed both sides.  OpenMP runs over independent units (points,
// instances); per-unit results do not depend on the thread count.
#include <omp.h>

#include <cstring>
#include <memory>

#include "oracle.hpp"
#include "../paper_2307_16894_b200/csrc/pdmath.h"
#include "../paper_2307_16894_b200/csrc/gmath.h"

using namespace orc;

namespace {

PlasticityParams param_from(const double* m) {
  PlasticityParams p;
  p.E = m[0];
  p.nu = m[1];
  p.sigma_y0 = m[2];
  p.H = m[3];
  return p;
}

struct OrcRve {
  RveProblem prob;
  double r0 = 0.25;
  Csr pattern;
};

struct OrcEngines {
  RomModel model;
  std::vector<RomMicroEngine> eng;
};

void set_threads(int nt) { omp_set_num_threads(nt > 0 ? nt : omp_get_num_procs()); }

}  // namespace

extern "C" {

// SoA over n points: F[4][n] flatten order, st[6][n] = Fp00,Fp10,Fp01,Fp11,
// Fp_zz,xi; P[4][n]; A[16][n] plane r+4c; extra[4][n] = dgamma, f_trial,
// q_trial, mises (nullable).  status[i] = 0 ok / 3 SolveError.  Returns the
// number of failed points.
long orc_material_batch(long n, const double* mats, int n_mats, const int* region, const double* F,
                        const double* st_in, double* P, double* A, double* st_out, int* status,
                        double* extra, double h_rel, int nthreads) {
  set_threads(nthreads);
  std::vector<PlasticityParams> pm;
  for (int k = 0; k < n_mats; ++k) pm.push_back(param_from(mats + 4 * k));
  long fails = 0;
#pragma omp parallel for schedule(static) reduction(+ : fails)
  for (long i = 0; i < n; ++i) {
    const PlasticityParams& p = pm[region ? region[i] : 0];
    PlasticState s0;
    for (int k = 0; k < 4; ++k) s0.Fp.a[k] = st_in[k * n + i];
    s0.Fp_zz = st_in[4 * n + i];
    s0.xi = st_in[5 * n + i];
    Mat2 f;
    for (int k = 0; k < 4; ++k) f.a[k] = F[k * n + i];
    try {
      PlasticState s1;
      const LargeResult r = large_strain_update(p, s0, f, &s1);
      if (P)
        for (int k = 0; k < 4; ++k) P[k * n + i] = r.P.a[k];
      if (st_out) {
        for (int k = 0; k < 4; ++k) st_out[k * n + i] = s1.Fp.a[k];
        st_out[4 * n + i] = s1.Fp_zz;
        st_out[5 * n + i] = s1.xi;
      }
      if (extra) {
        extra[i] = r.dgamma;
        extra[n + i] = r.f_trial;
        extra[2 * n + i] = r.q_trial;
        extra[3 * n + i] = r.mises;
      }
      if (A) {
        double a[16];
        large_strain_tangent(p, s0, f, h_rel, a);
        for (int k = 0; k < 16; ++k) A[k * n + i] = a[k];
      }
      if (status) status[i] = 0;
    } catch (const SolveError&) {
      if (status) status[i] = 3;
      ++fails;
    }
  }
  return fails;
}

void* orc_rve_create(int n_cells, double r0, const double* mats, int n_mats) {
  auto* h = new OrcRve;
  h->r0 = r0;
  h->prob.mesh = structured_q4(n_cells, r0);
  h->prob.cache = build_quad_cache(h->prob.mesh);
  h->prob.dofs = periodic_dof_map(h->prob.mesh);
  for (int k = 0; k < n_mats; ++k) h->prob.materials.push_back(param_from(mats + 4 * k));
  // CSR pattern: one elastic assembly at the identity (values discarded).
  RveProblem pat = h->prob;
  for (auto& m : pat.materials) m.sigma_y0 = 1e300;
  const int nq = pat.cache.n_qp();
  Morph id;
  id.fmu_inv.assign(nq, Mat2::identity());
  id.det.assign(nq, 1.0);
  std::vector<PlasticState> s0(nq);
  std::vector<double> w(pat.dofs.n_red, 0.0), f;
  assemble(pat, id, s0, nullptr, Mat2::identity(), w, true, f, &h->pattern, nullptr);
  return h;
}

void orc_rve_destroy(void* h) { delete static_cast<OrcRve*>(h); }

// out: n_nodes, n_elems, n_qp, n_red, nnz, anchor
void orc_rve_info(void* hp, long* out) {
  auto* h = static_cast<OrcRve*>(hp);
  out[0] = h->prob.mesh.n_nodes;
  out[1] = h->prob.mesh.n_elems;
  out[2] = h->prob.cache.n_qp();
  out[3] = h->prob.dofs.n_red;
  out[4] = (long)h->pattern.col.size();
  out[5] = h->prob.dofs.anchor;
}

void orc_rve_export(void* hp, double* nodes, int* elems, int* regions, double* grad, double* w,
                    int* node_dof, int* row_ptr, int* col) {
  auto* h = static_cast<OrcRve*>(hp);
  const auto& m = h->prob.mesh;
  if (nodes) std::memcpy(nodes, m.nodes.data(), m.nodes.size() * sizeof(double));
  if (elems) std::memcpy(elems, m.elems.data(), m.elems.size() * sizeof(int));
  if (regions) std::memcpy(regions, m.regions.data(), m.regions.size() * sizeof(int));
  if (grad) std::memcpy(grad, h->prob.cache.grad.data(), h->prob.cache.grad.size() * sizeof(double));
  if (w) std::memcpy(w, h->prob.cache.w.data(), h->prob.cache.w.size() * sizeof(double));
  if (node_dof)
    std::memcpy(node_dof, h->prob.dofs.node_dof.data(), h->prob.dofs.node_dof.size() * sizeof(int));
  if (row_ptr)
    std::memcpy(row_ptr, h->pattern.row_ptr.data(), h->pattern.row_ptr.size() * sizeof(int));
  if (col) std::memcpy(col, h->pattern.col.data(), h->pattern.col.size() * sizeof(int));
}

// Morph of one instance at every qp: fmu_inv[4][nqp], det[nqp].  Returns 0 or 3.
int orc_rve_morph(void* hp, double a, double b, double* fmu_inv, double* det_out) {
  auto* h = static_cast<OrcRve*>(hp);
  try {
    const Morph mo = derive(h->prob.mesh, h->prob.cache,
                            analytic_morph_d(h->prob.mesh, a, b, h->r0));
    const int nq = h->prob.cache.n_qp();
    for (int q = 0; q < nq; ++q) {
      for (int k = 0; k < 4; ++k) fmu_inv[(size_t)k * nq + q] = mo.fmu_inv[q].a[k];
      det_out[q] = mo.det[q];
    }
    return 0;
  } catch (const SolveError&) {
    return 3;
  }
}

// Batched assemble over n_inst instances (instance-major arrays):
// geom[2] (a,b), fbar[4], w_red[n_red], st0[6][nqp], st1[6][nqp] (nullable),
// f[n_red], kvals[nnz] (nullable => no tangent), p_field[4][nqp] (nullable).
long orc_rve_assemble(void* hp, long n_inst, const double* geom, const double* fbar,
                      const double* w_red, const double* st0, double* st1, double* f, double* kvals,
                      double* p_field, int* status, int nthreads) {
  set_threads(nthreads);
  auto* h = static_cast<OrcRve*>(hp);
  const RveProblem& prob = h->prob;
  const int nq = prob.cache.n_qp(), nr = prob.dofs.n_red;
  const long nnz = (long)h->pattern.col.size();
  long fails = 0;
#pragma omp parallel for schedule(dynamic, 1) reduction(+ : fails)
  for (long s = 0; s < n_inst; ++s) {
    try {
      const Morph mo = derive(prob.mesh, prob.cache,
                              analytic_morph_d(prob.mesh, geom[2 * s], geom[2 * s + 1], h->r0));
      std::vector<PlasticState> s0(nq), s1;
      const double* sp = st0 + (size_t)s * 6 * nq;
      for (int q = 0; q < nq; ++q) {
        for (int k = 0; k < 4; ++k) s0[q].Fp.a[k] = sp[(size_t)k * nq + q];
        s0[q].Fp_zz = sp[(size_t)4 * nq + q];
        s0[q].xi = sp[(size_t)5 * nq + q];
      }
      Mat2 fb;
      for (int k = 0; k < 4; ++k) fb.a[k] = fbar[4 * s + k];
      std::vector<double> w(w_red + (size_t)s * nr, w_red + (size_t)(s + 1) * nr), ff, pf;
      Csr K;
      assemble(prob, mo, s0, st1 ? &s1 : nullptr, fb, w, kvals != nullptr, ff, kvals ? &K : nullptr,
               p_field ? &pf : nullptr);
      std::memcpy(f + (size_t)s * nr, ff.data(), nr * sizeof(double));
      if (kvals) {
        if ((long)K.val.size() != nnz) throw SolveError("pattern mismatch");
        std::memcpy(kvals + (size_t)s * nnz, K.val.data(), nnz * sizeof(double));
      }
      if (p_field)
        for (int q = 0; q < nq; ++q)
          for (int k = 0; k < 4; ++k) p_field[(size_t)s * 4 * nq + (size_t)k * nq + q] = pf[4 * (size_t)q + k];
      if (st1) {
        double* o = st1 + (size_t)s * 6 * nq;
        for (int q = 0; q < nq; ++q) {
          for (int k = 0; k < 4; ++k) o[(size_t)k * nq + q] = s1[q].Fp.a[k];
          o[(size_t)4 * nq + q] = s1[q].Fp_zz;
          o[(size_t)5 * nq + q] = s1[q].xi;
        }
      }
      if (status) status[s] = 0;
    } catch (const SolveError&) {
      if (status) status[s] = 3;
      ++fails;
    }
  }
  return fails;
}

// Batched hyper-reduced solve (rom_solve, rom.cpp:177-200) over instances.
// ids[Q] ascending, weights[Q], mode_grads[Q][N][4]; geom[n_inst][2];
// sched[n_inst][K][4] (flatten order); outputs pbar[n_inst][K][4],
// iters[n_inst][K], resid[n_inst][K], a_final[n_inst][N]; status 0/3;
// abar[n_inst][16] (nullable): rom_effective_stiffness at the last increment
// the way run_online requests it (pipeline.cpp:456-483).
// Optional extra output of orc_rom_solve: init_resid[n_inst][K], the initial
// residual of every increment (its Newton tolerance is max(eps_rel * that,
// eps_abs)); set before the call, nullptr to stop.
static double* g_rom_init_resid = nullptr;
void orc_rom_set_init_resid(double* buf) { g_rom_init_resid = buf; }

long orc_rom_solve(void* hp, int N, int Q, const int* ids, const double* weights,
                   const double* mode_grads, long n_inst, const double* geom, const double* sched,
                   int K, double eps_rel, double eps_abs, int max_iter, int max_bisect, double* pbar,
                   int* iters, double* resid, double* a_final, int* status, double* abar,
                   int nthreads) {
  set_threads(nthreads);
  auto* h = static_cast<OrcRve*>(hp);
  const RveProblem& prob = h->prob;
  RomModel model;
  model.N = N;
  model.ids.assign(ids, ids + Q);
  model.weights.assign(weights, weights + Q);
  model.mode_grads.assign(mode_grads, mode_grads + (size_t)Q * N * 4);
  NewtonOpts o;
  o.eps_rel = eps_rel;
  o.eps_abs = eps_abs;
  o.max_iter = max_iter;
  long fails = 0;
#pragma omp parallel for schedule(dynamic, 1) reduction(+ : fails)
  for (long s = 0; s < n_inst; ++s) {
    try {
      const Morph mo = derive(prob.mesh, prob.cache,
                              analytic_morph_d(prob.mesh, geom[2 * s], geom[2 * s + 1], h->r0));
      std::vector<Mat2> fmi(Q);
      std::vector<double> dt(Q);
      for (int p = 0; p < Q; ++p) {  // slice_morph (rom.cpp:111-120)
        fmi[p] = mo.fmu_inv[ids[p]];
        dt[p] = mo.det[ids[p]];
      }
      std::vector<Mat2> sc(K);
      for (int k = 0; k < K; ++k)
        for (int c = 0; c < 4; ++c) sc[k].a[c] = sched[((size_t)s * K + k) * 4 + c];
      std::vector<double> af;
      std::vector<PlasticState> prev;
      const auto recs = rom_solve(prob, model, fmi, dt, sc, o, max_bisect, &af, &prev);
      if (abar && K > 0) rom_effective_stiffness(prob, model, fmi, dt, prev, sc[K - 1], af, abar + (size_t)s * 16);
      for (int k = 0; k < K; ++k) {
        for (int c = 0; c < 4; ++c) pbar[((size_t)s * K + k) * 4 + c] = recs[k].pbar.a[c];
        if (iters) iters[(size_t)s * K + k] = recs[k].iters;
        if (resid) resid[(size_t)s * K + k] = recs[k].residual;
        if (g_rom_init_resid) g_rom_init_resid[(size_t)s * K + k] = recs[k].initial_residual;
      }
      if (a_final) std::memcpy(a_final + (size_t)s * N, af.data(), N * sizeof(double));
      if (status) status[s] = 0;
    } catch (const SolveError&) {
      if (status) status[s] = 3;
      ++fails;
    }
  }
  return fails;
}

// rom_effective_stiffness (rom.cpp:202-241) per instance: geom[n][2],
// st0[n][6][Q] planes (Fp00, Fp10, Fp01, Fp11, Fp_zz, xi), fbar[n][4],
// a[n][N] -> abar[n][16]; status 0/3.
long orc_rom_effective_stiffness(void* hp, int N, int Q, const int* ids, const double* weights,
                                 const double* mode_grads, long n_inst, const double* geom,
                                 const double* st0, const double* fbar, const double* a,
                                 double* abar, int* status, int nthreads) {
  set_threads(nthreads);
  auto* h = static_cast<OrcRve*>(hp);
  const RveProblem& prob = h->prob;
  RomModel model;
  model.N = N;
  model.ids.assign(ids, ids + Q);
  model.weights.assign(weights, weights + Q);
  model.mode_grads.assign(mode_grads, mode_grads + (size_t)Q * N * 4);
  long fails = 0;
#pragma omp parallel for schedule(dynamic, 1) reduction(+ : fails)
  for (long s = 0; s < n_inst; ++s) {
    try {
      const Morph mo = derive(prob.mesh, prob.cache,
                              analytic_morph_d(prob.mesh, geom[2 * s], geom[2 * s + 1], h->r0));
      std::vector<Mat2> fmi(Q);
      std::vector<double> dt(Q);
      std::vector<PlasticState> s0(Q);
      const double* st = st0 + (size_t)s * 6 * Q;
      for (int p = 0; p < Q; ++p) {
        fmi[p] = mo.fmu_inv[ids[p]];
        dt[p] = mo.det[ids[p]];
        for (int c = 0; c < 4; ++c) s0[p].Fp.a[c] = st[(size_t)c * Q + p];
        s0[p].Fp_zz = st[(size_t)4 * Q + p];
        s0[p].xi = st[(size_t)5 * Q + p];
      }
      Mat2 fb;
      for (int c = 0; c < 4; ++c) fb.a[c] = fbar[(size_t)s * 4 + c];
      std::vector<double> av(a + (size_t)s * N, a + (size_t)(s + 1) * N);
      rom_effective_stiffness(prob, model, fmi, dt, s0, fb, av, abar + (size_t)s * 16);
      if (status) status[s] = 0;
    } catch (const SolveError&) {
      if (status) status[s] = 3;
      ++fails;
    }
  }
  return fails;
}

// Batched RomMicroEngine (twoscale.cpp:53-96): n engines on geometries
// geom[n][2]; bounds (nullable) [3][2].
void* orc_rom_engines_create(void* hp, int N, int Q, const int* ids, const double* weights,
                             const double* mode_grads, long n, const double* geom, const double* bounds,
                             double eps_rel, double eps_abs, int max_iter, int max_bisect) {
  auto* h = static_cast<OrcRve*>(hp);
  auto* e = new OrcEngines;
  e->model.N = N;
  e->model.ids.assign(ids, ids + Q);
  e->model.weights.assign(weights, weights + Q);
  e->model.mode_grads.assign(mode_grads, mode_grads + (size_t)Q * N * 4);
  e->eng.resize(n);
  for (long s = 0; s < n; ++s) {
    RomMicroEngine& g = e->eng[s];
    g.prob = &h->prob;
    g.model = &e->model;
    const Morph mo = derive(h->prob.mesh, h->prob.cache,
                            analytic_morph_d(h->prob.mesh, geom[2 * s], geom[2 * s + 1], h->r0));
    g.fmi.resize(Q);
    g.det.resize(Q);
    for (int p = 0; p < Q; ++p) {
      g.fmi[p] = mo.fmu_inv[ids[p]];
      g.det[p] = mo.det[ids[p]];
    }
    g.opts.eps_rel = eps_rel;
    g.opts.eps_abs = eps_abs;
    g.opts.max_iter = max_iter;
    g.max_bisect = max_bisect;
    if (bounds) g.bounds.assign(bounds, bounds + 6);
    g.states.assign(Q, PlasticState());
    g.a.assign(N, 0.0);
  }
  return e;
}

void orc_rom_engines_destroy(void* eh) { delete static_cast<OrcEngines*>(eh); }

// fbar[n][4] -> pbar[n][4], abar[n][16] (nullable), iters[n], status[n] 0/3
long orc_rom_engines_respond(void* eh, const double* fbar, double* pbar, double* abar, int* iters,
                             int* status, int nthreads) {
  set_threads(nthreads);
  auto* e = static_cast<OrcEngines*>(eh);
  const long n = (long)e->eng.size();
  long fails = 0;
#pragma omp parallel for schedule(dynamic, 1) reduction(+ : fails)
  for (long s = 0; s < n; ++s) {
    try {
      Mat2 fb, pb;
      for (int c = 0; c < 4; ++c) fb.a[c] = fbar[4 * s + c];
      int it = 0;
      e->eng[s].respond(fb, &pb, abar ? abar + 16 * s : nullptr, &it);
      for (int c = 0; c < 4; ++c) pbar[4 * s + c] = pb.a[c];
      if (iters) iters[s] = it;
      status[s] = 0;
    } catch (const SolveError&) {
      status[s] = 3;
      ++fails;
    }
  }
  return fails;
}

void orc_rom_engines_commit(void* eh) {
  for (auto& g : static_cast<OrcEngines*>(eh)->eng) g.commit();
}

void orc_rom_engines_out_of_range(void* eh, int* out) {
  auto* e = static_cast<OrcEngines*>(eh);
  for (size_t s = 0; s < e->eng.size(); ++s) out[s] = e->eng[s].out_of_range;
}

// Full-order solve_rve per instance (microfem.cpp:213-238): geom[n][2],
// sched[n][K][4] -> pbar[n][K][4], iters[n][K], resid[n][K], w_final[n][n_red],
// status 0/3.
long orc_fe_solve(void* hp, long n_inst, const double* geom, const double* sched, int K, double eps_rel,
                  double eps_abs, int max_iter, int max_bisect, double* pbar, int* iters, double* resid,
                  double* w_final, int* status, double* w_hist, double* p_hist, int nthreads) {
  set_threads(nthreads);
  auto* h = static_cast<OrcRve*>(hp);
  const RveProblem& prob = h->prob;
  NewtonOpts o;
  o.eps_rel = eps_rel;
  o.eps_abs = eps_abs;
  o.max_iter = max_iter;
  const int nr = prob.dofs.n_red;
  long fails = 0;
#pragma omp parallel for schedule(dynamic, 1) reduction(+ : fails)
  for (long s = 0; s < n_inst; ++s) {
    try {
      const Morph mo = derive(prob.mesh, prob.cache,
                              analytic_morph_d(prob.mesh, geom[2 * s], geom[2 * s + 1], h->r0));
      std::vector<Mat2> sc(K);
      for (int k = 0; k < K; ++k)
        for (int c = 0; c < 4; ++c) sc[k].a[c] = sched[((size_t)s * K + k) * 4 + c];
      std::vector<double> wf, wh, ph;
      const auto recs = fe_solve(prob, mo, sc, o, max_bisect, &wf, &wh, &ph);
      const int nq = prob.cache.n_qp();
      if (w_hist) std::memcpy(w_hist + (size_t)s * K * nr, wh.data(), wh.size() * sizeof(double));
      if (p_hist)  // [s][k][4][nq] from [k][q][4]
        for (int k = 0; k < K; ++k)
          for (int q = 0; q < nq; ++q)
            for (int c = 0; c < 4; ++c)
              p_hist[(((size_t)s * K + k) * 4 + c) * nq + q] = ph[((size_t)k * nq + q) * 4 + c];
      for (int k = 0; k < K; ++k) {
        for (int c = 0; c < 4; ++c) pbar[((size_t)s * K + k) * 4 + c] = recs[k].pbar.a[c];
        if (iters) iters[(size_t)s * K + k] = recs[k].iters;
        if (resid) resid[(size_t)s * K + k] = recs[k].residual;
      }
      if (w_final) std::memcpy(w_final + (size_t)s * nr, wf.data(), nr * sizeof(double));
      if (status) status[s] = 0;
    } catch (const SolveError&) {
      if (status) status[s] = 3;
      ++fails;
    }
  }
  return fails;
}

// effective_stiffness (microfem.cpp:240-313) per instance: geom[n][2],
// st0[n][6][nqp], fbar[n][4], w[n][n_red] -> abar[n][16]; status 0/3.
long orc_fe_effective_stiffness(void* hp, long n_inst, const double* geom, const double* st0, const double* fbar,
                                const double* w, double* abar, int* status, int nthreads) {
  set_threads(nthreads);
  auto* h = static_cast<OrcRve*>(hp);
  const RveProblem& prob = h->prob;
  const int nq = prob.cache.n_qp(), nr = prob.dofs.n_red;
  long fails = 0;
#pragma omp parallel for schedule(dynamic, 1) reduction(+ : fails)
  for (long s = 0; s < n_inst; ++s) {
    try {
      const Morph mo = derive(prob.mesh, prob.cache,
                              analytic_morph_d(prob.mesh, geom[2 * s], geom[2 * s + 1], h->r0));
      std::vector<PlasticState> s0(nq);
      const double* sp = st0 + (size_t)s * 6 * nq;
      for (int q = 0; q < nq; ++q) {
        for (int k = 0; k < 4; ++k) s0[q].Fp.a[k] = sp[(size_t)k * nq + q];
        s0[q].Fp_zz = sp[(size_t)4 * nq + q];
        s0[q].xi = sp[(size_t)5 * nq + q];
      }
      Mat2 fb;
      for (int k = 0; k < 4; ++k) fb.a[k] = fbar[4 * s + k];
      std::vector<double> wv(w + (size_t)s * nr, w + (size_t)(s + 1) * nr);
      fe_effective_stiffness(prob, mo, s0, fb, wv, abar + 16 * (size_t)s);
      if (status) status[s] = 0;
    } catch (const SolveError&) {
      if (status) status[s] = 3;
      ++fails;
    }
  }
  return fails;
}

// Macro Gauss point positions (host [n_qp][2]); returns n_qp.
long orc_macro_qp_positions(int nx, int ny, double w, double h, double* x) {
  const auto p = macro_qp_positions(nx, ny, w, h);
  if (x)
    for (size_t q = 0; q < p.size(); ++q) {
      x[2 * q] = p[q][0];
      x[2 * q + 1] = p[q][1];
    }
  return (long)p.size();
}

// run_twoscale with the oracle's RomMicroEngines (eh, one per macro qp) or
// LinearElasticEngine(E, nu) when eh is null; returns 0 or 3 (SolveError).
int orc_twoscale_run(void* eh, int nx, int ny, double width, double height, double peak, int steps, double eps_rel,
                     double eps_abs, int max_iter, double E, double nu, double* load_factor, double* compliance,
                     int* iters, double* u_final, double* residual_norm) {
  MacroCfg cfg;
  cfg.nx = nx;
  cfg.ny = ny;
  cfg.width = width;
  cfg.height = height;
  cfg.peak = peak;
  cfg.steps = steps;
  cfg.eps_rel = eps_rel;
  cfg.eps_abs = eps_abs;
  cfg.max_iter = max_iter;
  auto* e = static_cast<OrcEngines*>(eh);
  PlasticityParams lp;
  lp.E = E;
  lp.nu = nu;
  const double la = lp.lambda(), mu = lp.mu();
  double d[16];
  for (int i = 0; i < 2; ++i)  // elastic_tangent_2d (material.cpp:69-78)
    for (int j = 0; j < 2; ++j)
      for (int k = 0; k < 2; ++k)
        for (int l = 0; l < 2; ++l)
          d[(i + 2 * j) + 4 * (k + 2 * l)] = la * (i == j) * (k == l) + mu * ((i == k) * (j == l) + (i == l) * (j == k));
  auto respond = [&](int q, const double* F, double* pb, double* ab) {
    if (e) {
      Mat2 fb, p;
      for (int k = 0; k < 4; ++k) fb.a[k] = F[k];
      e->eng[q].respond(fb, &p, ab, nullptr);
      for (int k = 0; k < 4; ++k) pb[k] = p.a[k];
    } else {  // LinearElasticEngine::respond (twoscale.cpp:17-20)
      const double b[4] = {F[0] - 1.0, F[1] - 0.0, F[2] - 0.0, F[3] - 1.0};
      for (int r = 0; r < 4; ++r) {
        double v = 0.0;
        for (int t = 0; t < 4; ++t) v += d[r + 4 * t] * b[t];
        pb[r] = v;
      }
      for (int k = 0; k < 16; ++k) ab[k] = d[k];
    }
  };
  auto commit = [&]() {
    if (e)
      for (auto& g : e->eng) g.commit();
  };
  try {
    const TwoscaleResult r = twoscale(cfg, respond, commit);
    for (int k = 0; k < steps; ++k) {
      if (load_factor) load_factor[k] = r.load_factor[k];
      if (compliance) compliance[k] = r.compliance[k];
      if (iters) iters[k] = r.iters[k];
    }
    if (u_final) std::copy(r.u_final.begin(), r.u_final.end(), u_final);
    if (residual_norm) *residual_norm = r.residual_norm;
    return 0;
  } catch (const SolveError&) {
    return 3;
  }
}

// Weighted stress snapshots for ECM (ecm.cpp:10-18 on the parent cell):
// W[s][q][c] = flatten(P Fmu^-T det) with P from large_strain_update at
// F = I + grad u_s (assemble's F with Fbar = I, identity morph) from a virgin
// history.  U: column-major 2 n_nodes x L.  Returns the number of failures.
long orc_stress_snapshots(void* hp, const double* U, long L, double* W, int nthreads) {
  set_threads(nthreads);
  auto* h = static_cast<OrcRve*>(hp);
  const RveProblem& prob = h->prob;
  const int nq = prob.cache.n_qp();
  const long ndof = 2L * prob.mesh.n_nodes;
  long fails = 0;
#pragma omp parallel for schedule(static) reduction(+ : fails)
  for (long t = 0; t < L * nq; ++t) {
    const long s = t / nq;
    const int q = (int)(t - s * nq);
    const int e = prob.cache.elem_of[q];
    const double* g = &prob.cache.grad[(size_t)q * 8];
    Mat2 gw;
    for (int a = 0; a < 4; ++a) {
      const int node = prob.mesh.elems[4 * e + a];
      for (int i = 0; i < 2; ++i)
        for (int j = 0; j < 2; ++j) gw(i, j) += U[s * ndof + 2 * node + i] * g[2 * a + j];
    }
    const Mat2 I = Mat2::identity();
    const Mat2 gf = mul(gw, I);
    Mat2 F;
    for (int k = 0; k < 4; ++k) F.a[k] = I.a[k] + gf.a[k];
    try {
      const LargeResult r = large_strain_update(prob.material_at(q), PlasticState{}, F, nullptr);
      Mat2 wq = mul(r.P, transpose(I));
      for (int k = 0; k < 4; ++k) W[(s * nq + q) * 4 + k] = wq.a[k] * 1.0;
    } catch (const SolveError&) {
      ++fails;
    }
  }
  return fails;
}

// libm probes: 0 glibc exp, 1 glibc log, 2 pdm exp, 3 pdm log (host build of
// the portable variant), 4 gm exp, 5 gm log (host build of the device's
// restatement of glibc, csrc/gmath.h).
void orc_libm(int which, long n, const double* x, double* out) {
  for (long i = 0; i < n; ++i) {
    switch (which) {
      case 0: out[i] = std::exp(x[i]); break;
      case 1: out[i] = std::log(x[i]); break;
      case 2: out[i] = pdm::exp(x[i]); break;
      case 3: out[i] = pdm::log(x[i]); break;
      case 4: out[i] = gm::exp(x[i]); break;
      case 5: out[i] = gm::log(x[i]); break;
      case 6: out[i] = gm::exp_fast(x[i]); break;  // the material's fast paths on their domains
      default: out[i] = gm::log_core(x[i]); break;
    }
  }
}

// Bulk bitwise sweep gm:: vs glibc over n generated arguments (OpenMP;
// splitmix64 stream per index, so the set does not depend on the thread
// count).  which: 0 exp, 1 log.  mode 0: uniform in [lo, hi]; mode 1:
// log-uniform magnitude in [lo, hi] (lo > 0); mode 2: raw random bit
// patterns.  Returns the number of results that differ in any bit (two nans
// count as equal) and the first such argument in *bad.
long orc_libm_sweep(int which, long n, unsigned long long seed, int mode, double lo, double hi,
                    double* bad) {
  long mism = 0;
  double first = 0.0;
  long first_i = -1;
#pragma omp parallel for schedule(static) reduction(+ : mism)
  for (long i = 0; i < n; ++i) {
    unsigned long long z = seed + 0x9e3779b97f4a7c15ull * (unsigned long long)(i + 1);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    z ^= z >> 31;
    double x;
    if (mode == 2) {
      std::memcpy(&x, &z, sizeof(x));
    } else {
      const double u = (double)(z >> 11) * 0x1p-53;
      x = mode == 0 ? lo + (hi - lo) * u : std::exp2(std::log2(lo) + (std::log2(hi) - std::log2(lo)) * u);
    }
    const double g = which == 0 ? std::exp(x) : std::log(x);
    const double m = which == 0 ? gm::exp(x) : gm::log(x);
    unsigned long long bg, bm;
    std::memcpy(&bg, &g, 8);
    std::memcpy(&bm, &m, 8);
    if (bg != bm && !(std::isnan(g) && std::isnan(m))) {
      ++mism;
#pragma omp critical
      if (first_i < 0 || i < first_i) {
        first_i = i;
        first = x;
      }
    }
  }
  if (bad) *bad = first;
  return mism;
}

int orc_max_threads() { return omp_get_max_threads(); }

}  // extern "C"
