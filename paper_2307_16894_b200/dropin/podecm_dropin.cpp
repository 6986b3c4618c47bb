// Reference-signature drop-in over the C-ABI (see podecm_dropin.hpp).
//
// Defines, with the reference's own declarations:
//   podecm::large_strain_update / large_strain_tangent  (material.hpp:69-75)
//   podecm::assemble                                    (microfem.hpp:74-77)
//   podecm::rom_solve                                   (rom.hpp:86-88)
// plus the batch entry points of podecm_dropin.hpp.  Every call moves its
// inputs to the device, runs the sm_100a kernels of libpodecm_cuda.so and
// copies the results back; there is no host fallback.  Checked against the
// reference's own material.cpp / microfem.cpp / rom.cpp in
// tests/test_gpu_dropin.py (oracle/_ref).
#include "podecm_dropin.hpp"

#include <cuda_runtime.h>

#include <cstdlib>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "../../include/podecm_cuda.h"

namespace podecm {
namespace {

struct Device {
  podecm_ctx* ctx = nullptr;
  ~Device() {
    if (ctx) podecm_ctx_destroy(ctx);
  }
};

podecm_ctx* ctx() {
  thread_local Device d;
  if (!d.ctx) {
    const char* e = std::getenv("PODECM_DEVICE");
    if (podecm_ctx_create(e ? std::atoi(e) : 0, &d.ctx) != PODECM_OK)
      throw std::runtime_error("podecm drop-in: no CUDA device (the device path has no host fallback)");
  }
  return d.ctx;
}

void check(int rc, const char* what) {
  if (rc == PODECM_OK) return;
  const std::string msg = std::string(what) + ": " + podecm_last_error(ctx());
  if (rc == PODECM_ECONFIG) throw ConfigError(msg);
  if (rc == PODECM_ESOLVE) throw SolveError(msg);
  throw std::runtime_error(msg);
}

void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw std::runtime_error(std::string(what) + ": " + cudaGetErrorString(e));
}

// Device buffer (RAII), filled from / copied to host vectors.
template <typename T>
struct DBuf {
  T* p = nullptr;
  size_t n = 0;
  explicit DBuf(size_t count) : n(count) {
    if (n) cuda_check(cudaMalloc(&p, n * sizeof(T)), "cudaMalloc");
  }
  DBuf(const std::vector<T>& h) : DBuf(h.size()) { put(h); }
  ~DBuf() {
    if (p) cudaFree(p);
  }
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
  void put(const std::vector<T>& h) {
    if (n) cuda_check(cudaMemcpy(p, h.data(), n * sizeof(T), cudaMemcpyHostToDevice), "H2D");
  }
  std::vector<T> get() const {
    std::vector<T> h(n);
    if (n) cuda_check(cudaMemcpy(h.data(), p, n * sizeof(T), cudaMemcpyDeviceToHost), "D2H");
    return h;
  }
};

podecm_params to_params(const PlasticityParams& p) { return {p.E, p.nu, p.sigma_y0, p.H}; }

void put_mat2(const Mat2& m, double* planes, size_t stride, size_t i) {
  planes[0 * stride + i] = m(0, 0);
  planes[1 * stride + i] = m(1, 0);
  planes[2 * stride + i] = m(0, 1);
  planes[3 * stride + i] = m(1, 1);
}

Mat2 get_mat2(const double* planes, size_t stride, size_t i) {
  Mat2 m;
  m << planes[0 * stride + i], planes[2 * stride + i], planes[1 * stride + i], planes[3 * stride + i];
  return m;
}

void put_state(const PlasticState& s, double* planes, size_t stride, size_t i) {
  put_mat2(s.Fp, planes, stride, i);
  planes[4 * stride + i] = s.Fp_zz;
  planes[5 * stride + i] = s.xi;
}

PlasticState get_state(const double* planes, size_t stride, size_t i) {
  PlasticState s;
  s.Fp = get_mat2(planes, stride, i);
  s.Fp_zz = planes[4 * stride + i];
  s.xi = planes[5 * stride + i];
  return s;
}

// The device tables of one RveProblem: the structured Q4 unit cell built by
// the C-ABI, verified bit for bit against the caller's mesh, quadrature cache
// and periodic dof map (anything else is outside the device path).
struct Cell {
  podecm_rve* rve = nullptr;
  int n_cells = 0, n_qp = 0, n_red = 0, nnz = 0;
  std::vector<int32_t> row_ptr, col_idx;
  ~Cell() {
    if (rve) podecm_rve_destroy(rve);
  }
};

std::unique_ptr<Cell> make_cell(const RveProblem& prob) {
  const Mesh& mesh = *prob.mesh;
  const QuadCache& cache = *prob.cache;
  const int ne = mesh.n_elems();
  int n = 0;
  while ((n + 1) * (n + 1) <= ne) ++n;
  if (mesh.elements.cols() != 4 || n * n != ne || mesh.n_nodes() != (n + 1) * (n + 1) || n < 2)
    throw ConfigError("podecm drop-in: the device path covers the structured Q4 unit cell");
  std::vector<int32_t> regions(ne);
  for (int e = 0; e < ne; ++e) regions[e] = mesh.regions(e);
  std::vector<podecm_params> mats;
  for (const auto& m : prob.materials) mats.push_back(to_params(m));
  auto c = std::make_unique<Cell>();
  check(podecm_rve_create_q4_regions(ctx(), n, 0.25, regions.data(), mats.data(), (int)mats.size(), &c->rve),
        "podecm_rve_create_q4_regions");
  int64_t info[6];
  podecm_rve_info(c->rve, info);
  c->n_cells = n;
  c->n_qp = (int)info[2];
  c->n_red = (int)info[3];
  c->nnz = (int)info[4];
  std::vector<double> nodes(2 * (size_t)info[0]), grad((size_t)c->n_qp * 8), w(c->n_qp);
  std::vector<int32_t> elems(4 * (size_t)ne), node_dof(info[0]);
  c->row_ptr.resize(c->n_red + 1);
  c->col_idx.resize(c->nnz);
  podecm_rve_export(c->rve, nodes.data(), elems.data(), nullptr, grad.data(), w.data(), node_dof.data(),
                    c->row_ptr.data(), c->col_idx.data(), nullptr, nullptr);
  bool same = cache.n_qp() == c->n_qp && prob.dofs.n_red == c->n_red;
  for (int i = 0; same && i < mesh.n_nodes(); ++i)
    same = mesh.nodes(i, 0) == nodes[2 * i] && mesh.nodes(i, 1) == nodes[2 * i + 1] &&
           prob.dofs.node_dof(i) == node_dof[i];
  for (int e = 0; same && e < ne; ++e)
    for (int a = 0; a < 4; ++a) same = same && mesh.elements(e, a) == elems[4 * e + a];
  for (int q = 0; same && q < c->n_qp; ++q) {
    same = cache.w(q) == w[q] && cache.elem_of(q) == q / 4;
    for (int a = 0; a < 4; ++a)
      for (int j = 0; j < 2; ++j) same = same && cache.grad[q](a, j) == grad[(size_t)q * 8 + a * 2 + j];
  }
  if (!same)
    throw ConfigError("podecm drop-in: mesh / quadrature cache / dof map differ from the structured Q4 cell");
  return c;
}

podecm_newton to_newton(const NewtonOpts& o, int max_bisect) {
  podecm_newton n;
  n.eps_rel = o.eps_rel;
  n.eps_abs = o.eps_abs;
  n.force_ref = o.force_ref;
  n.max_iter = o.max_iter;
  n.max_bisect = max_bisect;
  return n;
}

}  // namespace

// ---- material -------------------------------------------------------------

void large_strain_batch(const PlasticityParams& p, const std::vector<PlasticState>& s0,
                        const std::vector<Mat2>& F, std::vector<LargeResult>* res,
                        std::vector<PlasticState>* s1, std::vector<Tensor4>* tangent,
                        std::vector<int>* status, double h_rel) {
  const size_t n = F.size();
  if (s0.size() != n) throw ConfigError("large_strain_batch: F and s0 sizes differ");
  if (n == 0) return;
  std::vector<double> hF(4 * n), hS(6 * n);
  for (size_t i = 0; i < n; ++i) {
    put_mat2(F[i], hF.data(), n, i);
    put_state(s0[i], hS.data(), n, i);
  }
  DBuf<double> dF(hF), dS(hS), dP(4 * n), dA(tangent ? 16 * n : 0), dSo(6 * n), dX(4 * n);
  DBuf<int32_t> dst(n);
  const podecm_params m = to_params(p);
  check(podecm_material_batch_ex(ctx(), nullptr, (int64_t)n, &m, 1, nullptr, dF.p, dS.p, dP.p,
                                 tangent ? dA.p : nullptr, dSo.p, dst.p, h_rel, dX.p),
        "podecm_material_batch_ex");
  const auto P = dP.get(), So = dSo.get(), X = dX.get();
  const auto st = dst.get();
  if (res) {
    res->assign(n, LargeResult{});
    for (size_t i = 0; i < n; ++i) {
      (*res)[i].P = get_mat2(P.data(), n, i);
      (*res)[i].dgamma = X[i];
      (*res)[i].f_trial = X[n + i];
      (*res)[i].q_trial = X[2 * n + i];
      (*res)[i].mises = X[3 * n + i];
    }
  }
  if (s1) {
    s1->resize(n);
    for (size_t i = 0; i < n; ++i) (*s1)[i] = get_state(So.data(), n, i);
  }
  if (tangent) {
    const auto A = dA.get();
    tangent->assign(n, Tensor4{});
    for (size_t i = 0; i < n; ++i)
      for (int k = 0; k < 16; ++k) (*tangent)[i].m.data()[k] = A[k * n + i];
  }
  if (status) status->assign(st.begin(), st.end());
}

LargeResult large_strain_update(const PlasticityParams& p, const PlasticState& s0, const Mat2& F,
                                PlasticState* s1) {
  std::vector<LargeResult> r;
  std::vector<PlasticState> so;
  std::vector<int> st;
  large_strain_batch(p, {s0}, {F}, &r, &so, nullptr, &st);
  if (st[0] != 0)
    throw SolveError("plasticity update hit a non-positive elastic stretch (det F = " +
                     std::to_string(F.determinant()) + ")");
  if (s1) *s1 = so[0];
  return r[0];
}

Tensor4 large_strain_tangent(const PlasticityParams& p, const PlasticState& s0, const Mat2& F,
                             double h_rel) {
  std::vector<Tensor4> a;
  std::vector<int> st;
  large_strain_batch(p, {s0}, {F}, nullptr, nullptr, &a, &st, h_rel);
  if (st[0] != 0)
    throw SolveError("plasticity update hit a non-positive elastic stretch (det F = " +
                     std::to_string(F.determinant()) + ")");
  return a[0];
}

// ---- assembly -------------------------------------------------------------

Assembly assemble(const RveProblem& prob, const MorphField& morph, const std::vector<PlasticState>& states0,
                  std::vector<PlasticState>* states1, const Mat2& fbar, const VecX& w_red,
                  const AssemblyOpts& opts) {
  const auto cell = make_cell(prob);
  const size_t nq = cell->n_qp;
  if (morph.fmu_inv.size() != nq || (size_t)morph.det_fmu.size() != nq || states0.size() != nq ||
      w_red.size() != cell->n_red)
    throw ConfigError("assemble: morph / states / w_red sizes do not match the cell");
  std::vector<double> hm(5 * nq), hs(6 * nq), hf(4), hw(cell->n_red);
  for (size_t q = 0; q < nq; ++q) {
    put_mat2(morph.fmu_inv[q], hm.data(), nq, q);
    hm[4 * nq + q] = morph.det_fmu((Eigen::Index)q);
    put_state(states0[q], hs.data(), nq, q);
  }
  put_mat2(fbar, hf.data(), 1, 0);
  for (int i = 0; i < cell->n_red; ++i) hw[i] = w_red(i);
  const bool tan = opts.tangent, tf = opts.tangent && opts.store_tangent_field;
  DBuf<double> dm(hm), ds(hs), dfb(hf), dw(hw), ds1(states1 ? 6 * nq : 0), df(cell->n_red),
      dk(tan ? cell->nnz : 0), dp(opts.store_stress ? 4 * nq : 0), da(tf ? 16 * nq : 0);
  DBuf<int32_t> dst(1);
  check(podecm_assemble_batch_ex(ctx(), nullptr, cell->rve, 1, nullptr, dm.p, dfb.p, dw.p, ds.p,
                                 states1 ? ds1.p : nullptr, df.p, tan ? dk.p : nullptr,
                                 opts.store_stress ? dp.p : nullptr, dst.p, tf ? da.p : nullptr),
        "podecm_assemble_batch_ex");
  if (dst.get()[0] != 0)
    throw SolveError("plasticity update hit a non-positive elastic stretch in the cell assembly");
  Assembly out;
  const auto f = df.get();
  out.f = VecX(cell->n_red);
  for (int i = 0; i < cell->n_red; ++i) out.f(i) = f[i];
  if (tan) {
    const auto k = dk.get();
    std::vector<Triplet> trips;
    trips.reserve(cell->nnz);
    for (int r = 0; r < cell->n_red; ++r)
      for (int s = cell->row_ptr[r]; s < cell->row_ptr[r + 1]; ++s) trips.emplace_back(r, cell->col_idx[s], k[s]);
    out.k.resize(cell->n_red, cell->n_red);
    out.k.setFromTriplets(trips.begin(), trips.end());
  }
  if (opts.store_stress) {
    const auto p = dp.get();
    out.p_field = MatX(4, (Eigen::Index)nq);
    for (size_t q = 0; q < nq; ++q)
      for (int c = 0; c < 4; ++c) out.p_field(c, (Eigen::Index)q) = p[c * nq + q];
  }
  if (tf) {
    const auto a = da.get();
    out.a_field.assign(nq, Tensor4{});
    for (size_t q = 0; q < nq; ++q)
      for (int c = 0; c < 16; ++c) out.a_field[q].m.data()[c] = a[c * nq + q];
  }
  if (states1) {
    const auto s1 = ds1.get();
    states1->resize(nq);
    for (size_t q = 0; q < nq; ++q) (*states1)[q] = get_state(s1.data(), nq, q);
  }
  return out;
}

// ---- hyper-reduced online stage -----------------------------------------------

std::vector<RomSolution> rom_solve_batch(const RveProblem& prob, const RomModel& model,
                                         const std::vector<MorphField>& morphs,
                                         const std::vector<LoadSchedule>& schedules,
                                         const NewtonOpts& opts, std::vector<int>* status) {
  const size_t n = morphs.size();
  if (schedules.size() != n) throw ConfigError("rom_solve_batch: one schedule per morph");
  std::vector<RomSolution> out(n);
  if (n == 0) return out;
  const int K = (int)schedules[0].fbar.size();
  for (const auto& s : schedules)
    if ((int)s.fbar.size() != K) throw ConfigError("rom_solve_batch: schedules of different lengths");
  const auto cell = make_cell(prob);
  const int N = model.n_modes(), Q = model.n_points();
  std::vector<int32_t> ids(model.ecm_ids.begin(), model.ecm_ids.end());
  std::vector<double> w(Q), mg((size_t)Q * N * 4);
  for (int p = 0; p < Q; ++p) {
    w[p] = model.ecm_weights(p);
    for (int i = 0; i < N; ++i)
      for (int c = 0; c < 4; ++c) mg[((size_t)p * N + i) * 4 + c] = model.mode_grads[p](i, c);
  }
  podecm_rom* rom = nullptr;
  check(podecm_rom_create(ctx(), cell->rve, N, Q, ids.data(), w.data(), mg.data(), &rom), "podecm_rom_create");
  std::unique_ptr<podecm_rom, void (*)(podecm_rom*)> guard(rom, podecm_rom_destroy);
  std::vector<double> hm(n * 5 * Q), hs((size_t)n * K * 4);
  for (size_t s = 0; s < n; ++s) {
    for (int p = 0; p < Q; ++p) {  // slice_morph (rom.cpp:111-120)
      double* mo = hm.data() + s * 5 * Q;
      put_mat2(morphs[s].fmu_inv.at(ids[p]), mo, Q, p);
      mo[4 * (size_t)Q + p] = morphs[s].det_fmu(ids[p]);
    }
    for (int k = 0; k < K; ++k) put_mat2(schedules[s].fbar[k], hs.data() + (s * K + k) * 4, 1, 0);
  }
  DBuf<double> dm(hm), dsc(hs), dpb((size_t)n * K * 4), drs((size_t)n * K), daf(n * N), dah((size_t)n * K * N);
  DBuf<int32_t> dit((size_t)n * K), dst(n);
  const podecm_newton no = to_newton(opts, 5);  // rom_solve_step_adaptive default (rom.hpp:71)
  check(podecm_rom_solve_batch_morph(ctx(), nullptr, rom, (int64_t)n, dm.p, dsc.p, K, &no, dpb.p, dit.p, drs.p,
                                     daf.p, dst.p, nullptr, dah.p),
        "podecm_rom_solve_batch_morph");
  const auto pb = dpb.get(), rs = drs.get(), ah = dah.get();
  const auto it = dit.get(), st = dst.get();
  for (size_t s = 0; s < n; ++s) {
    if (st[s] != 0) continue;
    out[s].steps.resize(K);
    for (int k = 0; k < K; ++k) {
      auto& rec = out[s].steps[k];
      rec.pbar = get_mat2(pb.data() + (s * K + k) * 4, 1, 0);
      rec.iters = it[s * K + k];
      rec.residual = rs[s * K + k];
      rec.a = VecX(N);
      for (int i = 0; i < N; ++i) rec.a(i) = ah[(s * K + k) * N + i];
    }
  }
  if (status) status->assign(st.begin(), st.end());
  return out;
}

RomSolution rom_solve(const RveProblem& prob, const RomModel& model, const MorphField& morph,
                      const LoadSchedule& schedule, const NewtonOpts& opts, bool record_states) {
  if (record_states)
    throw ConfigError("rom_solve: record_states (per-increment ECM-point histories) is not provided by "
                      "the device path");
  std::vector<int> st;
  auto sols = rom_solve_batch(prob, model, {morph}, {schedule}, opts, &st);
  if (st[0] != 0) throw SolveError("reduced cell Newton did not converge");
  return std::move(sols[0]);
}

}  // namespace podecm
