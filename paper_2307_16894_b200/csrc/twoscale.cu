// §8(f) item 2 — the FE² macro driver around the batched micro engines:
// run_twoscale (/root/reference/proj/src/twoscale.cpp:131-242) on the
// structured Quad8 plate of MacroConfig (twoscale.hpp:82-94).
//
// Per macro Newton iteration the deformation gradients of all macro Gauss
// points go to the batched RomMicroEngine in ONE respond call (GPU: reduced
// Newton + effective stiffness of every point), the macro residual and
// tangent are assembled on the host from (Pbar, Abar) in the reference's
// loop order, and the macro system (a few thousand dofs) is solved by a
// dense LU on the device (cuSOLVER getrf/getrs standing in for
// Eigen::SparseLU).  The mesh pieces restate structured_quad8
// (meshgen.cpp:72-113), the Quad8 shape functions and 2x2 rule
// (mesh.cpp:24-83), build_quad_cache (mesh.cpp:412-451),
// dirichlet_dof_map (mesh.cpp:374-386), boundary_edges (mesh.cpp:118-136),
// the edge rule (mesh.cpp:85-106) and traction_force (twoscale.cpp:106-129).
#include <cusolverDn.h>

#include <algorithm>
#include <array>
#include <cmath>
#include <string>
#include <utility>
#include <vector>

#include "common.cuh"

using namespace podecm_impl;

namespace {

constexpr int kBottomTag = 2, kTopTag = 3, kLeftTag = 4, kRightTag = 5, kOuterTag = 1;

struct Macro {
  int n_nodes = 0, n_elems = 0, n_qp = 0, n_red = 0;
  std::vector<double> nodes;                    // [n][2]
  std::vector<int> elems;                       // [e][8]
  std::vector<std::pair<int, int>> boundary;    // (node, tag), generation order
  std::vector<double> grad, w, x;               // [q][8][2], [q], [q][2]
  std::vector<int> elem_of, node_dof;
};

void shape_quad8(double x, double y, double n[8], double dn[8][2]) {
  static const double cx[8] = {-1, 1, 1, -1, 0, 1, 0, -1};
  static const double cy[8] = {-1, -1, 1, 1, -1, 0, 1, 0};
  for (int i = 0; i < 4; ++i) {
    const double xi = cx[i], eta = cy[i];
    n[i] = 0.25 * (1 + x * xi) * (1 + y * eta) * (x * xi + y * eta - 1);
    dn[i][0] = 0.25 * xi * (1 + y * eta) * (2 * x * xi + y * eta);
    dn[i][1] = 0.25 * eta * (1 + x * xi) * (2 * y * eta + x * xi);
  }
  for (int i = 4; i < 8; ++i) {
    const double xi = cx[i], eta = cy[i];
    if (xi == 0.0) {
      n[i] = 0.5 * (1 - x * x) * (1 + y * eta);
      dn[i][0] = -x * (1 + y * eta);
      dn[i][1] = 0.5 * (1 - x * x) * eta;
    } else {
      n[i] = 0.5 * (1 + x * xi) * (1 - y * y);
      dn[i][0] = 0.5 * xi * (1 - y * y);
      dn[i][1] = -y * (1 + x * xi);
    }
  }
}

int build_macro(const podecm_macro_cfg& c, Macro& m, std::string& err) {
  if (c.nx < 1 || c.ny < 1) {
    err = "structured_quad8 needs nx, ny >= 1";
    return PODECM_ECONFIG;
  }
  const int mx = 2 * c.nx + 1, my = 2 * c.ny + 1;
  std::vector<int> id((size_t)mx * my, -1);
  for (int j = 0; j < my; ++j)
    for (int i = 0; i < mx; ++i) {
      if (i % 2 == 1 && j % 2 == 1) continue;  // serendipity: no cell centres
      id[(size_t)j * mx + i] = m.n_nodes++;
      m.nodes.push_back(c.width * i / (mx - 1.0));
      m.nodes.push_back(c.height * j / (my - 1.0));
    }
  auto at = [&](int i, int j) { return id[(size_t)j * mx + i]; };
  for (int cj = 0; cj < c.ny; ++cj)
    for (int ci = 0; ci < c.nx; ++ci) {
      const int i = 2 * ci, j = 2 * cj;
      const int row[8] = {at(i, j),         at(i + 2, j),     at(i + 2, j + 2), at(i, j + 2),
                          at(i + 1, j),     at(i + 2, j + 1), at(i + 1, j + 2), at(i, j + 1)};
      m.elems.insert(m.elems.end(), row, row + 8);
      ++m.n_elems;
    }
  for (int j = 0; j < my; ++j)
    for (int i = 0; i < mx; ++i) {
      const int node = at(i, j);
      if (node < 0) continue;
      bool outer = false;
      if (j == 0) m.boundary.emplace_back(node, kBottomTag), outer = true;
      if (j == my - 1) m.boundary.emplace_back(node, kTopTag), outer = true;
      if (i == 0) m.boundary.emplace_back(node, kLeftTag), outer = true;
      if (i == mx - 1) m.boundary.emplace_back(node, kRightTag), outer = true;
      if (outer) m.boundary.emplace_back(node, kOuterTag);
    }
  // quadrature cache: 2x2 Gauss, w = 1 (mesh.cpp:74-80)
  const double g = 1.0 / std::sqrt(3.0);
  const double pts[4][2] = {{-g, -g}, {g, -g}, {g, g}, {-g, g}};
  m.n_qp = 4 * m.n_elems;
  m.grad.resize((size_t)m.n_qp * 16);
  m.w.resize(m.n_qp);
  m.x.resize((size_t)m.n_qp * 2);
  m.elem_of.resize(m.n_qp);
  for (int e = 0; e < m.n_elems; ++e)
    for (int q = 0; q < 4; ++q) {
      double n[8], dn[8][2];
      shape_quad8(pts[q][0], pts[q][1], n, dn);
      double jac[2][2] = {{0, 0}, {0, 0}}, xq[2] = {0, 0};
      for (int a = 0; a < 8; ++a) {
        const int nd = m.elems[8 * e + a];
        for (int i = 0; i < 2; ++i) {
          for (int j = 0; j < 2; ++j) jac[i][j] += m.nodes[2 * nd + i] * dn[a][j];
          xq[i] += m.nodes[2 * nd + i] * n[a];
        }
      }
      const double det = jac[0][0] * jac[1][1] - jac[1][0] * jac[0][1];
      if (!(det > 0.0)) {
        err = "element " + std::to_string(e) + " has non-positive Jacobian";
        return PODECM_ESOLVE;
      }
      const double inv[2][2] = {{jac[1][1] / det, -jac[0][1] / det}, {-jac[1][0] / det, jac[0][0] / det}};
      const int gq = 4 * e + q;
      for (int a = 0; a < 8; ++a)
        for (int j = 0; j < 2; ++j)
          m.grad[((size_t)gq * 8 + a) * 2 + j] = dn[a][0] * inv[0][j] + dn[a][1] * inv[1][j];
      m.w[gq] = 1.0 * det;
      m.x[2 * (size_t)gq] = xq[0];
      m.x[2 * (size_t)gq + 1] = xq[1];
      m.elem_of[gq] = e;
    }
  // dirichlet_dof_map: bottom edge clamped, free nodes numbered in order
  m.node_dof.assign(m.n_nodes, 0);
  for (const auto& b : m.boundary)
    if (b.second == kBottomTag) m.node_dof[b.first] = -1;
  for (int i = 0; i < m.n_nodes; ++i) {
    if (m.node_dof[i] == -1) continue;
    m.node_dof[i] = m.n_red;
    m.n_red += 2;
  }
  return PODECM_OK;
}

// traction_force (twoscale.cpp:106-129): parabolic downward traction on the
// top edges, 3-point Gauss edge rule on the quadratic edge.
std::vector<double> traction_force(const Macro& m, double width, double peak) {
  std::vector<double> f(2 * (size_t)m.n_nodes, 0.0);
  std::vector<char> top(m.n_nodes, 0);
  for (const auto& b : m.boundary)
    if (b.second == kTopTag) top[b.first] = 1;
  static const int quad_edges[4][3] = {{0, 1, 4}, {1, 2, 5}, {2, 3, 6}, {3, 0, 7}};
  const double g = std::sqrt(3.0 / 5.0);
  const double tp[3] = {-g, 0.0, g}, tw[3] = {5.0 / 9, 8.0 / 9, 5.0 / 9};
  for (int e = 0; e < m.n_elems; ++e)
    for (int s = 0; s < 4; ++s) {
      const int ed[3] = {m.elems[8 * e + quad_edges[s][0]], m.elems[8 * e + quad_edges[s][1]],
                         m.elems[8 * e + quad_edges[s][2]]};
      if (!(top[ed[0]] && top[ed[1]] && top[ed[2]])) continue;
      for (int k = 0; k < 3; ++k) {
        const double t = tp[k];
        const double n[3] = {0.5 * t * (t - 1), 0.5 * t * (t + 1), 1 - t * t};
        const double dn[3] = {t - 0.5, t + 0.5, -2 * t};
        double x[2] = {0, 0}, dx[2] = {0, 0};
        for (int i = 0; i < 3; ++i)
          for (int c = 0; c < 2; ++c) {
            x[c] += m.nodes[2 * ed[i] + c] * n[i];
            dx[c] += m.nodes[2 * ed[i] + c] * dn[i];
          }
        const double sx = 2.0 * x[0] / width - 1.0;
        const double ty = -peak * (1.0 - sx * sx);
        const double cf = tw[k] * std::sqrt(dx[0] * dx[0] + dx[1] * dx[1]) * ty;
        for (int i = 0; i < 3; ++i) f[2 * (size_t)ed[i] + 1] += cf * n[i];
      }
    }
  return f;
}

// elastic_tangent_2d (material.cpp:69-78), Tensor4 storage r + 4c
void elastic_tangent(double E, double nu, double d[16]) {
  const double la = E * nu / ((1 + nu) * (1 - 2 * nu)), mu = E / (2 * (1 + nu));
  for (int i = 0; i < 2; ++i)
    for (int j = 0; j < 2; ++j)
      for (int k = 0; k < 2; ++k)
        for (int l = 0; l < 2; ++l)
          d[(i + 2 * j) + 4 * (k + 2 * l)] =
              la * (i == j) * (k == l) + mu * ((i == k) * (j == l) + (i == l) * (j == k));
}

}  // namespace

extern "C" {

int podecm_macro_info(const podecm_macro_cfg* cfg, int64_t out[4]) {
  if (!cfg || !out) return PODECM_ECONFIG;
  Macro m;
  std::string err;
  if (int rc = build_macro(*cfg, m, err)) return rc;
  out[0] = m.n_nodes;
  out[1] = m.n_elems;
  out[2] = m.n_qp;
  out[3] = m.n_red;
  return PODECM_OK;
}

int podecm_macro_qp_positions(const podecm_macro_cfg* cfg, double* x) {
  if (!cfg || !x) return PODECM_ECONFIG;
  Macro m;
  std::string err;
  if (int rc = build_macro(*cfg, m, err)) return rc;
  std::copy(m.x.begin(), m.x.end(), x);
  return PODECM_OK;
}

}  // extern "C"

namespace {

// Dense macro tangent from its per-qp contributions: K[ent[e]] = sum of
// contrib[idx[p]], p in [ptr[e], ptr[e+1]), in the host loop's order (the
// same additions, from 0, as the column-major host assembly).
__global__ void k_macro_gather(int n_ent, const int64_t* ent, const int32_t* ptr, const int32_t* idx,
                               const double* contrib, double* K) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= n_ent) return;
  double v = 0.0;
  for (int p = ptr[e]; p < ptr[e + 1]; ++p) v += contrib[idx[p]];
  K[ent[e]] = v;
}

}  // namespace

extern "C" {

int podecm_twoscale_run(podecm_ctx* ctx, void* stream, const podecm_macro_cfg* cfg, podecm_rom_engines* eng,
                        const podecm_newton* micro_opts, double E, double nu, double* load_factor,
                        double* compliance, int32_t* iters, double* u_final, double* residual_norm,
                        int64_t* micro_evals) {
  if (!ctx || !cfg) return PODECM_ECONFIG;
  if (eng && !micro_opts) return set_err(ctx, PODECM_ECONFIG, "twoscale: micro_opts required with engines");
  Macro m;
  std::string err;
  if (int rc = build_macro(*cfg, m, err)) return set_err(ctx, rc, "twoscale: " + err);
  auto s = static_cast<cudaStream_t>(stream);
  const int nq = m.n_qp, n = m.n_red, steps = cfg->steps;
  const std::vector<double> fext_full = traction_force(m, cfg->width, cfg->peak_traction);
  std::vector<double> fext(n, 0.0);  // DofMap::reduce
  for (int i = 0; i < m.n_nodes; ++i)
    if (m.node_dof[i] >= 0) {
      fext[m.node_dof[i]] = fext_full[2 * (size_t)i];
      fext[m.node_dof[i] + 1] = fext_full[2 * (size_t)i + 1];
    }
  double dlin[16];
  elastic_tangent(E, nu, dlin);
  // device work: engine I/O and the dense LU
  double *d_F = nullptr, *d_P = nullptr, *d_A = nullptr, *d_K = nullptr, *d_b = nullptr, *d_work = nullptr;
  int *d_piv = nullptr, *d_info = nullptr;
  int32_t* d_st = nullptr;
  cusolverDnHandle_t dn = nullptr;
  int rc = PODECM_OK;
  auto cleanup = [&]() {
    for (void* p : {(void*)d_F, (void*)d_P, (void*)d_A, (void*)d_K, (void*)d_b, (void*)d_work, (void*)d_piv,
                    (void*)d_info, (void*)d_st})
      cudaFree(p);
    if (dn) cusolverDnDestroy(dn);
  };
  cudaError_t ce = cudaMalloc(&d_F, sizeof(double) * 4 * nq);
  if (!ce) ce = cudaMalloc(&d_P, sizeof(double) * 4 * nq);
  if (!ce) ce = cudaMalloc(&d_A, sizeof(double) * 16 * nq);
  if (!ce) ce = cudaMalloc(&d_K, sizeof(double) * (size_t)n * n);
  if (!ce) ce = cudaMalloc(&d_b, sizeof(double) * n);
  if (!ce) ce = cudaMalloc(&d_piv, sizeof(int) * n);
  if (!ce) ce = cudaMalloc(&d_info, sizeof(int));
  if (!ce) ce = cudaMalloc(&d_st, sizeof(int32_t) * nq);
  if (ce) {
    cleanup();
    return cuda_err(ctx, ce, "twoscale: allocation");
  }
  if (cusolverDnCreate(&dn) != CUSOLVER_STATUS_SUCCESS) {
    cleanup();
    return set_err(ctx, PODECM_ECUDA, "twoscale: cusolverDnCreate failed");
  }
  cusolverDnSetStream(dn, s);
  int lwork = 0;
  cusolverDnDgetrf_bufferSize(dn, n, n, d_K, n, &lwork);
  if (cudaMalloc(&d_work, sizeof(double) * std::max(lwork, 1))) {
    cleanup();
    return set_err(ctx, PODECM_ECUDA, "twoscale: getrf workspace");
  }
  // Macro tangent: the per-qp contributions w v of the host loop below are
  // gathered into the dense device K (k_macro_gather) instead of a dense host
  // K that is zero-filled and copied whole (12 MB) every macro iteration.
  std::vector<int64_t> tgt;
  for (int q = 0; q < nq; ++q) {
    const int e = m.elem_of[q];
    for (int a = 0; a < 8; ++a) {
      const int da = m.node_dof[m.elems[8 * e + a]];
      if (da < 0) continue;
      for (int b = 0; b < 8; ++b) {
        const int db = m.node_dof[m.elems[8 * e + b]];
        if (db < 0) continue;
        for (int r = 0; r < 2; ++r)
          for (int sc = 0; sc < 2; ++sc) tgt.push_back((int64_t)(db + sc) * n + (da + r));
      }
    }
  }
  const int64_t n_con = (int64_t)tgt.size();
  std::vector<int32_t> order(n_con);
  for (int64_t t = 0; t < n_con; ++t) order[t] = (int32_t)t;
  std::stable_sort(order.begin(), order.end(), [&](int32_t x, int32_t y) { return tgt[x] < tgt[y]; });
  std::vector<int64_t> ent;
  std::vector<int32_t> eptr;
  for (int64_t k = 0; k < n_con; ++k) {
    if (k == 0 || tgt[order[k]] != tgt[order[k - 1]]) {
      ent.push_back(tgt[order[k]]);
      eptr.push_back((int32_t)k);
    }
  }
  eptr.push_back((int32_t)n_con);
  const int n_ent = (int)ent.size();
  int64_t* d_ent = nullptr;
  int32_t *d_eptr = nullptr, *d_eidx = nullptr;
  double *d_con = nullptr, *h_con = nullptr;
  {
    cudaError_t e2 = cudaMalloc(&d_ent, sizeof(int64_t) * std::max(n_ent, 1));
    if (!e2) e2 = cudaMalloc(&d_eptr, sizeof(int32_t) * (n_ent + 1));
    if (!e2) e2 = cudaMalloc(&d_eidx, sizeof(int32_t) * std::max<int64_t>(n_con, 1));
    if (!e2) e2 = cudaMalloc(&d_con, sizeof(double) * std::max<int64_t>(n_con, 1));
    if (!e2) e2 = cudaMallocHost(&h_con, sizeof(double) * std::max<int64_t>(n_con, 1));
    if (!e2 && n_ent) e2 = cudaMemcpy(d_ent, ent.data(), sizeof(int64_t) * n_ent, cudaMemcpyHostToDevice);
    if (!e2) e2 = cudaMemcpy(d_eptr, eptr.data(), sizeof(int32_t) * (n_ent + 1), cudaMemcpyHostToDevice);
    if (!e2 && n_con) e2 = cudaMemcpy(d_eidx, order.data(), sizeof(int32_t) * n_con, cudaMemcpyHostToDevice);
    if (e2) {
      cudaFree(d_ent);
      cudaFree(d_eptr);
      cudaFree(d_eidx);
      cudaFree(d_con);
      cudaFreeHost(h_con);
      cleanup();
      return cuda_err(ctx, e2, "twoscale: macro gather map");
    }
  }
  auto cleanup_map = [&]() {
    cudaFree(d_ent);
    cudaFree(d_eptr);
    cudaFree(d_eidx);
    cudaFree(d_con);
    cudaFreeHost(h_con);
  };
  std::vector<double> u(n, 0.0), ufull(2 * (size_t)m.n_nodes), F(4 * (size_t)nq), P(4 * (size_t)nq),
      A(16 * (size_t)nq), fint(2 * (size_t)m.n_nodes), res(n);
  std::vector<int32_t> st(nq);
  int64_t evals = 0;
  const int up = steps / 2;
  auto expand = [&]() {
    std::fill(ufull.begin(), ufull.end(), 0.0);
    for (int i = 0; i < m.n_nodes; ++i)
      if (m.node_dof[i] >= 0) {
        ufull[2 * (size_t)i] = u[m.node_dof[i]];
        ufull[2 * (size_t)i + 1] = u[m.node_dof[i] + 1];
      }
  };
  for (int step = 0; rc == PODECM_OK && step < steps; ++step) {
    const double factor = step < up ? (double)(step + 1) / up : (double)(steps - 1 - step) / (steps - up);
    double tol = cfg->newton.eps_abs;
    int it_done = 0;
    for (int it = 0;; ++it) {
      expand();
      // F = I + h at every macro Gauss point, h(i, j) = sum_a u(node_a, i) g_a(j)
      for (int q = 0; q < nq; ++q) {
        const int e = m.elem_of[q];
        double h[2][2] = {{0, 0}, {0, 0}};
        for (int a = 0; a < 8; ++a) {
          const int nd = m.elems[8 * e + a];
          for (int i = 0; i < 2; ++i)
            for (int j = 0; j < 2; ++j) h[i][j] += ufull[2 * (size_t)nd + i] * m.grad[((size_t)q * 8 + a) * 2 + j];
        }
        F[4 * (size_t)q + 0] = 1.0 + h[0][0];
        F[4 * (size_t)q + 1] = 0.0 + h[1][0];
        F[4 * (size_t)q + 2] = 0.0 + h[0][1];
        F[4 * (size_t)q + 3] = 1.0 + h[1][1];
      }
      // MicroEngine::respond for every macro Gauss point at once
      if (eng) {
        cudaMemcpyAsync(d_F, F.data(), sizeof(double) * 4 * nq, cudaMemcpyHostToDevice, s);
        rc = podecm_rom_engines_respond(ctx, stream, eng, d_F, micro_opts, d_P, d_A, nullptr, d_st);
        if (rc) break;
        cudaMemcpyAsync(P.data(), d_P, sizeof(double) * 4 * nq, cudaMemcpyDeviceToHost, s);
        cudaMemcpyAsync(A.data(), d_A, sizeof(double) * 16 * nq, cudaMemcpyDeviceToHost, s);
        cudaMemcpyAsync(st.data(), d_st, sizeof(int32_t) * nq, cudaMemcpyDeviceToHost, s);
        cudaStreamSynchronize(s);
        for (int q = 0; q < nq; ++q)
          if (st[q]) {
            rc = set_err(ctx, PODECM_ESOLVE, "twoscale: micro engine " + std::to_string(q) + " failed");
            break;
          }
        if (rc) break;
      } else {  // LinearElasticEngine (twoscale.cpp:17-20): pbar = D : (F - I), abar = D
        for (int q = 0; q < nq; ++q) {
          double dfl[4] = {F[4 * (size_t)q] - 1.0, F[4 * (size_t)q + 1] - 0.0, F[4 * (size_t)q + 2] - 0.0,
                           F[4 * (size_t)q + 3] - 1.0};
          for (int r = 0; r < 4; ++r) {
            double v = 0.0;
            for (int t = 0; t < 4; ++t) v += dlin[r + 4 * t] * dfl[t];
            P[4 * (size_t)q + r] = v;
          }
          std::copy(dlin, dlin + 16, &A[16 * (size_t)q]);
        }
      }
      evals += nq;
      // macro residual (twoscale.cpp:171-204); the tangent only if Newton goes on
      std::fill(fint.begin(), fint.end(), 0.0);
      for (int q = 0; q < nq; ++q) {
        const int e = m.elem_of[q];
        const double w = m.w[q];
        const double* pb = &P[4 * (size_t)q];
        for (int a = 0; a < 8; ++a) {
          const int na = m.elems[8 * e + a];
          const double* ga = &m.grad[((size_t)q * 8 + a) * 2];
          fint[2 * (size_t)na] += w * (pb[0] * ga[0] + pb[2] * ga[1]);
          fint[2 * (size_t)na + 1] += w * (pb[1] * ga[0] + pb[3] * ga[1]);
        }
      }
      double rn = 0.0;
      for (int i = 0; i < m.n_nodes; ++i)
        if (m.node_dof[i] >= 0)
          for (int c = 0; c < 2; ++c) {
            const int d = m.node_dof[i] + c;
            res[d] = fint[2 * (size_t)i + c] - factor * fext[d];
          }
      for (int i = 0; i < n; ++i) rn += res[i] * res[i];
      rn = std::sqrt(rn);
      if (it == 0) tol = std::max(cfg->newton.eps_rel * rn, cfg->newton.eps_abs);
      if (rn <= tol) {
        it_done = it;
        break;
      }
      if (it >= cfg->newton.max_iter) {
        rc = set_err(ctx, PODECM_ESOLVE, "macro Newton did not converge at step " + std::to_string(step));
        break;
      }
      // dense K (column-major): contributions w v in the host loop order,
      // summed per entry on the device in that order
      {
        int64_t t = 0;
        for (int q = 0; q < nq; ++q) {
          const int e = m.elem_of[q];
          const double w = m.w[q];
          const double* ab = &A[16 * (size_t)q];
          for (int a = 0; a < 8; ++a) {
            const int da = m.node_dof[m.elems[8 * e + a]];
            if (da < 0) continue;
            const double* ga = &m.grad[((size_t)q * 8 + a) * 2];
            for (int b = 0; b < 8; ++b) {
              const int db = m.node_dof[m.elems[8 * e + b]];
              if (db < 0) continue;
              const double* gb = &m.grad[((size_t)q * 8 + b) * 2];
              for (int r = 0; r < 2; ++r)
                for (int sc = 0; sc < 2; ++sc) {
                  double v = 0.0;
                  for (int c = 0; c < 2; ++c)
                    for (int d = 0; d < 2; ++d) v += ga[c] * ab[(r + 2 * c) + 4 * (sc + 2 * d)] * gb[d];
                  h_con[t++] = w * v;
                }
            }
          }
        }
      }
      for (int i = 0; i < n; ++i) res[i] = -res[i];
      // every copy, launch and factorisation is checked (an error ends the
      // run with PODECM_ECUDA after the common cleanup)
      auto cu = [&](cudaError_t e, const char* what) {
        if (e != cudaSuccess && !rc) rc = cuda_err(ctx, e, what);
      };
      cu(cudaMemcpyAsync(d_con, h_con, sizeof(double) * n_con, cudaMemcpyHostToDevice, s), "macro contributions H2D");
      cu(cudaMemsetAsync(d_K, 0, sizeof(double) * (size_t)n * n, s), "macro tangent clear");
      if (n_ent > 0) {  // all dofs constrained: nothing to gather
        k_macro_gather<<<(n_ent + 255) / 256, 256, 0, s>>>(n_ent, d_ent, d_eptr, d_eidx, d_con, d_K);
        cu(cudaGetLastError(), "k_macro_gather launch");
        ctx->launches += 1;
      }
      cu(cudaMemcpyAsync(d_b, res.data(), sizeof(double) * n, cudaMemcpyHostToDevice, s), "macro residual H2D");
      if (!rc && (cusolverDnDgetrf(dn, n, n, d_K, n, d_work, d_piv, d_info) != CUSOLVER_STATUS_SUCCESS ||
                  cusolverDnDgetrs(dn, CUBLAS_OP_N, n, 1, d_K, n, d_piv, d_b, n, d_info) != CUSOLVER_STATUS_SUCCESS))
        rc = set_err(ctx, PODECM_ECUDA, "macro tangent: cuSOLVER getrf/getrs failed");
      int info = 0;
      cu(cudaMemcpyAsync(&info, d_info, sizeof(int), cudaMemcpyDeviceToHost, s), "macro info D2H");
      cu(cudaMemcpyAsync(res.data(), d_b, sizeof(double) * n, cudaMemcpyDeviceToHost, s), "macro update D2H");
      cu(cudaStreamSynchronize(s), "macro solve");
      if (rc) break;
      if (info != 0) {
        rc = set_err(ctx, PODECM_ESOLVE, "macro tangent factorization failed at step " + std::to_string(step));
        break;
      }
      for (int i = 0; i < n; ++i) u[i] += res[i];
    }
    if (rc) break;
    if (eng) rc = podecm_rom_engines_commit(ctx, stream, eng);
    expand();
    double comp = 0.0;
    for (size_t i = 0; i < ufull.size(); ++i) comp += fext_full[i] * ufull[i];
    if (load_factor) load_factor[step] = factor;
    if (compliance) compliance[step] = factor * comp;
    if (iters) iters[step] = it_done;
  }
  if (rc == PODECM_OK) {
    expand();
    if (u_final) std::copy(ufull.begin(), ufull.end(), u_final);
    double nrm = 0.0;
    for (double v : ufull) nrm += v * v;
    if (residual_norm) *residual_norm = std::sqrt(nrm);
    if (micro_evals) *micro_evals = evals;
  }
  cudaStreamSynchronize(s);
  cleanup_map();
  cleanup();
  return rc;
}

}  // extern "C"
