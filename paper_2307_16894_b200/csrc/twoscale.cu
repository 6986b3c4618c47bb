// §8(f) item 2 — the FE² macro driver around the batched micro engines:
// run_twoscale (/root/reference/proj/src/twoscale.cpp:131-242) on the
// structured Quad8 plate of MacroConfig (twoscale.hpp:82-94).
//
// Per macro Newton iteration everything stays on the device: F at all macro
// Gauss points (k_macro_F), ONE batched RomMicroEngine respond (reduced Newton
// + effective stiffness of every point), the macro residual and its norm
// (k_macro_res, k_macro_norm) and, when Newton goes on, the tangent
// contributions (k_macro_con) summed into the dense K (k_macro_gather), each
// in the reference loop's operation order, and the macro system (a few
// thousand dofs) solved by a dense LU (cuSOLVER getrf/getrs standing in for
// Eigen::SparseLU).  The host reads back two scalars per iteration (the
// residual norm for the convergence test, the first failed engine) and the
// displacement once per load step (compliance).  The mesh pieces restate structured_quad8
// (meshgen.cpp:72-113), the Quad8 shape functions and 2x2 rule
// (mesh.cpp:24-83), build_quad_cache (mesh.cpp:412-451),
// dirichlet_dof_map (mesh.cpp:374-386), boundary_edges (mesh.cpp:118-136),
// the edge rule (mesh.cpp:85-106) and traction_force (twoscale.cpp:106-129).
#include <cusolverDn.h>

#include <algorithm>
#include <array>
#include <cmath>
#include <string>
#include <type_traits>
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

// ---- the macro assembly on the device (twoscale.cpp:150-204) ---------------
// Each kernel keeps the reference loop's operation order per output value, so
// the macro residual, its norm and the tangent contributions are the values
// the host loop computes.

// F = I + h at every macro Gauss point, h(i, j) = sum_a u(node_a, i) g_a(j)
// over the element's 8 nodes in order (constrained nodes contribute u = 0).
__global__ void k_macro_F(int nq, const int32_t* __restrict__ qdof, const double* __restrict__ grad,
                          const double* __restrict__ u, double* __restrict__ F) {
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= nq) return;
  double h[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
  for (int a = 0; a < 8; ++a) {
    const int d = qdof[8 * q + a];
    const double ua[2] = {d >= 0 ? u[d] : 0.0, d >= 0 ? u[d + 1] : 0.0};
    const double* g = grad + ((size_t)q * 8 + a) * 2;
    for (int i = 0; i < 2; ++i)
      for (int j = 0; j < 2; ++j) h[i][j] += ua[i] * g[j];
  }
  F[4 * (size_t)q + 0] = 1.0 + h[0][0];
  F[4 * (size_t)q + 1] = 0.0 + h[1][0];
  F[4 * (size_t)q + 2] = 0.0 + h[0][1];
  F[4 * (size_t)q + 3] = 1.0 + h[1][1];
}

// LinearElasticEngine (twoscale.cpp:17-20): pbar = D : (F - I), abar = D.
struct Dlin {
  double d[16];
};
__global__ void k_macro_linear(int nq, Dlin D, const double* __restrict__ F, double* __restrict__ P,
                               double* __restrict__ A) {
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= nq) return;
  const double* f = F + 4 * (size_t)q;
  const double dfl[4] = {f[0] - 1.0, f[1] - 0.0, f[2] - 0.0, f[3] - 1.0};
  for (int r = 0; r < 4; ++r) {
    double v = 0.0;
    for (int t = 0; t < 4; ++t) v += D.d[r + 4 * t] * dfl[t];
    P[4 * (size_t)q + r] = v;
  }
  for (int t = 0; t < 16; ++t) A[16 * (size_t)q + t] = D.d[t];
}

// Residual of every free node: fint summed over its (q, a) incidences in the
// host loop's order (increasing q, from 0), minus factor fext; b = -res is the
// right-hand side of the Newton solve.
__global__ void k_macro_res(int n_free, const int32_t* __restrict__ fnode_dof, const int32_t* __restrict__ nptr,
                            const int32_t* __restrict__ nitem, const double* __restrict__ grad,
                            const double* __restrict__ w, const double* __restrict__ P,
                            const double* __restrict__ fext, double factor, double* __restrict__ res,
                            double* __restrict__ b) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n_free) return;
  double f0 = 0.0, f1 = 0.0;
  for (int k = nptr[i]; k < nptr[i + 1]; ++k) {
    const int it = nitem[k], q = it >> 3;
    const double* pb = P + 4 * (size_t)q;
    const double* ga = grad + (size_t)it * 2;
    const double wq = w[q];
    f0 += wq * (pb[0] * ga[0] + pb[2] * ga[1]);
    f1 += wq * (pb[1] * ga[0] + pb[3] * ga[1]);
  }
  const int d = fnode_dof[i];
  const double r0 = f0 - factor * fext[d], r1 = f1 - factor * fext[d + 1];
  res[d] = r0;
  res[d + 1] = r1;
  b[d] = -r0;
  b[d + 1] = -r1;
}

// ||res|| (sequential sum in dof order, as the host loop) and the first failed
// engine (-1 if none): one thread.
__global__ void k_macro_norm(int n, const double* __restrict__ res, int nq, const int32_t* __restrict__ st,
                             double* __restrict__ out_rn, int* __restrict__ out_fail) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  double rn = 0.0;
  for (int i = 0; i < n; ++i) rn += res[i] * res[i];
  *out_rn = sqrt(rn);
  int f = -1;
  if (st)
    for (int q = 0; q < nq; ++q)
      if (st[q]) {
        f = q;
        break;
      }
  *out_fail = f;
}

// Tangent contributions w (g_a^T A g_b)(r, sc) of every (q, a, b) with both
// dofs free, in the host loop's (q, a, b, r, sc) order.
__global__ void k_macro_con(int n_pairs, const int32_t* __restrict__ pairs, const double* __restrict__ grad,
                            const double* __restrict__ w, const double* __restrict__ A, double* __restrict__ con) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n_pairs) return;
  const int pk = pairs[t], q = pk >> 6, a = (pk >> 3) & 7, bb = pk & 7;
  const double* ab = A + 16 * (size_t)q;
  const double* ga = grad + ((size_t)q * 8 + a) * 2;
  const double* gb = grad + ((size_t)q * 8 + bb) * 2;
  const double wq = w[q];
  for (int r = 0; r < 2; ++r)
    for (int sc = 0; sc < 2; ++sc) {
      double v = 0.0;
      for (int c = 0; c < 2; ++c)
        for (int d = 0; d < 2; ++d) v += ga[c] * ab[(r + 2 * c) + 4 * (sc + 2 * d)] * gb[d];
      con[4 * (size_t)t + 2 * r + sc] = wq * v;
    }
}

__global__ void k_macro_update(int n, double* __restrict__ u, const double* __restrict__ du) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) u[i] += du[i];
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
  double* d_con = nullptr;
  {
    cudaError_t e2 = cudaMalloc(&d_ent, sizeof(int64_t) * std::max(n_ent, 1));
    if (!e2) e2 = cudaMalloc(&d_eptr, sizeof(int32_t) * (n_ent + 1));
    if (!e2) e2 = cudaMalloc(&d_eidx, sizeof(int32_t) * std::max<int64_t>(n_con, 1));
    if (!e2) e2 = cudaMalloc(&d_con, sizeof(double) * std::max<int64_t>(n_con, 1));
    if (!e2 && n_ent) e2 = cudaMemcpy(d_ent, ent.data(), sizeof(int64_t) * n_ent, cudaMemcpyHostToDevice);
    if (!e2) e2 = cudaMemcpy(d_eptr, eptr.data(), sizeof(int32_t) * (n_ent + 1), cudaMemcpyHostToDevice);
    if (!e2 && n_con) e2 = cudaMemcpy(d_eidx, order.data(), sizeof(int32_t) * n_con, cudaMemcpyHostToDevice);
    if (e2) {
      cudaFree(d_ent);
      cudaFree(d_eptr);
      cudaFree(d_eidx);
      cudaFree(d_con);
      cleanup();
      return cuda_err(ctx, e2, "twoscale: macro gather map");
    }
  }
  auto cleanup_map = [&]() {
    cudaFree(d_ent);
    cudaFree(d_eptr);
    cudaFree(d_eidx);
    cudaFree(d_con);
  };
  // ---- device-resident macro state and the maps of the device assembly
  std::vector<int32_t> qdof((size_t)nq * 8);
  for (int q = 0; q < nq; ++q)
    for (int a = 0; a < 8; ++a) qdof[8 * (size_t)q + a] = m.node_dof[m.elems[8 * m.elem_of[q] + a]];
  std::vector<int32_t> fnode_dof, nptr(1, 0), nitem;  // free nodes: incidences (q, a) in q order
  {
    std::vector<std::vector<int32_t>> inc(m.n_nodes);
    for (int q = 0; q < nq; ++q)
      for (int a = 0; a < 8; ++a) inc[m.elems[8 * m.elem_of[q] + a]].push_back(8 * q + a);
    for (int i = 0; i < m.n_nodes; ++i) {
      if (m.node_dof[i] < 0) continue;
      fnode_dof.push_back(m.node_dof[i]);
      nitem.insert(nitem.end(), inc[i].begin(), inc[i].end());
      nptr.push_back((int32_t)nitem.size());
    }
  }
  std::vector<int32_t> pairs;  // (q, a, b) with both dofs free, host loop order
  for (int q = 0; q < nq; ++q)
    for (int a = 0; a < 8; ++a) {
      if (qdof[8 * (size_t)q + a] < 0) continue;
      for (int b = 0; b < 8; ++b)
        if (qdof[8 * (size_t)q + b] >= 0) pairs.push_back((q << 6) | (a << 3) | b);
    }
  const int n_free = (int)fnode_dof.size(), n_pairs = (int)pairs.size();
  int32_t *d_qdof = nullptr, *d_fnd = nullptr, *d_nptr = nullptr, *d_nitem = nullptr, *d_pairs = nullptr;
  double *d_grad = nullptr, *d_w = nullptr, *d_fext = nullptr, *d_u = nullptr, *d_res = nullptr,
         *d_scal = nullptr, *h_scal = nullptr;
  auto cleanup_dev = [&]() {
    for (void* p : {(void*)d_qdof, (void*)d_fnd, (void*)d_nptr, (void*)d_nitem, (void*)d_pairs, (void*)d_grad,
                    (void*)d_w, (void*)d_fext, (void*)d_u, (void*)d_res, (void*)d_scal})
      cudaFree(p);
    cudaFreeHost(h_scal);
  };
  {
    auto upl = [&](auto** d, const auto& h) -> cudaError_t {
      using T = std::remove_reference_t<decltype(h[0])>;
      cudaError_t e = cudaMalloc(d, std::max<size_t>(1, h.size()) * sizeof(T));
      if (!e && !h.empty()) e = cudaMemcpy(*d, h.data(), h.size() * sizeof(T), cudaMemcpyHostToDevice);
      return e;
    };
    cudaError_t e2 = upl(&d_qdof, qdof);
    if (!e2) e2 = upl(&d_fnd, fnode_dof);
    if (!e2) e2 = upl(&d_nptr, nptr);
    if (!e2) e2 = upl(&d_nitem, nitem);
    if (!e2) e2 = upl(&d_pairs, pairs);
    if (!e2) e2 = upl(&d_grad, m.grad);
    if (!e2) e2 = upl(&d_w, m.w);
    if (!e2) e2 = upl(&d_fext, fext);
    if (!e2) e2 = cudaMalloc(&d_u, sizeof(double) * std::max(n, 1));
    if (!e2) e2 = cudaMemset(d_u, 0, sizeof(double) * std::max(n, 1));
    if (!e2) e2 = cudaMalloc(&d_res, sizeof(double) * std::max(n, 1));
    if (!e2) e2 = cudaMalloc(&d_scal, sizeof(double) * 2);
    if (!e2) e2 = cudaMallocHost(&h_scal, sizeof(double) * 2);
    if (e2) {
      cleanup_dev();
      cleanup_map();
      cleanup();
      return cuda_err(ctx, e2, "twoscale: device macro maps");
    }
  }
  Dlin dl;
  std::copy(dlin, dlin + 16, dl.d);
  std::vector<double> u(n, 0.0), ufull(2 * (size_t)m.n_nodes);
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
  // every copy, launch and factorisation is checked (an error ends the run
  // with PODECM_ECUDA after the common cleanup)
  auto cu = [&](cudaError_t e, const char* what) {
    if (e != cudaSuccess && !rc) rc = cuda_err(ctx, e, what);
  };
  const int gq = (nq + 127) / 128;
  for (int step = 0; rc == PODECM_OK && step < steps; ++step) {
    const double factor = step < up ? (double)(step + 1) / up : (double)(steps - 1 - step) / (steps - up);
    double tol = cfg->newton.eps_abs;
    int it_done = 0;
    for (int it = 0;; ++it) {
      // F at every macro Gauss point, then MicroEngine::respond for all of them at once
      k_macro_F<<<gq, 128, 0, s>>>(nq, d_qdof, d_grad, d_u, d_F);
      cu(cudaGetLastError(), "k_macro_F launch");
      if (eng) {
        if (!rc) rc = podecm_rom_engines_respond(ctx, stream, eng, d_F, micro_opts, d_P, d_A, nullptr, d_st);
      } else {
        k_macro_linear<<<gq, 128, 0, s>>>(nq, dl, d_F, d_P, d_A);
        cu(cudaGetLastError(), "k_macro_linear launch");
      }
      if (rc) break;
      evals += nq;
      // macro residual (twoscale.cpp:171-204) and its norm; the tangent only if Newton goes on
      if (n_free > 0) {
        k_macro_res<<<(n_free + 127) / 128, 128, 0, s>>>(n_free, d_fnd, d_nptr, d_nitem, d_grad, d_w, d_P, d_fext,
                                                         factor, d_res, d_b);
        cu(cudaGetLastError(), "k_macro_res launch");
      }
      k_macro_norm<<<1, 32, 0, s>>>(n, d_res, nq, eng ? d_st : nullptr, d_scal, reinterpret_cast<int*>(d_scal + 1));
      cu(cudaGetLastError(), "k_macro_norm launch");
      cu(cudaMemcpyAsync(h_scal, d_scal, sizeof(double) * 2, cudaMemcpyDeviceToHost, s), "macro norm D2H");
      cu(cudaStreamSynchronize(s), "macro residual");
      ctx->launches += 4;
      if (rc) break;
      const int failed = *reinterpret_cast<const int*>(h_scal + 1);
      if (failed >= 0) {
        rc = set_err(ctx, PODECM_ESOLVE, "twoscale: micro engine " + std::to_string(failed) + " failed");
        break;
      }
      const double rn = h_scal[0];
      if (it == 0) tol = std::max(cfg->newton.eps_rel * rn, cfg->newton.eps_abs);
      if (rn <= tol) {
        it_done = it;
        break;
      }
      if (it >= cfg->newton.max_iter) {
        rc = set_err(ctx, PODECM_ESOLVE, "macro Newton did not converge at step " + std::to_string(step));
        break;
      }
      // dense K (column-major): the contributions of the host loop order, summed
      // per entry in that order (k_macro_gather), then K du = -res, u += du
      if (n_pairs > 0) {
        k_macro_con<<<(n_pairs + 127) / 128, 128, 0, s>>>(n_pairs, d_pairs, d_grad, d_w, d_A, d_con);
        cu(cudaGetLastError(), "k_macro_con launch");
      }
      cu(cudaMemsetAsync(d_K, 0, sizeof(double) * (size_t)n * n, s), "macro tangent clear");
      if (n_ent > 0) {  // all dofs constrained: nothing to gather
        k_macro_gather<<<(n_ent + 255) / 256, 256, 0, s>>>(n_ent, d_ent, d_eptr, d_eidx, d_con, d_K);
        cu(cudaGetLastError(), "k_macro_gather launch");
      }
      {
        KTimer kt(ctx, s, "macro_lu");
        if (!rc && (cusolverDnDgetrf(dn, n, n, d_K, n, d_work, d_piv, d_info) != CUSOLVER_STATUS_SUCCESS ||
                    cusolverDnDgetrs(dn, CUBLAS_OP_N, n, 1, d_K, n, d_piv, d_b, n, d_info) != CUSOLVER_STATUS_SUCCESS))
          rc = set_err(ctx, PODECM_ECUDA, "macro tangent: cuSOLVER getrf/getrs failed");
      }
      k_macro_update<<<(n + 255) / 256, 256, 0, s>>>(n, d_u, d_b);
      cu(cudaGetLastError(), "k_macro_update launch");
      int info = 0;
      cu(cudaMemcpyAsync(&info, d_info, sizeof(int), cudaMemcpyDeviceToHost, s), "macro info D2H");
      cu(cudaStreamSynchronize(s), "macro solve");
      ctx->launches += 3;
      if (rc) break;
      if (info != 0) {
        rc = set_err(ctx, PODECM_ESOLVE, "macro tangent factorization failed at step " + std::to_string(step));
        break;
      }
    }
    if (rc) break;
    if (eng) rc = podecm_rom_engines_commit(ctx, stream, eng);
    cu(cudaMemcpyAsync(u.data(), d_u, sizeof(double) * n, cudaMemcpyDeviceToHost, s), "macro u D2H");
    cu(cudaStreamSynchronize(s), "macro step");
    if (rc) break;
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
  cleanup_dev();
  cleanup_map();
  cleanup();
  return rc;
}

}  // extern "C"
