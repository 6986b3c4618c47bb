// ORACLE — TEST INFRASTRUCTURE ONLY (see oracle.hpp).
// Restates /root/reference/proj/src/twoscale.cpp:98-242 (traction_force,
// run_twoscale) with structured_quad8 (meshgen.cpp:72-113), the Quad8 shape
// functions and 2x2 rule (mesh.cpp:24-83), build_quad_cache
// (mesh.cpp:412-451), dirichlet_dof_map (mesh.cpp:374-386) and
// boundary_edges (mesh.cpp:118-136).  The macro tangent is solved by the
// dense partial-pivot LU (lu_solve) in place of Eigen::SparseLU.
#include "oracle.hpp"

#include <algorithm>
#include <array>
#include <cmath>

namespace orc {

namespace {

struct Q8Mesh {
  std::vector<std::array<double, 2>> nodes;
  std::vector<std::array<int, 8>> elems;
  std::vector<std::pair<int, int>> boundary;
};

constexpr int kOuter = 1, kBottom = 2, kTop = 3, kLeft = 4, kRight = 5;

Q8Mesh structured_quad8(int nx, int ny, double w, double h) {
  if (nx < 1 || ny < 1) throw ConfigError("structured_quad8 needs nx, ny >= 1");
  Q8Mesh m;
  const int mx = 2 * nx + 1, my = 2 * ny + 1;
  std::vector<int> id(mx * my, -1);
  for (int j = 0; j < my; ++j)
    for (int i = 0; i < mx; ++i) {
      if (i % 2 == 1 && j % 2 == 1) continue;
      id[j * mx + i] = (int)m.nodes.size();
      m.nodes.push_back({w * i / (mx - 1.0), h * j / (my - 1.0)});
    }
  auto at = [&](int i, int j) { return id[j * mx + i]; };
  for (int cj = 0; cj < ny; ++cj)
    for (int ci = 0; ci < nx; ++ci) {
      const int i = 2 * ci, j = 2 * cj;
      m.elems.push_back({at(i, j), at(i + 2, j), at(i + 2, j + 2), at(i, j + 2), at(i + 1, j), at(i + 2, j + 1),
                         at(i + 1, j + 2), at(i, j + 1)});
    }
  for (int j = 0; j < my; ++j)
    for (int i = 0; i < mx; ++i) {
      const int node = at(i, j);
      if (node < 0) continue;
      bool outer = false;
      if (j == 0) m.boundary.emplace_back(node, kBottom), outer = true;
      if (j == my - 1) m.boundary.emplace_back(node, kTop), outer = true;
      if (i == 0) m.boundary.emplace_back(node, kLeft), outer = true;
      if (i == mx - 1) m.boundary.emplace_back(node, kRight), outer = true;
      if (outer) m.boundary.emplace_back(node, kOuter);
    }
  return m;
}

void shape(double x, double y, double n[8], double dn[8][2]) {  // mesh.cpp:37-61
  static const double cx[8] = {-1, 1, 1, -1, 0, 1, 0, -1};
  static const double cy[8] = {-1, -1, 1, 1, -1, 0, 1, 0};
  for (int i = 0; i < 4; ++i) {
    const double a = cx[i], b = cy[i];
    n[i] = 0.25 * (1 + x * a) * (1 + y * b) * (x * a + y * b - 1);
    dn[i][0] = 0.25 * a * (1 + y * b) * (2 * x * a + y * b);
    dn[i][1] = 0.25 * b * (1 + x * a) * (2 * y * b + x * a);
  }
  for (int i = 4; i < 8; ++i) {
    const double a = cx[i], b = cy[i];
    if (a == 0.0) {
      n[i] = 0.5 * (1 - x * x) * (1 + y * b);
      dn[i][0] = -x * (1 + y * b);
      dn[i][1] = 0.5 * (1 - x * x) * b;
    } else {
      n[i] = 0.5 * (1 + x * a) * (1 - y * y);
      dn[i][0] = 0.5 * a * (1 - y * y);
      dn[i][1] = -y * (1 + x * a);
    }
  }
}

struct Q8Cache {
  std::vector<std::array<double, 16>> grad;  // [a][2]
  std::vector<double> w;
  std::vector<std::array<double, 2>> x;
  std::vector<int> elem_of;
};

Q8Cache cache_of(const Q8Mesh& m) {
  Q8Cache c;
  const double g = 1.0 / std::sqrt(3.0);
  const double pts[4][2] = {{-g, -g}, {g, -g}, {g, g}, {-g, g}};
  for (size_t e = 0; e < m.elems.size(); ++e)
    for (int q = 0; q < 4; ++q) {
      double n[8], dn[8][2];
      shape(pts[q][0], pts[q][1], n, dn);
      Mat2 jac;
      std::array<double, 2> xq = {0, 0};
      for (int a = 0; a < 8; ++a) {
        const auto& p = m.nodes[m.elems[e][a]];
        for (int i = 0; i < 2; ++i) {
          for (int j = 0; j < 2; ++j) jac(i, j) += p[i] * dn[a][j];
          xq[i] += p[i] * n[a];
        }
      }
      const double det = jac(0, 0) * jac(1, 1) - jac(1, 0) * jac(0, 1);
      if (det <= 0.0) throw SolveError("element has non-positive Jacobian");
      const Mat2 inv = inverse(jac);
      std::array<double, 16> gr;
      for (int a = 0; a < 8; ++a)
        for (int j = 0; j < 2; ++j) gr[2 * a + j] = dn[a][0] * inv(0, j) + dn[a][1] * inv(1, j);
      c.grad.push_back(gr);
      c.w.push_back(1.0 * det);
      c.x.push_back(xq);
      c.elem_of.push_back((int)e);
    }
  return c;
}

// twoscale.cpp:106-129
std::vector<double> traction(const Q8Mesh& m, double width, double peak) {
  std::vector<double> f(2 * m.nodes.size(), 0.0);
  std::vector<char> tagged(m.nodes.size(), 0);
  for (const auto& b : m.boundary)
    if (b.second == kTop) tagged[b.first] = 1;
  static const int qe[4][3] = {{0, 1, 4}, {1, 2, 5}, {2, 3, 6}, {3, 0, 7}};
  const double g = std::sqrt(3.0 / 5.0);
  const double tp[3] = {-g, 0.0, g}, tw[3] = {5.0 / 9, 8.0 / 9, 5.0 / 9};
  for (const auto& el : m.elems)
    for (const auto& s : qe) {
      const int ed[3] = {el[s[0]], el[s[1]], el[s[2]]};
      if (!(tagged[ed[0]] && tagged[ed[1]] && tagged[ed[2]])) continue;
      for (int k = 0; k < 3; ++k) {
        const double t = tp[k];
        const double n[3] = {0.5 * t * (t - 1), 0.5 * t * (t + 1), 1 - t * t};
        const double dn[3] = {t - 0.5, t + 0.5, -2 * t};
        double x[2] = {0, 0}, dx[2] = {0, 0};
        for (int i = 0; i < 3; ++i)
          for (int c = 0; c < 2; ++c) {
            x[c] += m.nodes[ed[i]][c] * n[i];
            dx[c] += m.nodes[ed[i]][c] * dn[i];
          }
        const double s2 = 2.0 * x[0] / width - 1.0;
        const double ty = -peak * (1.0 - s2 * s2);
        const double cf = tw[k] * std::sqrt(dx[0] * dx[0] + dx[1] * dx[1]) * ty;
        for (int i = 0; i < 3; ++i) f[2 * ed[i] + 1] += cf * n[i];
      }
    }
  return f;
}

}  // namespace

std::vector<std::array<double, 2>> macro_qp_positions(int nx, int ny, double w, double h) {
  return cache_of(structured_quad8(nx, ny, w, h)).x;
}

// twoscale.cpp:131-242; respond(q, F, pbar[4], abar[16]) and commit() are the
// engines' MicroEngine calls.
TwoscaleResult twoscale(const MacroCfg& cfg, const std::function<void(int, const double*, double*, double*)>& respond,
                        const std::function<void()>& commit) {
  const Q8Mesh mesh = structured_quad8(cfg.nx, cfg.ny, cfg.width, cfg.height);
  const Q8Cache cache = cache_of(mesh);
  const int nn = (int)mesh.nodes.size(), nq = (int)cache.w.size();
  std::vector<int> node_dof(nn, 0);
  for (const auto& b : mesh.boundary)
    if (b.second == kBottom) node_dof[b.first] = -1;
  int n = 0;
  for (int i = 0; i < nn; ++i) {
    if (node_dof[i] == -1) continue;
    node_dof[i] = n;
    n += 2;
  }
  const std::vector<double> fext_full = traction(mesh, cfg.width, cfg.peak);
  std::vector<double> fext(n, 0.0);
  for (int i = 0; i < nn; ++i)
    if (node_dof[i] >= 0) {
      fext[node_dof[i]] = fext_full[2 * i];
      fext[node_dof[i] + 1] = fext_full[2 * i + 1];
    }
  TwoscaleResult out;
  std::vector<double> u(n, 0.0);
  auto expand = [&]() {
    std::vector<double> f(2 * nn, 0.0);
    for (int i = 0; i < nn; ++i)
      if (node_dof[i] >= 0) {
        f[2 * i] = u[node_dof[i]];
        f[2 * i + 1] = u[node_dof[i] + 1];
      }
    return f;
  };
  const int up = cfg.steps / 2;
  for (int step = 0; step < cfg.steps; ++step) {
    const double factor =
        step < up ? (double)(step + 1) / up : (double)(cfg.steps - 1 - step) / (cfg.steps - up);
    double tol = cfg.eps_abs;
    int iters = 0;
    for (int it = 0;; ++it) {
      const std::vector<double> uf = expand();
      std::vector<double> fint(2 * nn, 0.0), K((size_t)n * n, 0.0);
      for (int q = 0; q < nq; ++q) {
        const int e = cache.elem_of[q];
        const auto& g = cache.grad[q];
        Mat2 h;
        for (int a = 0; a < 8; ++a) {
          const int node = mesh.elems[e][a];
          for (int j = 0; j < 2; ++j) {
            h(0, j) += uf[2 * node] * g[2 * a + j];
            h(1, j) += uf[2 * node + 1] * g[2 * a + j];
          }
        }
        Mat2 F = Mat2::identity();
        for (int k = 0; k < 4; ++k) F.a[k] += h.a[k];
        double pb[4], ab[16];
        respond(q, F.a, pb, ab);
        const double w = cache.w[q];
        for (int a = 0; a < 8; ++a) {
          const int na = mesh.elems[e][a];
          const double ga[2] = {g[2 * a], g[2 * a + 1]};
          fint[2 * na] += w * (pb[0] * ga[0] + pb[2] * ga[1]);
          fint[2 * na + 1] += w * (pb[1] * ga[0] + pb[3] * ga[1]);
          const int da = node_dof[na];
          if (da < 0) continue;
          for (int b = 0; b < 8; ++b) {
            const int db = node_dof[mesh.elems[e][b]];
            if (db < 0) continue;
            const double gb[2] = {g[2 * b], g[2 * b + 1]};
            for (int r = 0; r < 2; ++r)
              for (int s = 0; s < 2; ++s) {
                double v = 0.0;
                for (int c = 0; c < 2; ++c)
                  for (int d = 0; d < 2; ++d) v += ga[c] * ab[(r + 2 * c) + 4 * (s + 2 * d)] * gb[d];
                K[(size_t)(db + s) * n + da + r] += w * v;
              }
          }
        }
      }
      std::vector<double> res(n);
      for (int i = 0; i < nn; ++i)
        if (node_dof[i] >= 0) {
          res[node_dof[i]] = fint[2 * i] - factor * fext[node_dof[i]];
          res[node_dof[i] + 1] = fint[2 * i + 1] - factor * fext[node_dof[i] + 1];
        }
      double rn = 0.0;
      for (double v : res) rn += v * v;
      rn = std::sqrt(rn);
      if (it == 0) tol = std::max(cfg.eps_rel * rn, cfg.eps_abs);
      if (rn <= tol) {
        iters = it;
        break;
      }
      if (it >= cfg.max_iter) throw SolveError("macro Newton did not converge at step " + std::to_string(step));
      for (double& v : res) v = -v;
      const std::vector<double> du = lu_solve(std::move(K), n, res);
      for (int i = 0; i < n; ++i) u[i] += du[i];
    }
    commit();
    const std::vector<double> uf = expand();
    double comp = 0.0;
    for (size_t i = 0; i < uf.size(); ++i) comp += fext_full[i] * uf[i];
    out.load_factor.push_back(factor);
    out.compliance.push_back(factor * comp);
    out.iters.push_back(iters);
  }
  out.u_final = expand();
  double nrm = 0.0;
  for (double v : out.u_final) nrm += v * v;
  out.residual_norm = std::sqrt(nrm);
  return out;
}

}  // namespace orc
