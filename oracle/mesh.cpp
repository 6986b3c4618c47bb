// ORACLE — TEST INFRASTRUCTURE ONLY (see oracle.hpp).
// Q4 analogue of /root/reference/proj/src/mesh.cpp (shape_eval :24-64,
// quadrature :66-83, periodic_pairs :307-358, periodic_dof_map :360-374,
// build_quad_cache :412-451) and MorphOperator::derive (morph.cpp:97-126),
// plus the analytic circle->ellipse map of BASELINE.json configs 0/2/3.
#include "oracle.hpp"

#include <algorithm>
#include <map>

namespace orc {

// Structured n x n Q4 grid: node id j*(n+1)+i at (i/n, j/n); cells row-major
// with CCW corners (i,j),(i+1,j),(i+1,j+1),(i,j+1) — the corner order of
// structured_quad8 (meshgen.cpp:97-100).  Region 1 = element centroid within
// r0 of the cell centre (BASELINE config 0).
Mesh structured_q4(int n, double r0) {
  if (n < 1) throw ConfigError("structured_q4 needs n >= 1");
  Mesh m;
  const int np = n + 1;
  m.n_nodes = np * np;
  m.n_elems = n * n;
  m.nodes.resize(2 * (size_t)m.n_nodes);
  for (int j = 0; j < np; ++j)
    for (int i = 0; i < np; ++i) {
      m.nodes[2 * (j * np + i)] = i / (double)n;
      m.nodes[2 * (j * np + i) + 1] = j / (double)n;
    }
  m.elems.resize(4 * (size_t)m.n_elems);
  m.regions.resize(m.n_elems);
  for (int cj = 0; cj < n; ++cj)
    for (int ci = 0; ci < n; ++ci) {
      const int e = cj * n + ci;
      const int c[4] = {cj * np + ci, cj * np + ci + 1, (cj + 1) * np + ci + 1, (cj + 1) * np + ci};
      double cx = 0, cy = 0;
      for (int a = 0; a < 4; ++a) {
        m.elems[4 * e + a] = c[a];
        cx += m.nodes[2 * c[a]];
        cy += m.nodes[2 * c[a] + 1];
      }
      cx = 0.25 * cx - 0.5;
      cy = 0.25 * cy - 0.5;
      m.regions[e] = std::sqrt(cx * cx + cy * cy) <= r0 ? 1 : 0;
    }
  return m;
}

namespace {
const double kCx[4] = {-1, 1, 1, -1};
const double kCy[4] = {-1, -1, 1, 1};
}  // namespace

// Bilinear shape derivatives at the 2x2 Gauss points (w = 1, g = 1/sqrt 3,
// point order of mesh.cpp:76-80); J = X^T dN (4-term sums in Eigen's SSE2
// redux order (t0+t2)+(t1+t3)), grad = dN J^-1, w = det J.
QuadCache build_quad_cache(const Mesh& m) {
  const double g = 1.0 / std::sqrt(3.0);
  const double qx[4] = {-g, g, g, -g}, qy[4] = {-g, -g, g, g};
  double dn[4][4][2];
  for (int q = 0; q < 4; ++q)
    for (int a = 0; a < 4; ++a) {
      dn[q][a][0] = 0.25 * kCx[a] * (1 + qy[q] * kCy[a]);
      dn[q][a][1] = 0.25 * kCy[a] * (1 + qx[q] * kCx[a]);
    }
  QuadCache c;
  const int nq = 4 * m.n_elems;
  c.grad.resize((size_t)nq * 8);
  c.w.resize(nq);
  c.elem_of.resize(nq);
  for (int e = 0; e < m.n_elems; ++e) {
    double X[4][2];
    for (int a = 0; a < 4; ++a) {
      X[a][0] = m.nodes[2 * m.elems[4 * e + a]];
      X[a][1] = m.nodes[2 * m.elems[4 * e + a] + 1];
    }
    for (int q = 0; q < 4; ++q) {
      Mat2 jac;
      for (int i = 0; i < 2; ++i)
        for (int j = 0; j < 2; ++j) {
          const double t0 = X[0][i] * dn[q][0][j], t1 = X[1][i] * dn[q][1][j];
          const double t2 = X[2][i] * dn[q][2][j], t3 = X[3][i] * dn[q][3][j];
          jac(i, j) = (t0 + t2) + (t1 + t3);
        }
      const double dj = det(jac);
      if (dj <= 0.0)
        throw SolveError("element " + std::to_string(e) + " has non-positive Jacobian");
      const Mat2 ji = inverse(jac);
      const int gq = 4 * e + q;
      for (int a = 0; a < 4; ++a)
        for (int j = 0; j < 2; ++j)
          c.grad[(size_t)gq * 8 + 2 * a + j] = dn[q][a][0] * ji(0, j) + dn[q][a][1] * ji(1, j);
      c.w[gq] = 1.0 * dj;
      c.elem_of[gq] = e;
    }
  }
  return c;
}

// mesh.cpp:307-374.  Anchor (0,0) pinned; right->left, top->bottom, the other
// three corners -> anchor; masters numbered 2 dofs each in node order.
DofMap periodic_dof_map(const Mesh& m, double tol) {
  auto near = [tol](double a, double b) { return std::abs(a - b) <= tol; };
  int anchor = -1;
  std::vector<int> corners, left, right, bottom, top;
  for (int i = 0; i < m.n_nodes; ++i) {
    const double x = m.nodes[2 * i], y = m.nodes[2 * i + 1];
    const bool x0 = near(x, 0), x1 = near(x, 1), y0 = near(y, 0), y1 = near(y, 1);
    if (x0 && y0)
      anchor = i;
    else if ((x1 && y0) || (x0 && y1) || (x1 && y1))
      corners.push_back(i);
    else if (x0)
      left.push_back(i);
    else if (x1)
      right.push_back(i);
    else if (y0)
      bottom.push_back(i);
    else if (y1)
      top.push_back(i);
  }
  if (anchor < 0 || corners.size() != 3)
    throw SolveError("periodic pairing requires all four corner nodes");
  std::map<int, int> slave_of;
  for (int c : corners) slave_of[c] = anchor;
  auto pair_faces = [&](std::vector<int>& ma, std::vector<int>& sl, int coord) {
    auto key = [&](int n) { return m.nodes[2 * n + coord]; };
    std::sort(ma.begin(), ma.end(), [&](int a, int b) { return key(a) < key(b); });
    std::sort(sl.begin(), sl.end(), [&](int a, int b) { return key(a) < key(b); });
    if (ma.size() != sl.size()) throw SolveError("periodic pairing: face node counts differ");
    for (size_t k = 0; k < ma.size(); ++k) {
      if (!near(key(ma[k]), key(sl[k]))) throw SolveError("periodic pairing: unmatched node");
      slave_of[sl[k]] = ma[k];
    }
  };
  pair_faces(left, right, 1);
  pair_faces(bottom, top, 0);

  DofMap d;
  d.anchor = anchor;
  d.node_dof.assign(m.n_nodes, -2);
  int next = 0;
  for (int i = 0; i < m.n_nodes; ++i) {
    if (i == anchor || slave_of.count(i)) continue;
    d.node_dof[i] = next;
    next += 2;
  }
  d.node_dof[anchor] = -1;
  for (const auto& kv : slave_of) d.node_dof[kv.first] = d.node_dof[kv.second];
  d.n_red = next;
  return d;
}

// Analytic morph of BASELINE configs 0/2/3: d(X) = s(r) [(a/r0-1)(X1-.5),
// (b/r0-1)(X2-.5)], s = 1 (r <= r0), (0.5-r)/(0.5-r0) (r0 < r < 0.5), 0.
std::vector<double> analytic_morph_d(const Mesh& m, double a, double b, double r0) {
  std::vector<double> d(2 * (size_t)m.n_nodes);
  const double ka = a / r0 - 1.0, kb = b / r0 - 1.0;
  for (int i = 0; i < m.n_nodes; ++i) {
    const double dx = m.nodes[2 * i] - 0.5, dy = m.nodes[2 * i + 1] - 0.5;
    const double r = std::sqrt(dx * dx + dy * dy);
    const double s = r <= r0 ? 1.0 : (r < 0.5 ? (0.5 - r) / (0.5 - r0) : 0.0);
    d[2 * i] = s * (ka * dx);
    d[2 * i + 1] = s * (kb * dy);
  }
  return d;
}

// morph.cpp:97-126.
Morph derive(const Mesh& m, const QuadCache& c, const std::vector<double>& d) {
  Morph f;
  const int nq = c.n_qp();
  f.fmu_inv.resize(nq);
  f.det.resize(nq);
  f.volume = 0;
  f.min_det = 1e300;
  for (int q = 0; q < nq; ++q) {
    const int e = c.elem_of[q];
    Mat2 gd;
    for (int a = 0; a < 4; ++a) {
      const int node = m.elems[4 * e + a];
      for (int i = 0; i < 2; ++i)
        for (int j = 0; j < 2; ++j) gd(i, j) += d[2 * node + i] * c.grad[(size_t)q * 8 + 2 * a + j];
    }
    Mat2 fmu = Mat2::identity();
    for (int k = 0; k < 4; ++k) fmu.a[k] = Mat2::identity().a[k] + gd.a[k];
    const double dt = det(fmu);
    f.det[q] = dt;
    f.min_det = std::min(f.min_det, dt);
    if (dt <= 0.0) throw SolveError("morph folds the mesh at quadrature point " + std::to_string(q));
    f.fmu_inv[q] = inverse(fmu);
    f.volume += c.w[q] * dt;
  }
  return f;
}

}  // namespace orc
