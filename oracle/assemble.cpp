// ORACLE — TEST INFRASTRUCTURE ONLY (see oracle.hpp).
// Restates /root/reference/proj/src/microfem.cpp:56-130 (assemble) for Q4
// elements, and Eigen::SparseMatrix::setFromTriplets (called at
// microfem.cpp:127): duplicates summed sequentially in triplet order,
// structural zeros kept, inner indices sorted.  Emits CSR of K (row = test
// dof ra+i, col = trial dof rb+j), see SURVEY.md §8(a) a11.
#include "oracle.hpp"

#include <algorithm>
#include <numeric>

namespace orc {

namespace {

struct Trip {
  int r, c;
  double v;
};

// Eigen set_from_triplets (SparseCore/SparseMatrix.h) restated for a
// row-compressed result.
void set_from_triplets(int n, const std::vector<Trip>& t, Csr& out) {
  std::vector<int> cnt(n + 1, 0);
  for (const Trip& x : t) cnt[x.r + 1]++;
  std::vector<int> start(n + 1, 0);
  for (int r = 0; r < n; ++r) start[r + 1] = start[r] + cnt[r + 1];
  std::vector<int> fill(start.begin(), start.end() - 1);
  std::vector<int> bc(t.size());
  std::vector<double> bv(t.size());
  for (const Trip& x : t) {  // insertion in triplet order
    bc[fill[x.r]] = x.c;
    bv[fill[x.r]] = x.v;
    fill[x.r]++;
  }
  out.n = n;
  out.row_ptr.assign(n + 1, 0);
  out.col.clear();
  out.val.clear();
  std::vector<int> where(n, -1);
  for (int r = 0; r < n; ++r) {
    const int row_begin = (int)out.col.size();
    for (int k = start[r]; k < start[r + 1]; ++k) {  // collapseDuplicates
      const int c = bc[k];
      if (where[c] >= row_begin) {
        out.val[where[c]] = out.val[where[c]] + bv[k];
      } else {
        where[c] = (int)out.col.size();
        out.col.push_back(c);
        out.val.push_back(bv[k]);
      }
    }
    // transposed copy in Eigen == sort inner indices
    const int row_end = (int)out.col.size();
    std::vector<int> perm(row_end - row_begin);
    std::iota(perm.begin(), perm.end(), row_begin);
    std::sort(perm.begin(), perm.end(), [&](int a, int b) { return out.col[a] < out.col[b]; });
    std::vector<int> sc;
    std::vector<double> sv;
    for (int p : perm) {
      sc.push_back(out.col[p]);
      sv.push_back(out.val[p]);
    }
    std::copy(sc.begin(), sc.end(), out.col.begin() + row_begin);
    std::copy(sv.begin(), sv.end(), out.val.begin() + row_begin);
    out.row_ptr[r + 1] = row_end;
  }
}

// A(i,j,k,l) = m(idx(i,j), idx(k,l)), storage r + 4c (types.hpp:24-33).
inline double A4(const double* m, int i, int j, int k, int l) {
  return m[(i + 2 * j) + 4 * (k + 2 * l)];
}

}  // namespace

void assemble(const RveProblem& prob, const Morph& morph, const std::vector<PlasticState>& s0,
              std::vector<PlasticState>* s1, const Mat2& fbar, const std::vector<double>& w_red,
              bool tangent, std::vector<double>& f, Csr* K, std::vector<double>* p_field,
              std::vector<double>* a_field) {
  const Mesh& mesh = prob.mesh;
  const QuadCache& cache = prob.cache;
  const int nqp = cache.n_qp();
  // DofMap::expand (mesh.cpp:390-400)
  std::vector<double> wf(2 * (size_t)mesh.n_nodes, 0.0);
  for (int i = 0; i < mesh.n_nodes; ++i) {
    const int d = prob.dofs.node_dof[i];
    if (d < 0) continue;
    wf[2 * i] = w_red[d];
    wf[2 * i + 1] = w_red[d + 1];
  }
  f.assign(prob.dofs.n_red, 0.0);
  if (p_field) p_field->assign(4 * (size_t)nqp, 0.0);
  if (a_field) a_field->assign(16 * (size_t)nqp, 0.0);
  if (s1) s1->resize(nqp);
  std::vector<Trip> trips;
  if (tangent) trips.reserve((size_t)nqp * 64);

  for (int q = 0; q < nqp; ++q) {
    const int e = cache.elem_of[q];
    const double* g = &cache.grad[(size_t)q * 8];
    const Mat2& fmi = morph.fmu_inv[q];
    Mat2 gw;
    for (int a = 0; a < 4; ++a) {
      const int node = mesh.elems[4 * e + a];
      for (int i = 0; i < 2; ++i)
        for (int j = 0; j < 2; ++j) gw(i, j) += wf[2 * node + i] * g[2 * a + j];
    }
    const Mat2 gf = mul(gw, fmi);
    Mat2 F;
    for (int k = 0; k < 4; ++k) F.a[k] = fbar.a[k] + gf.a[k];

    const PlasticityParams& mat = prob.material_at(q);
    const LargeResult lr = large_strain_update(mat, s0[q], F, s1 ? &(*s1)[q] : nullptr);
    if (p_field)
      for (int k = 0; k < 4; ++k) (*p_field)[4 * (size_t)q + k] = lr.P.a[k];

    const double wq = cache.w[q] * morph.det[q];
    double gt[4][2];
    for (int a = 0; a < 4; ++a)
      for (int j = 0; j < 2; ++j) gt[a][j] = g[2 * a] * fmi(0, j) + g[2 * a + 1] * fmi(1, j);

    for (int a = 0; a < 4; ++a) {
      const int ra = prob.dofs.node_dof[mesh.elems[4 * e + a]];
      if (ra < 0) continue;
      for (int i = 0; i < 2; ++i) f[ra + i] += wq * (lr.P(i, 0) * gt[a][0] + lr.P(i, 1) * gt[a][1]);
    }
    if (!tangent) continue;
    double a4[16];
    large_strain_tangent(mat, s0[q], F, 1e-7, a4);
    if (a_field)  // AssemblyOpts::store_tangent_field (microfem.hpp:62)
      for (int k = 0; k < 16; ++k) (*a_field)[16 * (size_t)q + k] = a4[k];
    for (int a = 0; a < 4; ++a) {
      const int ra = prob.dofs.node_dof[mesh.elems[4 * e + a]];
      if (ra < 0) continue;
      for (int b = 0; b < 4; ++b) {
        const int rb = prob.dofs.node_dof[mesh.elems[4 * e + b]];
        if (rb < 0) continue;
        for (int i = 0; i < 2; ++i)
          for (int j = 0; j < 2; ++j) {
            const double v =
                gt[a][0] * (A4(a4, i, 0, j, 0) * gt[b][0] + A4(a4, i, 0, j, 1) * gt[b][1]) +
                gt[a][1] * (A4(a4, i, 1, j, 0) * gt[b][0] + A4(a4, i, 1, j, 1) * gt[b][1]);
            trips.push_back({ra + i, rb + j, wq * v});
          }
      }
    }
  }
  if (tangent && K) set_from_triplets(prob.dofs.n_red, trips, *K);
}

}  // namespace orc
