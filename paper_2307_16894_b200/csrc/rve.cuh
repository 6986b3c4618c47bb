// RVE tables shared by the assembly (K2) and ROM (K3) kernels, and the
// device-side analytic morph (MorphOperator::derive semantics,
// /root/reference/proj/src/morph.cpp:97-126).
#pragma once

#include <vector>

#include "common.cuh"

struct podecm_rve {
  podecm_ctx* ctx = nullptr;
  int n_cells = 0;
  double r0 = 0.25;
  int n_nodes = 0, n_elems = 0, n_qp = 0, n_red = 0, anchor = -1;
  int64_t nnz = 0, n_trip = 0;
  int n_mats = 0;
  podecm_impl::MatTable mats{};
  // host tables
  std::vector<double> nodes, grad, w;
  std::vector<int32_t> elems, regions, node_dof, row_ptr, col_idx;
  std::vector<int32_t> slot_ptr, slot_terms;  // exported: triplet ids q*64 + tl
  std::vector<int32_t> slot_grp;              // device form: e*64 + tl per 4-qp group
  std::vector<int32_t> slot_gptr;             // groups per slot
  std::vector<int32_t> frow_gptr, frow_grp;   // residual rows: e*8 + (a*2+i) groups
  // slot-ordered element-sum layout: pos[e*72 + t] = index of element term t
  // (t < 64: K term tl, t >= 64: f term) in the concatenated group list
  // (slot groups, then residual-row groups); -1 = unused (anchor dofs).
  std::vector<int32_t> pos, gptr_all;
  int64_t n_groups = 0;
  // tiled assembly (k_asm_qp2t): CTA = one 8 x 4 element tile; an item (CSR
  // slot or residual row) whose element sums all come from one tile is summed
  // there from shared memory (same group order as the gather); the others
  // ("halo") go through a compact scratch and the halo gather.
  int n_tiles = 0;                            // 0: not tiled (mesh not divisible)
  std::vector<int32_t> t_elem;                // [n_tiles * 32] element of (tile, local element)
  std::vector<int32_t> t_lptr, t_litem;       // per tile: local items
  std::vector<uint64_t> t_lpack;              // their <= 4 SMEM offsets (le * 72 + term), 12 bits each, + count
  std::vector<int32_t> t_hitem, t_hgptr, t_hpos;  // halo items, their compact groups, positions
  int64_t n_hgroups = 0;
  // device tables
  int32_t *d_t_elem = nullptr, *d_t_lptr = nullptr, *d_t_litem = nullptr;
  uint64_t* d_t_lpack = nullptr;
  int32_t *d_t_hitem = nullptr, *d_t_hgptr = nullptr, *d_t_hpos = nullptr;
  double *d_nodes = nullptr, *d_grad = nullptr, *d_w = nullptr;
  int32_t *d_elems = nullptr, *d_regions = nullptr, *d_node_dof = nullptr;
  int32_t *d_slot_gptr = nullptr, *d_slot_grp = nullptr, *d_frow_gptr = nullptr,
          *d_frow_grp = nullptr, *d_pos = nullptr, *d_gptr_all = nullptr;
  // assembly scratch (per-qp K and f terms of a chunk of instances)
  double* d_scratch = nullptr;
  int64_t scratch_inst = 0;  // bytes of d_scratch
};

namespace podecm_dev {

// Analytic circle->ellipse map (BASELINE configs 0/2/3), same expression
// order as oracle/mesh.cpp analytic_morph_d.
__device__ __forceinline__ void morph_d(double X, double Y, double ka, double kb, double r0,
                                        double& d0, double& d1) {
  const double dx = X - 0.5, dy = Y - 0.5;
  const double r = sqrt(dx * dx + dy * dy);
  const double s = r <= r0 ? 1.0 : (r < 0.5 ? (0.5 - r) / (0.5 - r0) : 0.0);
  d0 = s * (ka * dx);
  d1 = s * (kb * dy);
}

// derive() at one quadrature point from the 4 nodal displacements:
// Fmu = I + sum_a d_a (x) g_a, det, Fmu^-1.
__device__ __forceinline__ double derive_qp(const double d[4][2], const double g[8], double fmi[4]) {
  double gd[4];
#pragma unroll
  for (int j = 0; j < 2; ++j)
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      double s = 0.0;
#pragma unroll
      for (int a = 0; a < 4; ++a) s = s + d[a][i] * g[2 * a + j];
      gd[i + 2 * j] = s;
    }
  double fmu[4];
  fmu[0] = 1.0 + gd[0];
  fmu[1] = 0.0 + gd[1];
  fmu[2] = 0.0 + gd[2];
  fmu[3] = 1.0 + gd[3];
  const double dt = fmu[0] * fmu[3] - fmu[1] * fmu[2];
  mat2_inv(fmu, fmi);
  return dt;
}

}  // namespace podecm_dev

namespace podecm_impl {
// Residual-row sums of column `col` of a stored tangent field [n][16][n_qp]
// (effective_stiffness right-hand sides, microfem.cpp:262-281), k_assemble.cu.
int assemble_field_rows(podecm_ctx* ctx, cudaStream_t s, podecm_rve* r, int64_t n, const double* geom,
                        const double* morph, const double* field, int col, double* out);
}  // namespace podecm_impl
