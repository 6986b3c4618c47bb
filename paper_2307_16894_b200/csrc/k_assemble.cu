// K2 — batched full-order assembly of the Q4 RVE (BASELINE configs 0 and 2).
//
// Two kernels per chunk of instances, no atomics, bitwise reproducible:
//   k_asm_qp2    one thread per (instance, quadrature point), a quad of lanes
//                per element: analytic morph (derive), F = Fbar + grad(w)
//                Fmu^-1, the material point (P, FD tangent, history), then
//                the element sums of the 64 K-terms wq * gt_a . A . gt_b and
//                8 f-terms (microfem.cpp:76-123), written to their
//                slot-ordered scratch positions;
//   k_asm_gather_fused  one thread per (instance, CSR slot or residual row):
//                a contiguous run of element sums added in element order.
// Exact mode (PODECM_ASM_EXACT=1: k_asm_qp + k_asm_gather) stores every
// per-qp term and sums each slot in the reference's triplet order — exactly
// the order Eigen's setFromTriplets collapses duplicates in
// (microfem.cpp:125-128).
#include <algorithm>
#include <cstdlib>

#include "rve.cuh"

using namespace podecm_dev;
using namespace podecm_impl;

namespace {

struct AsmArgs {
  int n_qp, n_red;
  int64_t nnz;
  int64_t inst0;  // first instance of the chunk
  int n_inst;     // instances in this chunk
  double r0;
  const double* nodes;
  const int32_t* elems;
  const int32_t* regions;
  const double* grad;
  const double* w;
  const int32_t* node_dof;
  const double* geom;
  const double* morph;
  const double* fbar;
  const double* w_red;
  const double* st0;
  double* st1;
  double* p_field;
  double* scratch;  // exact: [chunk inst][n_elems][72][4]; fused: [chunk inst][n_groups]
  const int32_t* pos;
  int64_t n_groups;
  int32_t* status;
  unsigned int* fail;
  bool tangent;
  double* a_field;  // nullable [n][16][n_qp] (AssemblyOpts::store_tangent_field)
  const double* field;  // field-rows mode: [n][16][n_qp] tangent field, column `field_col`
  int field_col;
  // tiled mode (k_asm_qp2t): tile tables (rve.cuh), local item outputs
  const int32_t* t_elem;
  const int32_t* t_lptr;
  const int32_t* t_litem;
  const uint64_t* t_lpack;
  const int32_t* t_hpos;
  double* kvals;
  double* f;
};

// 4-lane butterfly over the quad of lanes holding the 4 qps of one element:
// every lane ends with 2 of the 8 element sums, (t0 + t1) + (t2 + t3) for
// every entry whichever lane computes it (deterministic).  Lane k holds the
// entries u = 4 (k & 1) + 2 ((k >> 1) & 1) + {0, 1}.
__device__ __forceinline__ void quad_reduce8(const double v[8], int k, double out[2]) {
  const bool h1 = (k & 1) != 0, h2 = (k & 2) != 0;
  double w[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const double mine = h1 ? v[i + 4] : v[i];
    const double other = h1 ? v[i] : v[i + 4];
    w[i] = mine + __shfl_xor_sync(0xffffffffu, other, 1);
  }
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const double mine = h2 ? w[i + 2] : w[i];
    const double other = h2 ? w[i] : w[i + 2];
    out[i] = mine + __shfl_xor_sync(0xffffffffu, other, 2);
  }
}

// Exact mode (PODECM_ASM_EXACT=1): every per-qp term is stored element-
// blocked and the gather replays Eigen's setFromTriplets order exactly.  The
// default (k_asm_qp2 below) sums the 4 qp contributions of an element first
// (quad butterfly), so K and f differ from the strict triplet order only in
// the association inside one element (ulp level) and stay deterministic.
template <int MINB>
__global__ void __launch_bounds__(128, MINB) k_asm_qp(AsmArgs g, MatTable tab) {
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t total = (int64_t)g.n_inst * g.n_qp;
  const bool valid = tid < total;
  if (!valid) return;
  const int c = (int)(tid / g.n_qp);
  const int q = (int)(tid - (int64_t)c * g.n_qp);
  const int64_t inst = g.inst0 + c;
  const int e = q >> 2, k = q & 3;
  const int nq = g.n_qp;

  double gq[8];
#pragma unroll
  for (int t = 0; t < 8; ++t) gq[t] = __ldg(g.grad + (size_t)q * 8 + t);
  int node[4];
#pragma unroll
  for (int a = 0; a < 4; ++a) node[a] = __ldg(g.elems + 4 * e + a);

  // morph at this qp
  double fmi[4], det;
  if (g.morph) {
    const double* mo = g.morph + (size_t)inst * 5 * nq;
#pragma unroll
    for (int t = 0; t < 4; ++t) fmi[t] = __ldg(mo + (size_t)t * nq + q);
    det = __ldg(mo + (size_t)4 * nq + q);
  } else {
    const double ka = __ldg(g.geom + 2 * inst) / g.r0 - 1.0;
    const double kb = __ldg(g.geom + 2 * inst + 1) / g.r0 - 1.0;
    double d[4][2];
#pragma unroll
    for (int a = 0; a < 4; ++a)
      morph_d(__ldg(g.nodes + 2 * node[a]), __ldg(g.nodes + 2 * node[a] + 1), ka, kb, g.r0, d[a][0],
              d[a][1]);
    det = derive_qp(d, gq, fmi);
  }
  // fluctuation gradient gw(i,j) = sum_a w(2 node_a + i) g(a,j), then F
  const double* wr = g.w_red + (size_t)inst * g.n_red;
  double wn[4][2];
#pragma unroll
  for (int a = 0; a < 4; ++a) {
    const int dof = __ldg(g.node_dof + node[a]);
    wn[a][0] = dof >= 0 ? __ldg(wr + dof) : 0.0;
    wn[a][1] = dof >= 0 ? __ldg(wr + dof + 1) : 0.0;
  }
  double gw[4];
#pragma unroll
  for (int j = 0; j < 2; ++j)
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      double s = 0.0;
#pragma unroll
      for (int a = 0; a < 4; ++a) s = s + wn[a][i] * gq[2 * a + j];
      gw[i + 2 * j] = s;
    }
  double F[4];
  const double* fb = g.fbar + 4 * inst;
#pragma unroll
  for (int j = 0; j < 2; ++j)
#pragma unroll
    for (int i = 0; i < 2; ++i)
      F[i + 2 * j] = __ldg(fb + i + 2 * j) + (gw[i] * fmi[2 * j] + gw[i + 2] * fmi[1 + 2 * j]);

  // material point with frozen history
  int reg = __ldg(g.regions + e);
  const MatConst& p = tab.m[reg];
  const double* s0 = g.st0 + (size_t)inst * 6 * nq;
  double fp[4];
#pragma unroll
  for (int t = 0; t < 4; ++t) fp[t] = __ldg(s0 + (size_t)t * nq + q);
  Frozen z;
  freeze(fp, __ldg(s0 + (size_t)4 * nq + q), __ldg(s0 + (size_t)5 * nq + q), z);
  double P[4];
  FullOut fo;
  bool ok = lsu_eval<true>(p, z, F, P, &fo);
  if (g.st1 && valid) {
    double* s1 = g.st1 + (size_t)inst * 6 * nq;
#pragma unroll
    for (int t = 0; t < 4; ++t) s1[(size_t)t * nq + q] = fo.fp[t];
    s1[(size_t)4 * nq + q] = fo.fpzz;
    s1[(size_t)5 * nq + q] = fo.xi;
  }
  if (g.p_field && valid) {
    double* pf = g.p_field + (size_t)inst * 4 * nq;
#pragma unroll
    for (int t = 0; t < 4; ++t) pf[(size_t)t * nq + q] = P[t];
  }

  const double wq = __ldg(g.w + q) * det;
  double gt[4][2];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int j = 0; j < 2; ++j) gt[a][j] = gq[2 * a] * fmi[2 * j] + gq[2 * a + 1] * fmi[1 + 2 * j];

  {
    // element-blocked scratch: [c][e][72][4], entry (term, k)
    double* sc = g.scratch + ((size_t)c * (nq >> 2) + e) * 72 * 4 + k;
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int i = 0; i < 2; ++i)
        sc[(64 + a * 2 + i) * 4] = wq * (P[i] * gt[a][0] + P[i + 2] * gt[a][1]);
    if (ok && g.tangent) {
      // A(i,c,j,d) = A[(i+2c) + 4(j+2d)]: column e = j + 2d.  Columns arrive
      // in the order 0, 2, 1, 3, so after the second column of each j the 32
      // terms K(a i, b j) += wq * sum_cd gt_ac A(i,c,j,d) gt_bd are emitted
      // (microfem.cpp:113-117 order).
      double cd[2][4];
      auto sink = [&](int ecol, const double col[4]) {
        const int d = ecol >> 1, j = ecol & 1;
        if (g.a_field)
#pragma unroll
          for (int r = 0; r < 4; ++r) g.a_field[((size_t)inst * 16 + r + 4 * ecol) * nq + q] = col[r];
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          cd[0][r] = d == 0 ? col[r] : cd[0][r];
          cd[1][r] = d == 1 ? col[r] : cd[1][r];
        }
        if (d == 0) return;
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
          for (int b = 0; b < 4; ++b)
#pragma unroll
            for (int i = 0; i < 2; ++i) {
              const double v = gt[a][0] * (cd[0][i] * gt[b][0] + cd[1][i] * gt[b][1]) +
                               gt[a][1] * (cd[0][i + 2] * gt[b][0] + cd[1][i + 2] * gt[b][1]);
              sc[((a * 4 + b) * 4 + i * 2 + j) * 4] = wq * v;
            }
      };
      ok = fd_tangent<false>(p, z, F, 1e-7, sink);
    }
  }
  if (!ok && valid) {
    if (g.status) g.status[inst] = PODECM_ESOLVE;
    atomicAdd(g.fail, 1u);
  }
}


// per-qp SMEM planes of the two-phase kernel: A (16), P (4), gt (8), wq (1)
constexpr int kQPlanes = 29;

// ---- default kernel: two phases per thread ------------------------------------
// Phase 1 is the material point; its FD loop only streams tangent columns
// into this thread's SMEM row (as the C1 kernel streams them to HBM), so no
// element accumulator is live across the material evaluations.  Phase 2
// reads the thread's A, P, gt, wq back and forms the element sums with the
// quad butterfly.  Lanes past the end (whole quads, n_qp % 4 == 0) compute on
// a clamped index so the shuffles stay converged, and never store.
// (Measured on C2: 25.8 ms vs 30.6 ms for the single-phase kernel that
// contracted each tangent column into element terms inside the FD loop.)
constexpr int kQ2Thr = 128;

// TILED (k_asm_qp2t): the CTA is one 8 x 4 element tile (blockIdx.x) of one
// instance (blockIdx.y); element sums also go to shared memory, and after the
// element phase the CTA sums the tile's local items there (in the gather's
// group order: the same bits) and stores them; only halo terms go to the
// compact scratch.  Otherwise one thread per (instance, qp) in qp order.
template <int MINB, bool TILED = false>
__global__ void __launch_bounds__(kQ2Thr, MINB) k_asm_qp2(AsmArgs g, MatTable tab) {
  __shared__ double sq[kQPlanes * kQ2Thr];  // [plane][thread]
  const int lt = threadIdx.x;
  bool valid;
  int c, q;
  if constexpr (TILED) {
    valid = true;
    c = blockIdx.y;
    q = 4 * __ldg(g.t_elem + (size_t)blockIdx.x * 32 + (lt >> 2)) + (lt & 3);
  } else {
    const int64_t tid0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t total = (int64_t)g.n_inst * g.n_qp;
    valid = tid0 < total;
    const int64_t tid = valid ? tid0 : total - 1;  // whole quads stay converged
    c = (int)(tid / g.n_qp);
    q = (int)(tid - (int64_t)c * g.n_qp);
  }
  const int64_t inst = g.inst0 + c;
  const int e = q >> 2, k = q & 3;
  const int nq = g.n_qp;
  bool ok = true;
  {
    double gq[8];
#pragma unroll
    for (int t = 0; t < 8; ++t) gq[t] = __ldg(g.grad + (size_t)q * 8 + t);
    int node[4];
#pragma unroll
    for (int a = 0; a < 4; ++a) node[a] = __ldg(g.elems + 4 * e + a);
    double fmi[4], det;
    if (g.morph) {
      const double* mo = g.morph + (size_t)inst * 5 * nq;
#pragma unroll
      for (int t = 0; t < 4; ++t) fmi[t] = __ldg(mo + (size_t)t * nq + q);
      det = __ldg(mo + (size_t)4 * nq + q);
    } else {
      const double ka = __ldg(g.geom + 2 * inst) / g.r0 - 1.0;
      const double kb = __ldg(g.geom + 2 * inst + 1) / g.r0 - 1.0;
      double d[4][2];
#pragma unroll
      for (int a = 0; a < 4; ++a)
        morph_d(__ldg(g.nodes + 2 * node[a]), __ldg(g.nodes + 2 * node[a] + 1), ka, kb, g.r0, d[a][0],
                d[a][1]);
      det = derive_qp(d, gq, fmi);
    }
    const double* wr = g.w_red + (size_t)inst * g.n_red;
    double wn[4][2];
#pragma unroll
    for (int a = 0; a < 4; ++a) {
      const int dof = __ldg(g.node_dof + node[a]);
      wn[a][0] = dof >= 0 ? __ldg(wr + dof) : 0.0;
      wn[a][1] = dof >= 0 ? __ldg(wr + dof + 1) : 0.0;
    }
    double gw[4];
#pragma unroll
    for (int j = 0; j < 2; ++j)
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        double sm = 0.0;
#pragma unroll
        for (int a = 0; a < 4; ++a) sm = sm + wn[a][i] * gq[2 * a + j];
        gw[i + 2 * j] = sm;
      }
    double F[4];
    const double* fb = g.fbar + 4 * inst;
#pragma unroll
    for (int j = 0; j < 2; ++j)
#pragma unroll
      for (int i = 0; i < 2; ++i)
        F[i + 2 * j] = __ldg(fb + i + 2 * j) + (gw[i] * fmi[2 * j] + gw[i + 2] * fmi[1 + 2 * j]);
    sq[28 * kQ2Thr + lt] = __ldg(g.w + q) * det;
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int j = 0; j < 2; ++j)
        sq[(20 + 2 * a + j) * kQ2Thr + lt] = gq[2 * a] * fmi[2 * j] + gq[2 * a + 1] * fmi[1 + 2 * j];
    const MatConst& p = tab.m[__ldg(g.regions + e)];
    const double* s0 = g.st0 + (size_t)inst * 6 * nq;
    double fp[4];
#pragma unroll
    for (int t = 0; t < 4; ++t) fp[t] = __ldg(s0 + (size_t)t * nq + q);
    Frozen z;
    freeze(fp, __ldg(s0 + (size_t)4 * nq + q), __ldg(s0 + (size_t)5 * nq + q), z);
    double P[4];
    FullOut fo;
    ok = lsu_eval<true>(p, z, F, P, &fo);
    if (g.st1 && valid) {
      double* s1 = g.st1 + (size_t)inst * 6 * nq;
#pragma unroll
      for (int t = 0; t < 4; ++t) s1[(size_t)t * nq + q] = fo.fp[t];
      s1[(size_t)4 * nq + q] = fo.fpzz;
      s1[(size_t)5 * nq + q] = fo.xi;
    }
    if (g.p_field && valid) {
      double* pf = g.p_field + (size_t)inst * 4 * nq;
#pragma unroll
      for (int t = 0; t < 4; ++t) pf[(size_t)t * nq + q] = P[t];
    }
#pragma unroll
    for (int t = 0; t < 4; ++t) sq[(16 + t) * kQ2Thr + lt] = P[t];
    if (g.tangent) {
      auto sink = [&](int ecol, const double col[4]) {
#pragma unroll
        for (int r = 0; r < 4; ++r) sq[(r + 4 * ecol) * kQ2Thr + lt] = col[r];
      };
      const bool ok2 = fd_tangent<false>(p, z, F, 1e-7, sink);
      ok = ok && ok2;
    }
  }
  if (g.a_field && g.tangent && valid)
#pragma unroll
    for (int t = 0; t < 16; ++t) g.a_field[((size_t)inst * 16 + t) * nq + q] = sq[t * kQ2Thr + lt];
  // ---- phase 2: element sums from this thread's SMEM row
  const double wq = sq[28 * kQ2Thr + lt];
  double gt[4][2], P[4];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int j = 0; j < 2; ++j) gt[a][j] = sq[(20 + 2 * a + j) * kQ2Thr + lt];
#pragma unroll
  for (int t = 0; t < 4; ++t) P[t] = sq[(16 + t) * kQ2Thr + lt];
  double* sc = g.scratch + (size_t)c * g.n_groups;
  const int32_t* ps = (TILED ? g.t_hpos : g.pos) + (size_t)e * 72;
  const int u0 = 4 * (k & 1) + 2 * ((k >> 1) & 1);
  // TILED: this element's 72 sums in shared memory, [local element][72]
  // TILED: the element sums stay in sq, each written over planes this pass
  // has finished reading (rve_host.cu tile_smem_slot: f terms over the first
  // stress planes, the K terms of trial component j over the tangent
  // columns j and j + 2); __syncwarp orders the quad's reads before writes.
  const int qb = lt & ~3;  // first lane of this element's quad
  {
    double v[8], o[2];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int i = 0; i < 2; ++i) v[a * 2 + i] = wq * (P[i] * gt[a][0] + P[i + 2] * gt[a][1]);
    quad_reduce8(v, k, o);
    if (valid) {
      const int p0 = __ldg(ps + 64 + u0), p1 = __ldg(ps + 64 + u0 + 1);
      if (p0 >= 0) sc[p0] = o[0];
      if (p1 >= 0) sc[p1] = o[1];
      if (TILED) {
        __syncwarp();
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int u = u0 + h;
          sq[(16 + (u >> 2)) * kQ2Thr + qb + (u & 3)] = o[h];
        }
      }
    }
  }
  if (g.tangent) {
#pragma unroll 1
    for (int j = 0; j < 2; ++j) {
      double cd[2][4];
#pragma unroll
      for (int dd = 0; dd < 2; ++dd)
#pragma unroll
        for (int r = 0; r < 4; ++r) cd[dd][r] = sq[(r + 4 * (j + 2 * dd)) * kQ2Thr + lt];
      if (TILED) __syncwarp();
      double T[2][2][4];
#pragma unroll
      for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int cc = 0; cc < 2; ++cc)
#pragma unroll
          for (int b = 0; b < 4; ++b) T[i][cc][b] = fma(cd[1][i + 2 * cc], gt[b][1], cd[0][i + 2 * cc] * gt[b][0]);
#pragma unroll
      for (int a = 0; a < 4; ++a) {
        double v[8], o[2];
        const double w0 = wq * gt[a][0], w1 = wq * gt[a][1];
#pragma unroll
        for (int b = 0; b < 4; ++b)
#pragma unroll
          for (int i = 0; i < 2; ++i) v[b * 2 + i] = fma(w1, T[i][1][b], w0 * T[i][0][b]);
        quad_reduce8(v, k, o);
        if (valid) {
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int u = u0 + h, b = u >> 1, i = u & 1;
            const int tl = a * 16 + b * 4 + i * 2 + j;
            const int pp = __ldg(ps + tl);
            if (pp >= 0) sc[pp] = o[h];
            if (TILED) {
              const int idx = a * 8 + b * 2 + i;
              const int pl = (idx >> 2) < 4 ? 4 * j + (idx >> 2) : 8 + 4 * j + (idx >> 2) - 4;
              sq[pl * kQ2Thr + qb + (idx & 3)] = o[h];
            }
          }
        }
      }
    }
  }
  if (!ok && valid) {
    if (g.status) g.status[inst] = PODECM_ESOLVE;
    atomicAdd(g.fail, 1u);
  }
  if constexpr (TILED) {
    // The tile's local items: the gather's sum (first group, then + in group
    // order; residual rows start from 0.0 +) over the element sums in SMEM.
    // Items fed by one element row (= this warp's 8 elements: two thirds of
    // them) are summed by the warp right after its own element phase, so a
    // warp that is ahead works instead of idling at the CTA barrier; the items
    // spanning two rows follow after the barrier.
    const int32_t* lp = g.t_lptr + (size_t)blockIdx.x * 5;
    const int64_t nnz = g.nnz;
    constexpr int kU = 4;  // items per thread per round, all table loads issued first
    auto sum_items = [&](int l0, int l1, int first, int stride) {
      for (int base = l0; base < l1; base += kU * stride) {
        int its[kU];
        uint64_t pks[kU];
#pragma unroll
        for (int u = 0; u < kU; ++u) {
          const int li = base + u * stride + first;
          its[u] = li < l1 ? __ldg(g.t_litem + li) : -1;
          pks[u] = li < l1 ? __ldg(g.t_lpack + li) : 0ull;
        }
#pragma unroll
        for (int u = 0; u < kU; ++u) {
          const int it = its[u];
          if (it < 0) continue;
          const bool is_slot = it < nnz;
          if (is_slot && !g.tangent) continue;
          const uint64_t pk = pks[u];
          const int n = (int)(pk >> 48);
          double sm = sq[pk & 0xfff];
          if (!is_slot) sm = 0.0 + sm;
          if (n > 1) sm = sm + sq[(pk >> 12) & 0xfff];
          if (n > 2) sm = sm + sq[(pk >> 24) & 0xfff];
          if (n > 3) sm = sm + sq[(pk >> 36) & 0xfff];
          if (is_slot)
            __stcs(g.kvals + (size_t)inst * nnz + it, sm);
          else
            __stcs(g.f + (size_t)inst * g.n_red + (it - nnz), sm);
        }
      }
    };
    const int w = lt >> 5;
    const int r0 = __ldg(lp + w), r1 = __ldg(lp + w + 1), c0 = __ldg(lp + 4), c1 = __ldg(lp + 5);
    __syncwarp();
    sum_items(r0, r1, lt & 31, 32);
    __syncthreads();
    sum_items(c0, c1, lt, kQ2Thr);
  }
}


// Residual-row sums of a 2x2 "stress" taken from a stored tangent field:
// Pc = A(:, :, k, l) with column c = k + 2l of A, i.e. the element terms
// wq (Pc(i,0) gt_a0 + Pc(i,1) gt_a1) of effective_stiffness's right-hand
// sides (microfem.cpp:262-281), summed exactly like the residual.
__global__ void __launch_bounds__(256) k_asm_field_terms(AsmArgs g) {
  const int64_t tid0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t total = (int64_t)g.n_inst * g.n_qp;
  const bool valid = tid0 < total;
  const int64_t tid = valid ? tid0 : total - 1;
  const int c = (int)(tid / g.n_qp);
  const int q = (int)(tid - (int64_t)c * g.n_qp);
  const int64_t inst = g.inst0 + c;
  const int e = q >> 2, k = q & 3;
  const int nq = g.n_qp;
  double gq[8];
#pragma unroll
  for (int t = 0; t < 8; ++t) gq[t] = __ldg(g.grad + (size_t)q * 8 + t);
  double fmi[4], det;
  if (g.morph) {
    const double* mo = g.morph + (size_t)inst * 5 * nq;
#pragma unroll
    for (int t = 0; t < 4; ++t) fmi[t] = __ldg(mo + (size_t)t * nq + q);
    det = __ldg(mo + (size_t)4 * nq + q);
  } else {
    const double ka = __ldg(g.geom + 2 * inst) / g.r0 - 1.0;
    const double kb = __ldg(g.geom + 2 * inst + 1) / g.r0 - 1.0;
    double d[4][2];
#pragma unroll
    for (int a = 0; a < 4; ++a) {
      const int nd = __ldg(g.elems + 4 * e + a);
      morph_d(__ldg(g.nodes + 2 * nd), __ldg(g.nodes + 2 * nd + 1), ka, kb, g.r0, d[a][0], d[a][1]);
    }
    det = derive_qp(d, gq, fmi);
  }
  const double wq = __ldg(g.w + q) * det;
  double gt[4][2], P[4];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int j = 0; j < 2; ++j) gt[a][j] = gq[2 * a] * fmi[2 * j] + gq[2 * a + 1] * fmi[1 + 2 * j];
#pragma unroll
  for (int t = 0; t < 4; ++t) P[t] = g.field[((size_t)inst * 16 + t + 4 * g.field_col) * nq + q];
  double v[8], o[2];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int i = 0; i < 2; ++i) v[a * 2 + i] = wq * (P[i] * gt[a][0] + P[i + 2] * gt[a][1]);
  quad_reduce8(v, k, o);
  if (valid) {
    double* sc = g.scratch + (size_t)c * g.n_groups;
    const int32_t* ps = g.pos + (size_t)e * 72;
    const int u0 = 4 * (k & 1) + 2 * ((k >> 1) & 1);
    const int p0 = __ldg(ps + 64 + u0), p1 = __ldg(ps + 64 + u0 + 1);
    if (p0 >= 0) sc[p0] = o[0];
    if (p1 >= 0) sc[p1] = o[1];
  }
}

struct GatherArgs {
  int n_red, n_elems;
  int64_t nnz;
  int64_t inst0;
  int n_inst;
  const int32_t* slot_gptr;
  const int32_t* slot_grp;
  const int32_t* frow_gptr;
  const int32_t* frow_grp;
  const double* scratch;
  double* f;
  double* kvals;
};

// One thread per (instance, item): items [0, nnz) are CSR slots (if kvals),
// items [nnz, nnz + n_red) residual rows.
__global__ void __launch_bounds__(256) k_asm_gather(GatherArgs g) {
  const int64_t n_items = (g.kvals ? g.nnz : 0) + g.n_red;
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (tid >= n_items * g.n_inst) return;
  const int c = (int)(tid / n_items);
  const int64_t it = tid - (int64_t)c * n_items;
  const double* sc = g.scratch + (size_t)c * g.n_elems * 72 * 4;
  const int64_t inst = g.inst0 + c;
  if (g.kvals && it < g.nnz) {
    const int b0 = __ldg(g.slot_gptr + it), b1 = __ldg(g.slot_gptr + it + 1);
    double s = 0.0;
    for (int m = b0; m < b1; ++m) {
      const int grp = __ldg(g.slot_grp + m);  // e*64 + tl
      const int e = grp >> 6, tl = grp & 63;
      const double4 t = *reinterpret_cast<const double4*>(sc + ((size_t)e * 72 + tl) * 4);
      if (m == b0) {
        s = t.x;  // setFromTriplets: first duplicate is copied, the rest added
      } else {
        s = s + t.x;
      }
      s = s + t.y;
      s = s + t.z;
      s = s + t.w;
    }
    g.kvals[(size_t)inst * g.nnz + it] = s;
  } else {
    const int64_t row = it - (g.kvals ? g.nnz : 0);
    const int b0 = __ldg(g.frow_gptr + row), b1 = __ldg(g.frow_gptr + row + 1);
    double s = 0.0;  // out.f = VecX::Zero(...); f(ra+i) += ...
    for (int m = b0; m < b1; ++m) {
      const int grp = __ldg(g.frow_grp + m);  // e*8 + fl
      const int e = grp >> 3, fl = grp & 7;
      const double4 t = *reinterpret_cast<const double4*>(sc + ((size_t)e * 72 + 64 + fl) * 4);
      s = s + t.x;
      s = s + t.y;
      s = s + t.z;
      s = s + t.w;
    }
    g.f[(size_t)inst * g.n_red + row] = s;
  }
}

// Default gather: the element sums already sit in slot order, so every CSR
// slot / residual row is a contiguous run scratch[gptr[i] .. gptr[i+1]) summed
// in element order (first term copied for K, setFromTriplets style; 0 + ...
// for f).  One thread per (instance, item): a streaming segmented reduction.
__global__ void __launch_bounds__(256) k_asm_gather_fused(GatherArgs g, const int32_t* __restrict__ gptr,
                                                          int64_t n_groups) {
  // grid: x over items (slots then rows), y over the chunk's instances
  const int n_items = (int)((g.kvals ? g.nnz : 0) + g.n_red);
  const int it = blockIdx.x * blockDim.x + threadIdx.x;
  if (it >= n_items) return;
  const int c = blockIdx.y;
  const int nnz = g.kvals ? (int)g.nnz : 0;
  const bool is_slot = it < nnz;
  const int gi = g.kvals ? it : it + (int)g.nnz;  // index into gptr (slots then rows)
  const int b0 = __ldg(gptr + gi), b1 = __ldg(gptr + gi + 1);
  const double* sc = g.scratch + (size_t)c * n_groups;
  // runs hold 1-4 element sums on the Q4 cell: all four loads are issued
  // before the (ordered) additions, so a thread keeps up to 4 in flight
  const int n = b1 - b0;
  const double v0 = n > 0 ? __ldcs(sc + b0) : 0.0;
  const double v1 = n > 1 ? __ldcs(sc + b0 + 1) : 0.0;
  const double v2 = n > 2 ? __ldcs(sc + b0 + 2) : 0.0;
  const double v3 = n > 3 ? __ldcs(sc + b0 + 3) : 0.0;
  double sm = v0;
  if (!is_slot) sm = 0.0 + sm;
  if (n > 1) sm = sm + v1;
  if (n > 2) sm = sm + v2;
  if (n > 3) sm = sm + v3;
  for (int m = b0 + 4; m < b1; ++m) sm = sm + __ldcs(sc + m);
  const int64_t inst = g.inst0 + c;
  if (is_slot)
    g.kvals[(size_t)inst * g.nnz + it] = sm;
  else
    g.f[(size_t)inst * g.n_red + (it - nnz)] = sm;
}

// Tiled mode: the halo items only (items [0, nnz) CSR slots, then residual
// rows), each a contiguous run of the compact scratch, summed in group order.
__global__ void __launch_bounds__(256) k_asm_gather_halo(GatherArgs g, const int32_t* __restrict__ hitem,
                                                         const int32_t* __restrict__ hgptr, int n_halo,
                                                         int64_t n_hgroups) {
  const int h = blockIdx.x * blockDim.x + threadIdx.x;
  if (h >= n_halo) return;
  const int it = __ldg(hitem + h);
  const bool is_slot = it < g.nnz;
  if (is_slot && !g.kvals) return;
  const int c = blockIdx.y;
  const int b0 = __ldg(hgptr + h), b1 = __ldg(hgptr + h + 1);
  const double* sc = g.scratch + (size_t)c * n_hgroups;
  const int n = b1 - b0;
  const double v0 = n > 0 ? __ldcs(sc + b0) : 0.0;
  const double v1 = n > 1 ? __ldcs(sc + b0 + 1) : 0.0;
  const double v2 = n > 2 ? __ldcs(sc + b0 + 2) : 0.0;
  const double v3 = n > 3 ? __ldcs(sc + b0 + 3) : 0.0;
  double sm = v0;
  if (!is_slot) sm = 0.0 + sm;
  if (n > 1) sm = sm + v1;
  if (n > 2) sm = sm + v2;
  if (n > 3) sm = sm + v3;
  for (int m = b0 + 4; m < b1; ++m) sm = sm + __ldcs(sc + m);
  const int64_t inst = g.inst0 + c;
  if (is_slot)
    g.kvals[(size_t)inst * g.nnz + it] = sm;
  else
    g.f[(size_t)inst * g.n_red + (it - g.nnz)] = sm;
}

__global__ void k_morph(int64_t n_inst, int nq, double r0, const double* nodes, const int32_t* elems,
                        const double* grad, const double* geom, double* fmu_inv, double* det,
                        int32_t* status, unsigned int* fail) {
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (tid >= n_inst * nq) return;
  const int64_t inst = tid / nq;
  const int q = (int)(tid - inst * nq);
  const int e = q >> 2;
  const double ka = geom[2 * inst] / r0 - 1.0, kb = geom[2 * inst + 1] / r0 - 1.0;
  double d[4][2], gq[8], fmi[4];
  for (int t = 0; t < 8; ++t) gq[t] = grad[(size_t)q * 8 + t];
  for (int a = 0; a < 4; ++a) {
    const int nd = elems[4 * e + a];
    morph_d(nodes[2 * nd], nodes[2 * nd + 1], ka, kb, r0, d[a][0], d[a][1]);
  }
  const double dt = derive_qp(d, gq, fmi);
  for (int t = 0; t < 4; ++t) fmu_inv[(size_t)inst * 4 * nq + (size_t)t * nq + q] = fmi[t];
  det[(size_t)inst * nq + q] = dt;
  if (!(dt > 0.0)) {
    if (status) status[inst] = PODECM_ESOLVE;
    atomicAdd(fail, 1u);
  }
}

}  // namespace

namespace podecm_impl {

// field != nullptr: field-rows mode (f = residual-row sums of the stored
// tangent field's column field_col, see k_asm_field_terms); else the assembly.
int assemble_impl(podecm_ctx* ctx, void* stream, podecm_rve* r, int64_t n_inst, const double* geom,
                  const double* morph, const double* fbar, const double* w_red, const double* st0, double* st1,
                  double* f, double* kvals, double* p_field, int32_t* status, double* a_field,
                  const double* field, int field_col) {
  if (!ctx || !r) return PODECM_ECONFIG;
  if (n_inst < 0) return set_err(ctx, PODECM_ECONFIG, "negative instance count");
  if (n_inst == 0) return PODECM_OK;
  if ((!geom && !morph) || !f || (!field && (!fbar || !w_red || !st0)))
    return set_err(ctx, PODECM_ECONFIG, "geom|morph, fbar, w_red, st0 and f are required");
  auto s = static_cast<cudaStream_t>(stream);
  // exact triplet-order mode, read per call (tests/test_gpu_assembly.py runs
  // both modes in one process)
  const bool exact_env = [] {
    const char* e = getenv("PODECM_ASM_EXACT");
    return e && atoi(e) != 0;
  }();
  const bool exact = exact_env && !field;
  if (field) kvals = nullptr;
  static const int minb = [] {
    const char* e = getenv("PODECM_ASM_MINB");
    return e ? atoi(e) : 4;
  }();
  // tiled assembly (default where the cell divides into 8 x 4 element tiles;
  // PODECM_ASM_TILED=0: the per-qp grid with every element sum gathered)
  const bool tiled = !exact && !field && r->n_tiles > 0 && [] {
    const char* e = getenv("PODECM_ASM_TILED");
    return !(e && atoi(e) == 0);
  }();
  const size_t per_inst =
      (exact ? (size_t)r->n_elems * 72 * 4 : (size_t)(tiled ? r->n_hgroups : r->n_groups)) * sizeof(double);
  // Chunk of instances per (qp kernel, gather) pair: the scratch budget
  // (PODECM_ASM_CHUNK_MB, default 768 MB; 81 instances of 128^2).  Large grids
  // beat L2 residency here: 48 MB chunks (5 instances, 3.5 waves of the qp
  // kernel) cost 36 ms per C2 step against 30 ms at 768 MB.
  static const int64_t chunk_mb = [] {
    const char* e = getenv("PODECM_ASM_CHUNK_MB");
    return (int64_t)(e ? std::max(1, atoi(e)) : 768);
  }();
  int64_t chunk = std::max<int64_t>(1, (chunk_mb << 20) / (int64_t)per_inst);
  chunk = std::min<int64_t>(chunk, n_inst);
  // scratch_inst counts BYTES: the modes have different per-instance
  // footprints and may alternate on one cell
  if (r->scratch_inst < (int64_t)per_inst * chunk) {
    cudaFree(r->d_scratch);
    r->d_scratch = nullptr;
    PODECM_CUDA_TRY(ctx, cudaMalloc(&r->d_scratch, per_inst * chunk));
    r->scratch_inst = (int64_t)per_inst * chunk;
  }
  if (status && !field) PODECM_CUDA_TRY(ctx, cudaMemsetAsync(status, 0, n_inst * sizeof(int32_t), s));
  for (int64_t i0 = 0; i0 < n_inst; i0 += chunk) {
    const int nc = (int)std::min<int64_t>(chunk, n_inst - i0);
    double* scratch = r->d_scratch;
    AsmArgs a;
    a.n_qp = r->n_qp;
    a.n_red = r->n_red;
    a.nnz = r->nnz;
    a.inst0 = i0;
    a.n_inst = nc;
    a.r0 = r->r0;
    a.nodes = r->d_nodes;
    a.elems = r->d_elems;
    a.regions = r->d_regions;
    a.grad = r->d_grad;
    a.w = r->d_w;
    a.node_dof = r->d_node_dof;
    a.geom = geom;
    a.morph = morph;
    a.fbar = fbar;
    a.w_red = w_red;
    a.st0 = st0;
    a.st1 = st1;
    a.p_field = p_field;
    a.scratch = scratch;
    a.pos = r->d_pos;
    a.n_groups = r->n_groups;
    a.status = status;
    a.fail = ctx->d_fail;
    a.tangent = kvals != nullptr;
    a.a_field = a_field;
    a.field = field;
    a.field_col = field_col;
    a.t_elem = r->d_t_elem;
    a.t_lptr = r->d_t_lptr;
    a.t_litem = r->d_t_litem;
    a.t_lpack = r->d_t_lpack;
    a.t_hpos = r->d_t_hpos;
    a.kvals = kvals;
    a.f = f;
    if (tiled) a.n_groups = r->n_hgroups;
    const int64_t nthr = (int64_t)nc * r->n_qp;
    if (tiled) {
      KTimer kt(ctx, s, "k_asm_qp2t");
      if (minb == 5)
        k_asm_qp2<5, true><<<dim3(r->n_tiles, nc), kQ2Thr, 0, s>>>(a, r->mats);
      else
        k_asm_qp2<4, true><<<dim3(r->n_tiles, nc), kQ2Thr, 0, s>>>(a, r->mats);
    } else if (field) {
      KTimer kt(ctx, s, "k_asm_field_terms");
      k_asm_field_terms<<<grid_for(nthr, 256), 256, 0, s>>>(a);
    } else if (exact) {
      KTimer kt(ctx, s, "k_asm_qp");
      k_asm_qp<5><<<grid_for(nthr, 128), 128, 0, s>>>(a, r->mats);
    } else {
      KTimer kt(ctx, s, "k_asm_qp2");
      if (minb == 5)
        k_asm_qp2<5><<<grid_for(nthr, kQ2Thr), kQ2Thr, 0, s>>>(a, r->mats);
      else
        k_asm_qp2<4><<<grid_for(nthr, kQ2Thr), kQ2Thr, 0, s>>>(a, r->mats);
    }
    GatherArgs gg;
    gg.n_red = r->n_red;
    gg.n_elems = r->n_elems;
    gg.nnz = r->nnz;
    gg.inst0 = i0;
    gg.n_inst = nc;
    gg.slot_gptr = r->d_slot_gptr;
    gg.slot_grp = r->d_slot_grp;
    gg.frow_gptr = r->d_frow_gptr;
    gg.frow_grp = r->d_frow_grp;
    gg.scratch = scratch;
    gg.f = f;
    gg.kvals = kvals;
    const int64_t nitems = ((kvals ? r->nnz : 0) + r->n_red) * nc;
    cudaStream_t gs = s;
    {
      KTimer kt(ctx, gs, "k_asm_gather");
      if (tiled) {
        const int nh = (int)r->t_hitem.size();
        k_asm_gather_halo<<<dim3(grid_for(nh, 256), nc), 256, 0, gs>>>(gg, r->d_t_hitem, r->d_t_hgptr, nh,
                                                                       r->n_hgroups);
      } else if (exact) {
        k_asm_gather<<<grid_for(nitems, 256), 256, 0, gs>>>(gg);
      } else {
        k_asm_gather_fused<<<dim3(grid_for(nitems / nc, 256), nc), 256, 0, gs>>>(gg, r->d_gptr_all, r->n_groups);
      }
    }
    PODECM_LAUNCHED(ctx, 2);
  }
  return PODECM_OK;
}


int assemble_field_rows(podecm_ctx* ctx, cudaStream_t s, podecm_rve* r, int64_t n, const double* geom,
                        const double* morph, const double* field, int col, double* out) {
  return assemble_impl(ctx, s, r, n, geom, morph, nullptr, nullptr, nullptr, nullptr, out, nullptr, nullptr,
                       nullptr, nullptr, field, col);
}

}  // namespace podecm_impl

extern "C" {

int podecm_rve_morph(podecm_ctx* ctx, void* stream, podecm_rve* r, int64_t n_inst,
                     const double* geom, double* fmu_inv, double* det, int32_t* status) {
  if (!ctx || !r || !geom || !fmu_inv || !det) return set_err(ctx, PODECM_ECONFIG, "null argument");
  if (n_inst <= 0) return PODECM_OK;
  auto s = static_cast<cudaStream_t>(stream);
  if (status) PODECM_CUDA_TRY(ctx, cudaMemsetAsync(status, 0, n_inst * sizeof(int32_t), s));
  const int64_t total = n_inst * r->n_qp;
  k_morph<<<grid_for(total, 256), 256, 0, s>>>(n_inst, r->n_qp, r->r0, r->d_nodes, r->d_elems,
                                               r->d_grad, geom, fmu_inv, det, status, ctx->d_fail);
  PODECM_LAUNCHED(ctx, 1);
  return PODECM_OK;
}

int podecm_assemble_batch(podecm_ctx* ctx, void* stream, podecm_rve* r, int64_t n_inst,
                          const double* geom, const double* morph, const double* fbar,
                          const double* w_red, const double* st0, double* st1, double* f,
                          double* kvals, double* p_field, int32_t* status) {
  return assemble_impl(ctx, stream, r, n_inst, geom, morph, fbar, w_red, st0, st1, f, kvals, p_field, status,
                       nullptr, nullptr, 0);
}

int podecm_assemble_batch_ex(podecm_ctx* ctx, void* stream, podecm_rve* r, int64_t n_inst,
                             const double* geom, const double* morph, const double* fbar,
                             const double* w_red, const double* st0, double* st1, double* f,
                             double* kvals, double* p_field, int32_t* status, double* a_field) {
  if (a_field && !kvals) return set_err(ctx, PODECM_ECONFIG, "a_field requires the tangent (kvals)");
  return assemble_impl(ctx, stream, r, n_inst, geom, morph, fbar, w_red, st0, st1, f, kvals, p_field, status,
                       a_field, nullptr, 0);
}

}  // extern "C"
