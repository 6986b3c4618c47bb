// K4b — Empirical Cubature Method greedy selection (BASELINE config 4).
//
// Replaces weighted_stress_field / ecm_integrand / ecm_select /
// restore_feasible (/root/reference/proj/src/ecm.cpp:10-204) without ever
// materialising the integrand J ((N L + 1) x n_qp, 105 GB at config 4): J is
// kept factored as J[(i,s), q] = sum_c H[q][i][c] W[s][q][c] (mode gradient
// x weighted stress snapshot) plus the all-ones volume row.
//
//   k_ecm_mode_grads   H[q][i][c] (build_rom's formula at every qp)
//   k_ecm_stress       W[s][q][c]: stress-only material update of snapshot s
//                      (virgin history, identity morph => W = P)
//   k_ecm_colnorm      ||J_q||^2 = sum_cd (H_q^T H_q)_cd (W_q^T W_q)_cd + 1
//   k_ecm_score        corr = J^T r as one DMMA GEMM T = R W (R = r reshaped
//                      N x L) fused with the H contraction, the score
//                      corr/||J_q|| and a per-CTA argmax (strict '>', first
//                      index wins, positive scores only: ecm.cpp:164-173)
//   refit              least squares on the selected columns by an
//                      incrementally updated QR (classical Gram-Schmidt with
//                      re-orthogonalisation); the Lawson-Hanson feasibility
//                      steps of restore_feasible (ecm.cpp:56-90) run on the
//                      host over k <= max_points weights; a drop rebuilds the
//                      QR of the kept set.
#include <algorithm>
#include <cmath>
#include <numeric>
#include <unordered_map>
#include <utility>
#include <vector>

#include "rve.cuh"
#include "dmma_gemm.cuh"

using namespace podecm_dev;
using namespace podecm_impl;

namespace {

__global__ void k_ecm_mode_grads(int nq, int N, int64_t ndof, const int32_t* elems,
                                 const double* grad, const double* modes, double* H) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (int64_t)nq * N) return;
  const int q = (int)(t / N), i = (int)(t - (int64_t)q * N);
  const int e = q >> 2;
  double h[4] = {0.0, 0.0, 0.0, 0.0};  // h(0,0), h(1,0), h(0,1), h(1,1)
  for (int a = 0; a < 4; ++a) {
    const int node = elems[4 * e + a];
    const double ux = modes[(int64_t)i * ndof + 2 * node], uy = modes[(int64_t)i * ndof + 2 * node + 1];
    const double g0 = grad[(size_t)q * 8 + 2 * a], g1 = grad[(size_t)q * 8 + 2 * a + 1];
    h[0] = h[0] + ux * g0;  // h.row(0) += u_x g.row(a)  (rom.cpp:96-100)
    h[2] = h[2] + ux * g1;
    h[1] = h[1] + uy * g0;
    h[3] = h[3] + uy * g1;
  }
  for (int c = 0; c < 4; ++c) H[((int64_t)q * N + i) * 4 + c] = h[c];
}

__global__ void __launch_bounds__(128, 5) k_ecm_stress(int64_t L, int nq, int64_t ndof,
                                                        const int32_t* elems, const int32_t* regions,
                                                        const double* grad, const double* U,
                                                        MatTable tab, double* W, int32_t* status,
                                                        unsigned int* fail) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= L * nq) return;
  const int64_t s = t / nq;
  const int q = (int)(t - s * nq);
  const int e = q >> 2;
  double gw[4] = {0.0, 0.0, 0.0, 0.0};
  for (int a = 0; a < 4; ++a) {
    const int node = elems[4 * e + a];
    const double ux = U[s * ndof + 2 * node], uy = U[s * ndof + 2 * node + 1];
    const double g0 = grad[(size_t)q * 8 + 2 * a], g1 = grad[(size_t)q * 8 + 2 * a + 1];
    gw[0] = gw[0] + ux * g0;
    gw[2] = gw[2] + ux * g1;
    gw[1] = gw[1] + uy * g0;
    gw[3] = gw[3] + uy * g1;
  }
  // F = I + gw * I (identity morph, microfem.cpp:87)
  double F[4];
  F[0] = 1.0 + (gw[0] * 1.0 + gw[2] * 0.0);
  F[1] = 0.0 + (gw[1] * 1.0 + gw[3] * 0.0);
  F[2] = 0.0 + (gw[0] * 0.0 + gw[2] * 1.0);
  F[3] = 1.0 + (gw[1] * 0.0 + gw[3] * 1.0);
  const double fp[4] = {1.0, 0.0, 0.0, 1.0};
  Frozen z;
  freeze(fp, 1.0, 0.0, z);
  double P[4];
  const bool ok = lsu_eval<false>(tab.m[regions[e]], z, F, P, nullptr);
  // W = P Fmu^-T det = P for the identity morph (ecm.cpp:10-18)
  double* w = W + (s * nq + q) * 4;
  for (int c = 0; c < 4; ++c) w[c] = P[c];
  if (!ok) {
    if (status) status[0] = PODECM_ESOLVE;
    atomicAdd(fail, 1u);
  }
}

// sum_{i,s} J[(i,s),q]^2 + vol via the 4x4 Gram factorisation
__global__ void k_ecm_colnorm(int64_t L, int nq, int N, const double* H, const double* W, int vol,
                              double* cn) {
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= nq) return;
  double ww[10] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
  for (int64_t s = 0; s < L; ++s) {
    const double4 v = *reinterpret_cast<const double4*>(W + (s * nq + q) * 4);
    const double a[4] = {v.x, v.y, v.z, v.w};
    int k = 0;
    for (int c = 0; c < 4; ++c)
      for (int d = c; d < 4; ++d, ++k) ww[k] = fma(a[c], a[d], ww[k]);
  }
  double hh[10] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
  for (int i = 0; i < N; ++i) {
    const double* h = H + ((int64_t)q * N + i) * 4;
    int k = 0;
    for (int c = 0; c < 4; ++c)
      for (int d = c; d < 4; ++d, ++k) hh[k] = fma(h[c], h[d], hh[k]);
  }
  double ssum = 0.0;
  int k = 0;
  for (int c = 0; c < 4; ++c)
    for (int d = c; d < 4; ++d, ++k) ssum += (c == d ? 1.0 : 2.0) * hh[k] * ww[k];
  cn[q] = sqrt(fmax(ssum, 0.0) + (vol ? 1.0 : 0.0));
}

// corr_q = sum_{i,s,c} r[i L + s] H[q][i][c] W[s][q][c] + r_vol, score, CTA argmax.
// CTA: 16 qps (64 columns of T), 7 warps x 8 rows (N <= 56), K-loop over s.
constexpr int kSQ = 16, kSC = 64, kSK = 16, kSLD = kSK + 4;

// Bases wider than 56 modes run in row blocks: N rows of r starting at the
// block, H rows strided by ldH, and corr_out accumulated (accumulate != 0).
__global__ void __launch_bounds__(224) k_ecm_score(int64_t L, int nq, int N, const double* r,
                                                   const double* r_vol_p, const double* H, const double* W,
                                                   const double* cn, const uint8_t* unavailable,
                                                   double* cta_best, int* cta_idx, double* corr_out, int ldH,
                                                   int accumulate) {
  __shared__ double sR[2][56][kSLD];
  __shared__ double sW[2][kSC][kSLD];
  __shared__ double red[7][kSQ];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int gid = lane >> 2, tig = lane & 3;
  const int q0 = blockIdx.x * kSQ;
  double acc[8][2];
#pragma unroll
  for (int ct = 0; ct < 8; ++ct) acc[ct][0] = acc[ct][1] = 0.0;
  auto load = [&](int buf, int64_t s0) {
    for (int t = tid; t < 56 * kSK; t += blockDim.x) {
      const int i = t / kSK, k = t % kSK;
      const int64_t s = s0 + k;
      sR[buf][i][k] = (i < N && s < L) ? r[(int64_t)i * L + s] : 0.0;
    }
    for (int t = tid; t < kSK * kSC; t += blockDim.x) {
      const int k = t / kSC, col = t % kSC;
      const int64_t s = s0 + k;
      const int q = q0 + col / 4;
      sW[buf][col][k] = (s < L && q < nq) ? W[(s * nq + q0) * 4 + col] : 0.0;
    }
  };
  const int64_t nk = (L + kSK - 1) / kSK;
  load(0, 0);
  __syncthreads();
  for (int64_t kt = 0; kt < nk; ++kt) {
    const int buf = (int)(kt & 1);
    if (kt + 1 < nk) load(buf ^ 1, (kt + 1) * kSK);
#pragma unroll
    for (int kk = 0; kk < kSK / 4; ++kk) {
      const double af = sR[buf][warp * 8 + gid][kk * 4 + tig];
#pragma unroll
      for (int ct = 0; ct < 8; ++ct) dmma884(acc[ct][0], acc[ct][1], af, sW[buf][ct * 8 + gid][kk * 4 + tig]);
    }
    __syncthreads();
  }
  // epilogue: thread holds T[i][col], i = 8 warp + gid, col = 8 ct + 2 tig + h
  const int i = warp * 8 + gid;
  double part[8];
#pragma unroll
  for (int ct = 0; ct < 8; ++ct) {
    const int ql = 2 * ct + (tig >> 1);
    const int q = q0 + ql;
    double v = 0.0;
    if (i < N && q < nq) {
      const double* h = H + ((int64_t)q * ldH + i) * 4;
      const int c0 = 2 * (tig & 1);
      v = h[c0] * acc[ct][0] + h[c0 + 1] * acc[ct][1];
    }
    // reduce over gid (rows) and tig&1 (c pairs): lanes sharing tig>>1
#pragma unroll
    for (int o = 4; o < 32; o <<= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    v += __shfl_xor_sync(0xffffffffu, v, 1);
    part[ct] = v;
  }
  if (gid == 0 && (tig & 1) == 0)
#pragma unroll
    for (int ct = 0; ct < 8; ++ct) red[warp][2 * ct + (tig >> 1)] = part[ct];
  __syncthreads();
  if (tid < kSQ) {
    const int q = q0 + tid;
    double best = 0.0;
    int bi = -1;
    if (q < nq && !unavailable[q] && cn[q] != 0.0) {
      double corr = 0.0;
      for (int w = 0; w < 7; ++w) corr += red[w][tid];
      if (r_vol_p) corr += *r_vol_p;
      if (corr_out) corr_out[q] = accumulate ? corr_out[q] + corr : corr;
      const double sc = corr / cn[q];
      if (sc > 0.0) {
        best = sc;
        bi = q;
      }
    }
    // CTA argmax: larger score wins, ties -> smaller index
    for (int o = 8; o > 0; o >>= 1) {
      const double ob = __shfl_down_sync(0x0000ffffu, best, o, 16);
      const int oi = __shfl_down_sync(0x0000ffffu, bi, o, 16);
      if (oi >= 0 && (bi < 0 || ob > best || (ob == best && oi < bi))) {
        best = ob;
        bi = oi;
      }
    }
    if (tid == 0) {
      cta_best[blockIdx.x] = best;
      cta_idx[blockIdx.x] = bi;
    }
  }
}


// Gram-updated scoring.  With r = rhs - J_sel x,
//   corr = J^T r = J^T rhs - sum_k x_k (J^T J_{s_k}),
// and column s of J^T J factors through the 4x4 blocks of the integrand:
//   (J^T J)[q, s] = sum_{c,d} (H_q^T H_s)[c,d] (W_q^T W_s)[c,d] + vol,
// H_q = H[q] (N x 4), W_q = W[:, q, :] (L x 4).  One new column per selected
// point costs one streaming pass over W with 16 FMAs per 32 bytes (HBM-bound)
// instead of the N L 4 n_qp DMMA GEMM of a direct J^T r pass.
constexpr int kGramSplit = 4;  // L-range splits (partials summed in fixed order)

// Gram columns (J^T J)[:, sel_c] for C <= kGramCols selected / speculative
// points in ONE pass over W, on the FP64 tensor cores.  For a block of 64
// candidates the 4x4 blocks mw(q, c) = sum_l W_q[l] W_sel_c[l]^T are one
// DMMA GEMM: rows (q, c') of W^T (the W stream, each element loaded once,
// 64 B runs), columns (c, d) of the staged selected rows, K = the snapshots
// of this split.  An m8n8k4 f64 DMMA accumulates every element as the
// sequential FMA chain over k, so mw is bit-identical to the scalar
// fma(W_q[c'], W_sel[d], .) loop in snapshot order; mh (over the modes) and
// g = sum_t fma(mh[t], mw[t], .) are then formed per (candidate, column)
// exactly as in the single-column form.  Each column is therefore the value
// a one-column pass produces.
constexpr int kGramCols = 4;
constexpr int kGramLC = 64;  // snapshots staged per round (multiple of 4)
template <int C>
__global__ void __launch_bounds__(256) k_ecm_gram_cols(int64_t L, int nq, int N, const int* __restrict__ sels,
                                                       const double* H, const double* W, double* gpart) {
  constexpr int NT = (C + 1) / 2;  // n-tiles: 2 columns x 4 components each
  constexpr int MT = 4;            // m-tiles per warp: 4 x 8 rows = 8 candidates
  __shared__ double sw[kGramLC][NT * 8 + 1];  // staged W_sel rows, column n = 4 c + d
  __shared__ double se[64][C][17];            // mw of every (candidate, column)
  __shared__ int ssel[C];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int gid = lane >> 2, tig = lane & 3;
  const int q0 = blockIdx.x * 64;
  const int sp = blockIdx.y;
  const int64_t l0 = L * sp / kGramSplit, l1 = L * (sp + 1) / kGramSplit;
  if (threadIdx.x < C) ssel[threadIdx.x] = sels[threadIdx.x];
  double acc[MT][NT][2];
#pragma unroll
  for (int mt = 0; mt < MT; ++mt)
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) acc[mt][nt][0] = acc[mt][nt][1] = 0.0;
  // A fragment rows: (q, c') = row r of the warp's 32 rows; W^T[(q, c')][l] = W[l][q][c']
  const int64_t rowbase = (int64_t)(q0 + warp * 8) * 4;  // first (q, c') row of the warp
  const int64_t nrow = (int64_t)nq * 4;
  for (int64_t lb = l0; lb < l1; lb += kGramLC) {
    const int nl = (int)((l1 - lb) < kGramLC ? (l1 - lb) : kGramLC);
    __syncthreads();
    for (int t = threadIdx.x; t < kGramLC * NT * 8; t += 256) {
      const int lc = t / (NT * 8), n = t - lc * (NT * 8), c = n >> 2, d = n & 3;
      sw[lc][n] = (lc < nl && c < C) ? __ldg(W + ((lb + lc) * nq + ssel[c]) * 4 + d) : 0.0;
    }
    __syncthreads();
#pragma unroll 4
    for (int k0 = 0; k0 < nl; k0 += 4) {
      const int lk = k0 + tig;  // this thread's k (snapshot) of the step
      const bool kin = lk < nl;
      double a[MT], b[NT];
#pragma unroll
      for (int mt = 0; mt < MT; ++mt) {
        const int64_t row = rowbase + mt * 8 + gid;
        a[mt] = (kin && row < nrow) ? __ldcs(W + (lb + lk) * nrow + row) : 0.0;
      }
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) b[nt] = sw[lk < kGramLC ? lk : 0][nt * 8 + gid];
#pragma unroll
      for (int mt = 0; mt < MT; ++mt)
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) dmma884(acc[mt][nt][0], acc[mt][nt][1], a[mt], kin ? b[nt] : 0.0);
    }
  }
  // acc[mt][nt][h]: row (q, c') = warp*32 + mt*8 + gid, column n = nt*8 + 2 tig + h = 4 c + d
#pragma unroll
  for (int mt = 0; mt < MT; ++mt)
#pragma unroll
    for (int nt = 0; nt < NT; ++nt)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int r = warp * 32 + mt * 8 + gid, n = nt * 8 + 2 * tig + h, c = n >> 2, d = n & 3;
        if (c < C) se[r >> 2][c][(r & 3) * 4 + d] = acc[mt][nt][h];
      }
  __syncthreads();
  for (int t = threadIdx.x; t < 64 * C; t += 256) {
    const int ql = t / C, c = t - ql * C, q = q0 + ql;
    if (q >= nq) continue;
    const int sel = ssel[c];
    double mh[16];
#pragma unroll
    for (int u = 0; u < 16; ++u) mh[u] = 0.0;
    for (int i = 0; i < N; ++i) {
      const double* hq = H + ((int64_t)q * N + i) * 4;
      const double* hs = H + ((int64_t)sel * N + i) * 4;
      const double av[4] = {hq[0], hq[1], hq[2], hq[3]};
      const double bv[4] = {__ldg(hs), __ldg(hs + 1), __ldg(hs + 2), __ldg(hs + 3)};
#pragma unroll
      for (int cc = 0; cc < 4; ++cc)
#pragma unroll
        for (int d = 0; d < 4; ++d) mh[cc * 4 + d] = fma(av[cc], bv[d], mh[cc * 4 + d]);
    }
    double g = 0.0;
#pragma unroll
    for (int u = 0; u < 16; ++u) g = fma(mh[u], se[ql][c][u], g);
    gpart[((int64_t)c * kGramSplit + sp) * nq + q] = g;
  }
}

template <int... I>
void launch_gram_cols(int C, dim3 grid, cudaStream_t s, int64_t L, int nq, int N, const int* sels, const double* H,
                      const double* W, double* gpart, std::integer_sequence<int, I...>) {
  (..., (C == I + 1 ? (void)k_ecm_gram_cols<I + 1><<<grid, 256, 0, s>>>(L, nq, N, sels, H, W, gpart) : (void)0));
}

// G[k][q] = sum of the split partials (+ vol)
__global__ void k_ecm_gram_finish(int nq, const double* gpart, int vol, double* gcol) {
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= nq) return;
  double g = vol ? 1.0 : 0.0;
  for (int sp = 0; sp < kGramSplit; ++sp) g += gpart[(int64_t)sp * nq + q];
  gcol[q] = g;
}

// corr_q = c0_q - sum_k x_k G[k][q]; score = corr / ||J_q||; CTA argmax
__global__ void __launch_bounds__(256) k_ecm_score_gram(int nq, int k, const double* c0, const double* G,
                                                        const double* x, const double* cn,
                                                        const uint8_t* unavailable, double* cta_best,
                                                        int* cta_idx) {
  __shared__ double sb[256];
  __shared__ int si[256];
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  double best = 0.0;
  int bi = -1;
  if (q < nq && !unavailable[q] && cn[q] != 0.0) {
    double corr = c0[q];
    for (int j = 0; j < k; ++j) corr = fma(-x[j], G[(int64_t)j * nq + q], corr);
    const double sc = corr / cn[q];
    if (sc > 0.0) {
      best = sc;
      bi = q;
    }
  }
  sb[threadIdx.x] = best;
  si[threadIdx.x] = bi;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if (threadIdx.x < o) {
      const double ob = sb[threadIdx.x + o];
      const int oi = si[threadIdx.x + o];
      if (oi >= 0 && (si[threadIdx.x] < 0 || ob > sb[threadIdx.x] || (ob == sb[threadIdx.x] && oi < si[threadIdx.x]))) {
        sb[threadIdx.x] = ob;
        si[threadIdx.x] = oi;
      }
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    cta_best[blockIdx.x] = sb[0];
    cta_idx[blockIdx.x] = si[0];
  }
}

// Speculation set for the Gram columns: out[0] = the selected point, out[1..T]
// = the next best CTA winners of the same scoring pass (larger score, then
// smaller index; -1 where there is none).  Candidates only: whether they are
// selected later is decided by the exact scores of their own iteration.
__global__ void k_ecm_runners(int n, const double* best, const int* idx, const int* best_i, int T, int* out) {
  __shared__ double sb[1024];
  __shared__ int si[1024];
  __shared__ int picked[16];
  if (threadIdx.x == 0) picked[0] = *best_i;
  __syncthreads();
  for (int r = 1; r <= T; ++r) {
    double b = 0.0;
    int i = -1;
    for (int k = threadIdx.x; k < n; k += blockDim.x) {
      const int oi = idx[k];
      bool skip = oi < 0;
      for (int u = 0; u < r; ++u) skip = skip || oi == picked[u];
      const double ob = best[k];
      if (!skip && (i < 0 || ob > b || (ob == b && oi < i))) {
        b = ob;
        i = oi;
      }
    }
    sb[threadIdx.x] = b;
    si[threadIdx.x] = i;
    __syncthreads();
    for (int o = blockDim.x / 2; o > 0; o >>= 1) {
      if (threadIdx.x < o) {
        const double ob = sb[threadIdx.x + o];
        const int oi = si[threadIdx.x + o];
        if (oi >= 0 && (si[threadIdx.x] < 0 || ob > sb[threadIdx.x] || (ob == sb[threadIdx.x] && oi < si[threadIdx.x]))) {
          sb[threadIdx.x] = ob;
          si[threadIdx.x] = oi;
        }
      }
      __syncthreads();
    }
    if (threadIdx.x == 0) picked[r] = si[0];
    __syncthreads();
  }
  if (threadIdx.x <= T) out[threadIdx.x] = picked[threadIdx.x];
}

__global__ void k_ecm_argmax(int n, const double* best, const int* idx, double* out_b, int* out_i) {
  __shared__ double sb[1024];
  __shared__ int si[1024];
  double b = 0.0;
  int i = -1;
  for (int k = threadIdx.x; k < n; k += blockDim.x) {
    const int oi = idx[k];
    const double ob = best[k];
    if (oi >= 0 && (i < 0 || ob > b || (ob == b && oi < i))) {
      b = ob;
      i = oi;
    }
  }
  sb[threadIdx.x] = b;
  si[threadIdx.x] = i;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) {
      const double ob = sb[threadIdx.x + o];
      const int oi = si[threadIdx.x + o];
      if (oi >= 0 && (si[threadIdx.x] < 0 || ob > sb[threadIdx.x] || (ob == sb[threadIdx.x] && oi < si[threadIdx.x]))) {
        sb[threadIdx.x] = ob;
        si[threadIdx.x] = oi;
      }
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    *out_b = sb[0];
    *out_i = si[0];
  }
}

// column q of J: m = N L (+1) entries
__global__ void k_ecm_column(int64_t L, int nq, int N, int q, const double* H, const double* W, int vol,
                             double* col) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t m = (int64_t)N * L;
  if (t < m) {
    const int i = (int)(t / L);
    const int64_t s = t - (int64_t)i * L;
    const double* h = H + ((int64_t)q * N + i) * 4;
    const double* w = W + (s * nq + q) * 4;
    col[t] = h[0] * w[0] + h[1] * w[1] + h[2] * w[2] + h[3] * w[3];
  } else if (vol && t == m) {
    col[t] = 1.0;
  }
}

// v -= sum_j A[:,j] h[j]  (j < k)
__global__ void k_axpy_cols(int64_t m, int k, const double* A, const double* h, double* v) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= m) return;
  double s = v[r];
  int j = 0;
  for (; j + 8 <= k; j += 8) {  // 8 column loads in flight, FMAs in column order
    double a[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) a[u] = __ldcs(A + (int64_t)(j + u) * m + r);
#pragma unroll
    for (int u = 0; u < 8; ++u) s = fma(-a[u], __ldg(h + j + u), s);
  }
  for (; j < k; ++j) s = fma(-A[(int64_t)j * m + r], h[j], s);
  v[r] = s;
}

// out = b - sum_j A[:,j] x[j]; also per-CTA sum of squares and max |.|
__global__ void __launch_bounds__(256) k_resid(int64_t m, int k, const double* A, const double* x,
                                               const double* b, double* out, double* part_ss,
                                               double* part_max) {
  __shared__ double s1[256], s2[256];
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  double v = 0.0;
  if (r < m) {
    v = b[r];
    int j = 0;
    for (; j + 8 <= k; j += 8) {  // 8 column loads in flight, updates in column order
      double a[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) a[u] = __ldcs(A + (int64_t)(j + u) * m + r);
#pragma unroll
      for (int u = 0; u < 8; ++u) v = v - __ldg(x + j + u) * a[u];
    }
    for (; j < k; ++j) v = v - x[j] * A[(int64_t)j * m + r];
    out[r] = v;
  }
  s1[threadIdx.x] = v * v;
  s2[threadIdx.x] = fabs(v);
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if (threadIdx.x < o) {
      s1[threadIdx.x] += s1[threadIdx.x + o];
      s2[threadIdx.x] = fmax(s2[threadIdx.x], s2[threadIdx.x + o]);
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    part_ss[blockIdx.x] = s1[0];
    part_max[blockIdx.x] = s2[0];
  }
}



// Hw[i][(q,c)] = w_q H[q][i][c] (the full-quadrature weights folded into H)
__global__ void k_ecm_hw(int nq, int N, const double* H, const double* w, double* Hw) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (int64_t)nq * N * 4) return;
  const int c = (int)(t & 3);
  const int64_t qi = t >> 2;
  const int q = (int)(qi / N), i = (int)(qi - (int64_t)q * N);
  Hw[(int64_t)i * 4 * nq + (int64_t)q * 4 + c] = w[q] * H[t];
}

// Multi-CTA building blocks of the incremental QR (all reductions are
// two-stage with a fixed order: deterministic).
constexpr int kQrBlocks = 296;  // 2 CTAs per SM

// part[b][j] = sum over rows of slab b of A[j*m + r] v[r], j < k.  Each warp
// takes 4 columns at a time (4 independent accumulators, 5 loads in flight per
// lane per row step), lanes over rows; a fixed shuffle tree per column.
__global__ void __launch_bounds__(256) k_dots_part(int64_t m, int k, const double* A, const double* v,
                                                   double* part) {
  const int b = blockIdx.x, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t r0 = m * b / gridDim.x, r1 = m * (b + 1) / gridDim.x;
  for (int j0 = warp * 4; j0 < k; j0 += 32) {
    const int nj = min(4, k - j0);
    const double* a0 = A + (int64_t)j0 * m;
    const double* a1 = nj > 1 ? a0 + m : a0;
    const double* a2 = nj > 2 ? a0 + 2 * m : a0;
    const double* a3 = nj > 3 ? a0 + 3 * m : a0;
    double p0 = 0.0, p1 = 0.0, p2 = 0.0, p3 = 0.0;
#pragma unroll 4
    for (int64_t r = r0 + lane; r < r1; r += 32) {
      const double x = __ldg(v + r);
      p0 = fma(__ldcs(a0 + r), x, p0);
      p1 = fma(__ldcs(a1 + r), x, p1);
      p2 = fma(__ldcs(a2 + r), x, p2);
      p3 = fma(__ldcs(a3 + r), x, p3);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      p0 += __shfl_xor_sync(0xffffffffu, p0, o);
      p1 += __shfl_xor_sync(0xffffffffu, p1, o);
      p2 += __shfl_xor_sync(0xffffffffu, p2, o);
      p3 += __shfl_xor_sync(0xffffffffu, p3, o);
    }
    if (lane == 0) {
      double* out = part + (int64_t)b * k + j0;
      out[0] = p0;
      if (nj > 1) out[1] = p1;
      if (nj > 2) out[2] = p2;
      if (nj > 3) out[3] = p3;
    }
  }
}

// sum of x[b * stride], b < nb, by one warp: lanes stride b, fixed shuffle tree
__device__ __forceinline__ double warp_sum_strided(const double* x, int nb, int64_t stride, int lane) {
  double s = 0.0;
  for (int b = lane; b < nb; b += 32) s += x[(int64_t)b * stride];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  return s;
}

// out[j] = sum_b part[b][j] (one warp per column, fixed order)
__global__ void __launch_bounds__(256) k_dots_finish(int nb, int k, const double* part, double* out) {
  const int j = blockIdx.x * 8 + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (j >= k) return;
  const double s = warp_sum_strided(part + j, nb, k, lane);
  if (lane == 0) out[j] = s;
}

// part[b] = sum over slab b of x[r] y[r]
__global__ void __launch_bounds__(256) k_dot_part(int64_t m, const double* x, const double* y, double* part) {
  __shared__ double red[256];
  const int64_t r0 = m * blockIdx.x / gridDim.x, r1 = m * (blockIdx.x + 1) / gridDim.x;
  double p = 0.0;
  for (int64_t r = r0 + threadIdx.x; r < r1; r += blockDim.x) p = fma(x[r], y[r], p);
  red[threadIdx.x] = p;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) part[blockIdx.x] = red[0];
}

// R[:, k] = h1 + h2, r_kk = sqrt(sum part) (one thread block)
__global__ void k_qr_rcol(int nb, int k, int kmax, const double* part, const double* h1, const double* h2,
                          double* R) {
  for (int j = threadIdx.x; j < k; j += blockDim.x) R[(size_t)k * kmax + j] = (0.0 + h1[j]) + h2[j];
  if (threadIdx.x < 32) {
    const double s = warp_sum_strided(part, nb, 1, threadIdx.x);
    if (threadIdx.x == 0) R[(size_t)k * kmax + k] = sqrt(s);
  }
}

// qcol = v / r_kk; part[b] = sum over slab of qcol[r] rhs[r]
__global__ void __launch_bounds__(256) k_qr_scale_dot(int64_t m, const double* v, const double* rkk,
                                                      const double* rhs, double* qcol, double* part) {
  __shared__ double red[256];
  const double nrm = *rkk;
  const int64_t r0 = m * blockIdx.x / gridDim.x, r1 = m * (blockIdx.x + 1) / gridDim.x;
  double p = 0.0;
  for (int64_t r = r0 + threadIdx.x; r < r1; r += blockDim.x) {
    const double x = v[r] / nrm;
    qcol[r] = x;
    p = fma(x, rhs[r], p);
  }
  red[threadIdx.x] = p;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) part[blockIdx.x] = red[0];
}

__global__ void k_sum_to(int nb, const double* part, double* out) {
  const double s = warp_sum_strided(part, nb, 1, threadIdx.x);
  if (threadIdx.x == 0) *out = s;
}

// Incremental QR of the selected integrand columns (classical Gram-Schmidt
// with one re-orthogonalisation pass).  The m-long work (projections, norm,
// Q column, Q^T b) stays on the device; the new R column (k + 1 values) and
// qtb entry are copied to a host mirror, where the k x k back substitution
// and the Lawson-Hanson feasibility logic run (one sync per refit).
struct Ecm {
  podecm_ctx* ctx;
  cudaStream_t s;
  int64_t m;
  int kmax;
  double *Jsel, *Q, *tmp, *h1, *h2, *R, *qtb;
  const double* rhs;
  double* part;  // [kQrBlocks][kmax] partial sums
  int k = 0;
  double *hR, *hq;  // pinned host mirrors (column-major kmax x kmax, kmax)

  void append() {  // append column Jsel[:, k]
    double* v = tmp;
    cudaMemcpyAsync(v, Jsel + (int64_t)k * m, sizeof(double) * m, cudaMemcpyDeviceToDevice, s);
    if (k > 0) {
      for (int pass = 0; pass < 2; ++pass) {  // CGS2: project twice
        double* h = pass ? h2 : h1;
        {
          KTimer kt(ctx, s, "ecm_qr_dots");
          k_dots_part<<<kQrBlocks, 256, 0, s>>>(m, k, Q, v, part);
          k_dots_finish<<<grid_for(k, 8), 256, 0, s>>>(kQrBlocks, k, part, h);
        }
        KTimer kt(ctx, s, "ecm_qr_axpy");
        k_axpy_cols<<<grid_for(m, 256), 256, 0, s>>>(m, k, Q, h, v);
      }
    }
    KTimer kt(ctx, s, "ecm_qr_finish");
    k_dot_part<<<kQrBlocks, 256, 0, s>>>(m, v, v, part);
    k_qr_rcol<<<1, 256, 0, s>>>(kQrBlocks, k, kmax, part, h1, h2, R);
    k_qr_scale_dot<<<kQrBlocks, 256, 0, s>>>(m, v, R + (size_t)k * kmax + k, rhs, Q + (int64_t)k * m, part);
    k_sum_to<<<1, 32, 0, s>>>(kQrBlocks, part, qtb + k);
    cudaMemcpyAsync(hR + (size_t)k * kmax, R + (size_t)k * kmax, sizeof(double) * (k + 1),
                    cudaMemcpyDeviceToHost, s);
    cudaMemcpyAsync(hq + k, qtb + k, sizeof(double), cudaMemcpyDeviceToHost, s);
    ctx->launches += k > 0 ? 10 : 4;
    ++k;
  }

  std::vector<double> solve() {  // R z = Q^T b (host back substitution)
    cudaStreamSynchronize(s);
    std::vector<double> z(k);
    for (int i = k - 1; i >= 0; --i) {
      double s0 = hq[i];
      for (int j = i + 1; j < k; ++j) s0 -= hR[(size_t)j * kmax + i] * z[j];
      z[i] = s0 / hR[(size_t)i * kmax + i];
    }
    return z;
  }
};

}  // namespace

extern "C" {

int podecm_ecm_mode_grads(podecm_ctx* ctx, void* stream, podecm_rve* rve, const double* modes,
                          int N, double* H) {
  if (!ctx || !rve || !modes || !H || N <= 0) return PODECM_ECONFIG;
  auto s = static_cast<cudaStream_t>(stream);
  const int64_t n = (int64_t)rve->n_qp * N;
  k_ecm_mode_grads<<<grid_for(n, 256), 256, 0, s>>>(rve->n_qp, N, 2 * (int64_t)rve->n_nodes,
                                                    rve->d_elems, rve->d_grad, modes, H);
  PODECM_LAUNCHED(ctx, 1);
  return PODECM_OK;
}

int podecm_ecm_stress_snapshots(podecm_ctx* ctx, void* stream, podecm_rve* rve, const double* U,
                                int64_t L, double* W, int32_t* status) {
  if (!ctx || !rve || !U || !W || L <= 0) return PODECM_ECONFIG;
  auto s = static_cast<cudaStream_t>(stream);
  if (status) PODECM_CUDA_TRY(ctx, cudaMemsetAsync(status, 0, sizeof(int32_t), s));
  const int64_t n = L * rve->n_qp;
  {
    KTimer kt(ctx, s, "k_ecm_stress");
    k_ecm_stress<<<grid_for(n, 128), 128, 0, s>>>(L, rve->n_qp, 2 * (int64_t)rve->n_nodes,
                                                  rve->d_elems, rve->d_regions, rve->d_grad, U,
                                                  rve->mats, W, status, ctx->d_fail);
  }
  PODECM_LAUNCHED(ctx, 1);
  return PODECM_OK;
}

int podecm_ecm_select(podecm_ctx* ctx, void* stream, podecm_rve* rve, const double* H, int N,
                      const double* W, int64_t L, const podecm_ecm_opts* opts, int32_t* ids,
                      double* weights, int* n_sel, double* resid_rel, int* iterations) {
  return podecm_ecm_select_sharded(ctx, stream, rve, H, N, W, L, nullptr, opts, ids, weights, n_sel, resid_rel,
                                   iterations);
}

// The greedy of ecm_select over this rank's candidate shard (comm != NULL;
// SURVEY §8(e)): rhs = J w summed over the shards, each iteration's local
// best (score, global index) reduced with the reference's strict-'>' first-
// index rule, the selected column broadcast from its owner, the refit (QR +
// restore_feasible) and the residual replicated on every rank.  Every rank
// takes the same decisions, so the result equals the single-rank greedy's
// up to the summation order of rhs.  Direct scoring (a J^T r pass over the
// local candidates per iteration).
int podecm_ecm_select_sharded(podecm_ctx* ctx, void* stream, podecm_rve* rve, const double* H, int N,
                              const double* W, int64_t L, const podecm_ecm_comm* comm,
                              const podecm_ecm_opts* opts, int32_t* ids, double* weights, int* n_sel,
                              double* resid_rel, int* iterations) {
  if (!ctx || !rve || !H || !W || !opts || !ids || !weights || !n_sel) return PODECM_ECONFIG;
  if (comm && (!comm->allreduce_sum || !comm->argmax || !comm->bcast || comm->q0 < 0 || comm->nq_local < 0 ||
               comm->q0 + comm->nq_local > rve->n_qp))
    return set_err(ctx, PODECM_ECONFIG, "ecm: invalid candidate shard / communicator");
  const int64_t q0 = comm ? comm->q0 : 0;
  // scoring mode, read per call: Gram-updated (default) or PODECM_ECM_SCORE=
  // direct (a J^T r DMMA pass every iteration); the sharded greedy scores
  // directly
  const bool gram_env = [] {
    const char* e = getenv("PODECM_ECM_SCORE");
    return !(e && !strcmp(e, "direct"));
  }() && !comm;
  if (N < 1 || N > (gram_env ? 1024 : 56))
    return set_err(ctx, PODECM_ECONFIG, gram_env ? "ecm: need 1 <= N <= 1024 displacement modes"
                                                 : "ecm: the direct scoring mode needs 1 <= N <= 56");
  auto s = static_cast<cudaStream_t>(stream);
  const int nq = comm ? (int)comm->nq_local : rve->n_qp;  // candidates of this rank
  const int nq_all = rve->n_qp;
  const int vol = opts->volume_row ? 1 : 0;
  const int64_t m = (int64_t)N * L + vol;
  const int cap = opts->max_points > 0 ? std::min(opts->max_points, nq_all) : nq_all;
  // device workspaces (J_sel, Q: m x kq; R: kq^2) hold at most kMaxSel columns
  constexpr int kMaxSel = 1024;
  const int kq = std::min(cap, kMaxSel);
  int rc = PODECM_OK;
  auto fail = [&](int code, const char* msg) { return set_err(ctx, code, msg); };

  double *Hw = nullptr, *rhs = nullptr, *r = nullptr, *cn = nullptr, *cta_b = nullptr, *best_b = nullptr;
  double *Jsel = nullptr, *Q = nullptr, *tmp = nullptr, *hbuf = nullptr, *xdev = nullptr, *pss = nullptr, *pmx = nullptr;
  int *cta_i = nullptr, *best_i = nullptr;
  uint8_t* unav = nullptr;
  const int n_cta = (nq + kSQ - 1) / kSQ;
  const int n_rb = grid_for(m, 256);
  auto alloc = [&](auto** p, size_t n) {
    if (!rc && cudaMalloc(p, std::max<size_t>(n, 1) * sizeof(**p)) != cudaSuccess)
      rc = fail(PODECM_ECUDA, "ecm: device allocation failed");
  };
  alloc(&Hw, (size_t)N * 4 * nq);
  alloc(&rhs, m);
  alloc(&r, m);
  alloc(&cn, nq);
  alloc(&cta_b, n_cta);
  alloc(&cta_i, n_cta);
  alloc(&best_b, 1);
  alloc(&best_i, 1);
  alloc(&Jsel, (size_t)m * kq);
  alloc(&Q, (size_t)m * kq);
  alloc(&tmp, m);
  alloc(&hbuf, kq);
  double *h2buf = nullptr, *Rdev = nullptr, *qtbdev = nullptr, *zdev = nullptr;
  alloc(&h2buf, kq);
  alloc(&Rdev, (size_t)kq * kq);
  alloc(&qtbdev, kq);
  alloc(&zdev, kq);
  alloc(&xdev, kq);
  alloc(&pss, n_rb);
  alloc(&pmx, n_rb);
  alloc(&unav, nq);
  const bool gram = gram_env;
  double *c0 = nullptr, *Gsel = nullptr, *gpart = nullptr;
  const int n_cta_g = grid_for(nq, 256);
  // speculative Gram columns (Gram mode): every pass over W also computes the
  // columns of up to kSpec runner-up candidates into a column cache, so a
  // later selection of one of them costs a 8 nq-byte copy instead of a pass
  // over the whole W (PODECM_ECM_SPEC=0 turns it off; the ids, weights and
  // every score are the same either way)
  const int kSpec = [] {
    const char* e = getenv("PODECM_ECM_SPEC");
    const int v = e ? atoi(e) : 3;
    return v < 0 ? 0 : (v > kGramCols - 1 ? kGramCols - 1 : v);
  }();
  int *spec_dev = nullptr, *sels_dev = nullptr, *pspec = nullptr, *psels = nullptr;
  double* pool = nullptr;
  int pool_cap = 0, pool_used = 0;
  std::unordered_map<int, int> cached;  // candidate -> pool column
  if (gram) {
    alloc(&c0, nq);
    alloc(&Gsel, (size_t)kq * nq);
    alloc(&gpart, (size_t)(kSpec + 1) * kGramSplit * nq);
    alloc(&spec_dev, kSpec + 1);
    alloc(&sels_dev, kSpec + 1);
    if (!rc && cudaMallocHost(&pspec, 2 * (kSpec + 1) * sizeof(int)) != cudaSuccess)
      rc = fail(PODECM_ECUDA, "ecm: pinned allocation failed");
    psels = pspec ? pspec + kSpec + 1 : nullptr;
    if (kSpec > 0 && nq > 0) {
      pool_cap = (int)std::min<int64_t>((int64_t)kSpec * kq, (int64_t(1) << 30) / ((int64_t)nq * 8));
      if (pool_cap > 0 && cudaMalloc(&pool, (size_t)pool_cap * nq * sizeof(double)) != cudaSuccess) {
        cudaGetLastError();  // no room for the cache: run without speculation
        pool = nullptr;
        pool_cap = 0;
      }
    }
  }
  double* cta_bg = nullptr;
  int* cta_ig = nullptr;
  alloc(&cta_bg, n_cta_g);
  alloc(&cta_ig, n_cta_g);
  std::vector<int> selected;
  std::vector<double> x;
  double rhs_norm = 0.0, rnorm = 0.0;
  int iters = 0;
  if (!rc) {
    cudaMemsetAsync(unav, 0, nq, s);
    // rhs = J w: Hw[i][(q,c)] = w_q H[q][i][c]; rhs[(i,s)] = sum_k Hw[i][k] W[s][k]
    k_ecm_hw<<<grid_for((int64_t)nq * N * 4, 256), 256, 0, s>>>(nq, N, H, rve->d_w + q0, Hw);
    GemmArgs a{};
    a.M = N;
    a.N = L;
    a.K = 4 * (int64_t)nq;
    a.A = Hw;
    a.a_rs = 4 * (int64_t)nq;
    a.a_cs = 1;
    a.B = W;
    a.b_rs = 1;
    a.b_cs = 4 * (int64_t)nq;
    a.C = rhs;
    a.c_rs = L;  // rhs[i * L + s]
    a.c_cs = 1;
    dim3 grid((unsigned)((a.N + kGBN - 1) / kGBN), (unsigned)((a.M + kGBM - 1) / kGBM));
    if (nq > 0) k_gemm_dmma<<<grid, 128, 0, s>>>(a);
    else cudaMemsetAsync(rhs, 0, sizeof(double) * N * L, s);
    if (comm) {  // rhs = sum over the candidate shards
      std::vector<double> hp((size_t)N * L);
      cudaMemcpyAsync(hp.data(), rhs, sizeof(double) * hp.size(), cudaMemcpyDeviceToHost, s);
      cudaStreamSynchronize(s);
      if (comm->allreduce_sum(comm->user, hp.data(), (int64_t)hp.size()) != 0)
        rc = fail(PODECM_ECUDA, "ecm: rhs all-reduce failed");
      cudaMemcpyAsync(rhs, hp.data(), sizeof(double) * hp.size(), cudaMemcpyHostToDevice, s);
      cudaStreamSynchronize(s);
    }
    if (vol) {
      double wsum = 0.0;
      for (int q = 0; q < nq_all; ++q) wsum += rve->w[q];
      cudaMemcpyAsync(rhs + m - 1, &wsum, sizeof(double), cudaMemcpyHostToDevice, s);
    }
    k_ecm_colnorm<<<grid_for(nq, 128), 128, 0, s>>>(L, nq, N, H, W, vol, cn);
    cudaMemcpyAsync(r, rhs, sizeof(double) * m, cudaMemcpyDeviceToDevice, s);
    ctx->launches += 2;
    std::vector<double> hr(m);
    cudaMemcpyAsync(hr.data(), rhs, sizeof(double) * m, cudaMemcpyDeviceToHost, s);
    cudaStreamSynchronize(s);
    double ss = 0.0;
    for (double v : hr) ss += v * v;
    rhs_norm = std::sqrt(ss);
    rnorm = rhs_norm;
  }
  const double row_tol = opts->eps * rhs_norm / std::sqrt((double)m);
  double rmax = rhs_norm;  // max |r| of the initial residual computed below
  if (!rc) {
    std::vector<double> hr(m);
    cudaMemcpyAsync(hr.data(), r, sizeof(double) * m, cudaMemcpyDeviceToHost, s);
    cudaStreamSynchronize(s);
    rmax = 0.0;
    for (double v : hr) rmax = std::max(rmax, std::fabs(v));
  }
  if (!rc) cudaMemsetAsync(h2buf, 0, sizeof(double) * kq, s);
  double* qpart = nullptr;
  alloc(&qpart, (size_t)kQrBlocks * kq);
  // pinned host staging for the per-iteration round trips: R mirror, Q^T b,
  // residual partials, x, the argmax index and the 'unavailable' flag
  double* pin = nullptr;
  const size_t n_pin = (size_t)kq * kq + 2 * (size_t)kq + 2 * (size_t)n_rb + 2;
  if (!rc && cudaMallocHost(&pin, n_pin * sizeof(double)) != cudaSuccess)
    rc = fail(PODECM_ECUDA, "ecm: pinned allocation failed");
  double* pR = pin;
  double* pq = pR + (size_t)kq * kq;
  double* px = pq + kq;
  double* ps = px + kq;
  double* pm = ps + n_rb;
  int* pbest = reinterpret_cast<int*>(pm + n_rb);
  uint8_t* pone = reinterpret_cast<uint8_t*>(pm + n_rb + 1);
  if (pin) {
    std::fill(pR, pR + (size_t)kq * kq, 0.0);
    *pone = 1;
  }
  Ecm qr{ctx, s, m, kq, Jsel, Q, tmp, hbuf, h2buf, Rdev, qtbdev, rhs, qpart, 0, pR, pq};
  auto converged = [&]() {
    if (rhs_norm == 0.0) return true;
    return rnorm <= opts->eps * rhs_norm && rmax <= row_tol;
  };
  bool stopped_at_count = false;
  while (!rc && !converged()) {
    if ((int)selected.size() >= cap) {
      if (opts->stop_at_count) {
        stopped_at_count = true;
        break;
      }
      rc = fail(PODECM_ESOLVE, "cubature did not reach the requested accuracy within the point budget");
      break;
    }
    if ((int)selected.size() >= kq) {
      rc = fail(PODECM_ECONFIG, "ecm: more than 1024 selected points is not supported by this build");
      break;
    }
    // corr = J^T r ; argmax of corr / ||J_q|| over available columns
    int w_n = n_cta_g;  // the per-CTA winners the argmax reduced (for the speculation set)
    const double* w_b = cta_bg;
    const int* w_i = cta_ig;
    if (gram && iters > 0) {
      {
        KTimer kt(ctx, s, "k_ecm_score_gram");
        k_ecm_score_gram<<<n_cta_g, 256, 0, s>>>(nq, (int)x.size(), c0, Gsel, xdev, cn, unav, cta_bg, cta_ig);
      }
      k_ecm_argmax<<<1, 1024, 0, s>>>(n_cta_g, cta_bg, cta_ig, best_b, best_i);
    } else {
      if (N <= 56) {
        KTimer kt(ctx, s, "k_ecm_score");
        k_ecm_score<<<n_cta, 224, 0, s>>>(L, nq, N, r, vol ? r + m - 1 : nullptr, H, W, cn, unav, cta_b, cta_i,
                                          gram ? c0 : nullptr, N, 0);  // first pass: r = rhs, keep J^T rhs
        k_ecm_argmax<<<1, 1024, 0, s>>>(n_cta, cta_b, cta_i, best_b, best_i);
        w_n = n_cta;
        w_b = cta_b;
        w_i = cta_i;
      } else {  // wide basis (Gram mode only): c0 = J^T rhs in row blocks of 56 modes, then score it
        KTimer kt(ctx, s, "k_ecm_score");
        for (int i0 = 0; i0 < N; i0 += 56) {
          const int nb = std::min(56, N - i0);
          k_ecm_score<<<n_cta, 224, 0, s>>>(L, nq, nb, r + (int64_t)i0 * L, (vol && i0 == 0) ? r + m - 1 : nullptr,
                                            H + (int64_t)i0 * 4, W, cn, unav, cta_b, cta_i, c0, N, i0 > 0);
          ctx->launches += 1;
        }
        k_ecm_score_gram<<<n_cta_g, 256, 0, s>>>(nq, 0, c0, Gsel, xdev, cn, unav, cta_bg, cta_ig);
        k_ecm_argmax<<<1, 1024, 0, s>>>(n_cta_g, cta_bg, cta_ig, best_b, best_i);
      }
    }
    ctx->launches += 2;
    const bool spec = gram && pool_cap > 0;
    if (spec) {  // the selected point and its runners-up in one read-back
      k_ecm_runners<<<1, 1024, 0, s>>>(w_n, w_b, w_i, best_i, kSpec, spec_dev);
      ctx->launches += 1;
      cudaMemcpyAsync(pspec, spec_dev, sizeof(int) * (kSpec + 1), cudaMemcpyDeviceToHost, s);
    } else {
      cudaMemcpyAsync(pbest, best_i, sizeof(int), cudaMemcpyDeviceToHost, s);
    }
    cudaStreamSynchronize(s);
    int best = spec ? pspec[0] : *pbest;  // local index
    int owner = 0;
    int64_t gbest = best < 0 ? -1 : q0 + best;
    if (comm) {  // global best: larger score, then smaller global index
      double sc = 0.0;
      if (best >= 0) {
        cudaMemcpyAsync(pm, best_b, sizeof(double), cudaMemcpyDeviceToHost, s);
        cudaStreamSynchronize(s);
        sc = *pm;
      }
      if (comm->argmax(comm->user, &sc, &gbest, &owner) != 0) {
        rc = fail(PODECM_ECUDA, "ecm: argmax exchange failed");
        break;
      }
      best = (gbest >= q0 && gbest < q0 + nq) ? (int)(gbest - q0) : -1;
    }
    if (gbest < 0) {
      rc = fail(PODECM_ESOLVE, "cubature stalled: no remaining point improves the residual");
      break;
    }
    selected.push_back((int)gbest);
    if (best >= 0) cudaMemcpyAsync(unav + best, pone, 1, cudaMemcpyHostToDevice, s);
    x.push_back(0.0);
    // materialise the new column (its owner; broadcast to the other shards)
    // and extend the QR
    if (best >= 0) {
      KTimer kt(ctx, s, "k_ecm_column");
      k_ecm_column<<<grid_for(m, 256), 256, 0, s>>>(L, nq, N, best, H, W, vol, Jsel + (int64_t)qr.k * m);
      ctx->launches += 1;
    }
    if (comm) {
      std::vector<double> col(m);
      if (best >= 0) cudaMemcpyAsync(col.data(), Jsel + (int64_t)qr.k * m, sizeof(double) * m, cudaMemcpyDeviceToHost, s);
      cudaStreamSynchronize(s);
      if (comm->bcast(comm->user, col.data(), m, owner) != 0) {
        rc = fail(PODECM_ECUDA, "ecm: column broadcast failed");
        break;
      }
      cudaMemcpyAsync(Jsel + (int64_t)qr.k * m, col.data(), sizeof(double) * m, cudaMemcpyHostToDevice, s);
      cudaStreamSynchronize(s);
    }
    if (gram) {  // column (J^T J)[:, best] for the scores of the next iterations
      double* gdst = Gsel + (int64_t)qr.k * nq;
      const auto hit = cached.find(best);
      if (hit != cached.end()) {  // computed speculatively by an earlier pass
        cudaMemcpyAsync(gdst, pool + (int64_t)hit->second * nq, sizeof(double) * nq, cudaMemcpyDeviceToDevice, s);
        cached.erase(hit);
      } else {
        int C = 1;
        psels[0] = best;
        for (int k = 1; spec && k <= kSpec; ++k) {
          const int c = pspec[k];
          if (c >= 0 && c != best && !cached.count(c) && pool_used + C <= pool_cap) psels[C++] = c;
        }
        cudaMemcpyAsync(sels_dev, psels, sizeof(int) * C, cudaMemcpyHostToDevice, s);
        KTimer kt(ctx, s, "k_ecm_gram_col");
        launch_gram_cols(C, dim3(grid_for(nq, 64), kGramSplit), s, L, nq, N, sels_dev, H, W, gpart,
                         std::make_integer_sequence<int, kGramCols>{});
        k_ecm_gram_finish<<<n_cta_g, 256, 0, s>>>(nq, gpart, vol, gdst);
        for (int k = 1; k < C; ++k) {
          k_ecm_gram_finish<<<n_cta_g, 256, 0, s>>>(nq, gpart + (int64_t)k * kGramSplit * nq, vol,
                                                    pool + (int64_t)pool_used * nq);
          cached[psels[k]] = pool_used++;
        }
        ctx->launches += 1 + C;
      }
    }
    qr.append();
    // restore_feasible (ecm.cpp:56-90)
    while (!selected.empty()) {
      std::vector<double> z = qr.solve();
      double zmin = 1e300;
      for (double v : z) zmin = std::min(zmin, v);
      if (zmin > 0.0) {
        x = z;
        break;
      }
      double alpha = 1.0;
      for (size_t k = 0; k < z.size(); ++k)
        if (z[k] <= 0.0) alpha = std::min(alpha, x[k] / (x[k] - z[k]));
      double xmax = 0.0;
      for (size_t k = 0; k < x.size(); ++k) {
        x[k] += alpha * (z[k] - x[k]);
        xmax = std::max(xmax, std::fabs(x[k]));
      }
      const double zero_tol = 1e-12 * std::max(xmax, 1e-30);
      std::vector<int> keep_ids;
      std::vector<double> keep_x;
      std::vector<int> keep_pos;
      for (size_t k = 0; k < x.size(); ++k)
        if (x[k] > zero_tol) {
          keep_ids.push_back(selected[k]);
          keep_x.push_back(x[k]);
          keep_pos.push_back((int)k);
        }
      // compact Jsel columns and rebuild the QR of the kept set
      for (size_t k = 0; k < keep_pos.size(); ++k)
        if (keep_pos[k] != (int)k) {
          cudaMemcpyAsync(Jsel + (int64_t)k * m, Jsel + (int64_t)keep_pos[k] * m, sizeof(double) * m,
                          cudaMemcpyDeviceToDevice, s);
          if (gram)
            cudaMemcpyAsync(Gsel + (int64_t)k * nq, Gsel + (int64_t)keep_pos[k] * nq, sizeof(double) * nq,
                            cudaMemcpyDeviceToDevice, s);
        }
      selected = keep_ids;
      x = keep_x;
      qr.k = 0;
      for (size_t k = 0; k < selected.size(); ++k) qr.append();
    }
    ++iters;
    // resid = rhs - J_sel x
    std::copy(x.begin(), x.end(), px);
    cudaMemcpyAsync(xdev, px, sizeof(double) * x.size(), cudaMemcpyHostToDevice, s);
    {
      KTimer kt(ctx, s, "k_resid");
      k_resid<<<n_rb, 256, 0, s>>>(m, (int)x.size(), Jsel, xdev, rhs, r, pss, pmx);
    }
    ctx->launches += 1;
    cudaMemcpyAsync(ps, pss, sizeof(double) * n_rb, cudaMemcpyDeviceToHost, s);
    cudaMemcpyAsync(pm, pmx, sizeof(double) * n_rb, cudaMemcpyDeviceToHost, s);
    cudaStreamSynchronize(s);
    double ss = 0.0;
    rmax = 0.0;
    for (int b = 0; b < n_rb; ++b) {
      ss += ps[b];
      rmax = std::max(rmax, pm[b]);
    }
    rnorm = std::sqrt(ss);
  }
  (void)stopped_at_count;
  if (!rc) {
    std::vector<int> order(selected.size());
    std::iota(order.begin(), order.end(), 0);
    std::sort(order.begin(), order.end(), [&](int p, int q) { return selected[p] < selected[q]; });
    for (size_t k = 0; k < order.size(); ++k) {
      ids[k] = selected[order[k]];
      weights[k] = x[order[k]];
    }
    *n_sel = (int)selected.size();
    if (resid_rel) *resid_rel = rhs_norm == 0.0 ? 0.0 : rnorm / rhs_norm;
    if (iterations) *iterations = iters;
  }
  cudaFree(Hw);
  cudaFree(rhs);
  cudaFree(r);
  cudaFree(cn);
  cudaFree(cta_b);
  cudaFree(cta_i);
  cudaFree(best_b);
  cudaFree(best_i);
  cudaFree(Jsel);
  cudaFree(Q);
  cudaFree(tmp);
  cudaFree(hbuf);
  cudaFree(h2buf);
  cudaFree(Rdev);
  cudaFree(qtbdev);
  cudaFree(zdev);
  cudaFree(xdev);
  cudaFree(pss);
  cudaFree(pmx);
  cudaFree(unav);
  cudaFree(qpart);
  if (pin) cudaFreeHost(pin);
  cudaFree(c0);
  cudaFree(Gsel);
  cudaFree(gpart);
  cudaFree(spec_dev);
  cudaFree(sels_dev);
  cudaFree(pool);
  cudaFreeHost(pspec);
  cudaFree(cta_bg);
  cudaFree(cta_ig);
  return rc;
}

}  // extern "C"
