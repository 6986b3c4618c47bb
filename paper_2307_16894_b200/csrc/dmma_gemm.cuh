// Tiled FP64 tensor-core GEMM on sm_100a: mma.sync.m8n8k4.f64 (DMMA).
// tcgen05.mma has no f64 kind on sm_100a, so the FP64
// tensor path is the warp-level DMMA instruction; this is the building block
// of the POD Gram (S^T G S) and the POD mode map (S V).
//
//   C(i,j) = sum_k A(i,k) B(k,j)   with
//   A(i,k) = A[i*a_rs + k*a_cs], B(k,j) = B[k*b_rs + j*b_cs],
//   C(i,j) = C[i*c_rs + j*c_cs]   (signed 64-bit strides).
// Optional: diag (nullable) scales the k-th term, A(i,k) g_k B(k,j) (the
// diagonal Gram of pod_diag); sym = only tiles with j-block >= i-block are
// computed and mirrored (S^T S).
#pragma once

#include <cstdint>

namespace podecm_dev {

constexpr int kGBM = 64, kGBN = 64, kGBK = 16, kGLD = kGBK + 4;
constexpr int kMaxPeers = 8;  // ranks of a fused peer epilogue (one NVLink domain)

__device__ __forceinline__ void dmma884(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

struct GemmArgs {
  int64_t M, N, K;
  const double* A;
  int64_t a_rs, a_cs;
  const double* B;
  int64_t b_rs, b_cs;
  double* C;
  int64_t c_rs, c_cs;
  const double* diag;  // nullable, length K
  int sym;
  // split-K (gridDim.z slices): slice z covers k in [z kslice, (z+1) kslice)
  // and writes its partial product at C + z zc (kslice 0: no split)
  int64_t kslice, zc;
  // peer epilogue (peer_world > 0): element (i, j) goes to the receive slot
  // of the rank owning row i (rows [row0[o], row0[o+1]) belong to rank o):
  // peer[o] + (peer_rank * (row0[o+1] - row0[o]) + i - row0[o]) * c_rs + j,
  // a store into that rank's memory (CUDA IPC / peer mapping, NVLink) — the
  // reduce-scatter of a row-sharded Gram fused into the GEMM that produces it
  int peer_world, peer_rank;
  double* peer[kMaxPeers];
  int64_t row0[kMaxPeers + 1];
};

// 128 threads = 2x2 warps, warp tile 32x32 (4x4 DMMA tiles).  Internal
// linkage: every translation unit that launches it gets its own copy.
template <bool SPLIT>
static __global__ void __launch_bounds__(128) k_gemm_dmma_t(GemmArgs g) {
  __shared__ double sA[2][kGBM][kGLD];
  __shared__ double sB[2][kGBN][kGLD];
  const int bi = blockIdx.y, bj = blockIdx.x;
  if (g.sym && bj < bi) return;
  if (SPLIT) {  // this CTA's K slice
    const int64_t k0 = (int64_t)blockIdx.z * g.kslice;
    g.A += k0 * g.a_cs;
    g.B += k0 * g.b_rs;
    if (g.diag) g.diag += k0;
    g.K = g.K - k0 < g.kslice ? g.K - k0 : g.kslice;
    g.C += (int64_t)blockIdx.z * g.zc;
  }
  const int64_t i0 = (int64_t)bi * kGBM, j0 = (int64_t)bj * kGBN;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int wm = warp >> 1, wn = warp & 1, gid = lane >> 2, tig = lane & 3;
  double acc[4][4][2];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;

  // loader mapping: contiguous along k when the k-stride is 1, else along i/j
  auto load = [&](int buf, int64_t k0) {
    for (int t = tid; t < kGBM * kGBK; t += 128) {
      int r, k;
      if (g.a_cs == 1) { r = t / kGBK; k = t % kGBK; } else { r = t % kGBM; k = t / kGBM; }
      const int64_t gi = i0 + r, gk = k0 + k;
      double v = 0.0;
      if (gi < g.M && gk < g.K) {
        v = g.A[gi * g.a_rs + gk * g.a_cs];
        if (g.diag) v *= g.diag[gk];
      }
      sA[buf][r][k] = v;
    }
    for (int t = tid; t < kGBN * kGBK; t += 128) {
      int c, k;
      if (g.b_rs == 1) { c = t / kGBK; k = t % kGBK; } else { c = t % kGBN; k = t / kGBN; }
      const int64_t gj = j0 + c, gk = k0 + k;
      sB[buf][c][k] = (gj < g.N && gk < g.K) ? g.B[gk * g.b_rs + gj * g.b_cs] : 0.0;
    }
  };

  const int64_t nk = (g.K + kGBK - 1) / kGBK;
  load(0, 0);
  __syncthreads();
  for (int64_t kt = 0; kt < nk; ++kt) {
    const int buf = (int)(kt & 1);
    if (kt + 1 < nk) load(buf ^ 1, (kt + 1) * kGBK);
#pragma unroll
    for (int kk = 0; kk < kGBK / 4; ++kk) {
      double af[4], bf[4];
#pragma unroll
      for (int a = 0; a < 4; ++a) af[a] = sA[buf][wm * 32 + a * 8 + gid][kk * 4 + tig];
#pragma unroll
      for (int b = 0; b < 4; ++b) bf[b] = sB[buf][wn * 32 + b * 8 + gid][kk * 4 + tig];
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) dmma884(acc[a][b][0], acc[a][b][1], af[a], bf[b]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int64_t i = i0 + wm * 32 + a * 8 + gid;
        const int64_t j = j0 + wn * 32 + b * 8 + 2 * tig + h;
        if (i < g.M && j < g.N) {
          if (g.peer_world > 0) {  // symmetric Gram partial: row i and (mirrored) row j to their owners
            auto put = [&](int64_t r, int64_t c, double v) {
              int o = 0;
              while (o + 1 < g.peer_world && r >= g.row0[o + 1]) ++o;
              const int64_t rows = g.row0[o + 1] - g.row0[o];
              g.peer[o][((int64_t)g.peer_rank * rows + r - g.row0[o]) * g.c_rs + c] = v;
            };
            put(i, j, acc[a][b][h]);
            if (g.sym && bj != bi) put(j, i, acc[a][b][h]);
          } else {
            g.C[i * g.c_rs + j * g.c_cs] = acc[a][b][h];
            if (g.sym && bj != bi) g.C[j * g.c_rs + i * g.c_cs] = acc[a][b][h];
          }
        }
      }
}

// the plain GEMM and the split-K one (gridDim.z K slices, GemmArgs.kslice)
#define k_gemm_dmma k_gemm_dmma_t<false>
#define k_gemm_dmma_split k_gemm_dmma_t<true>

}  // namespace podecm_dev
