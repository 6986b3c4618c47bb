// K3 — batched ECM hyper-reduced online stage (BASELINE config 3).
//
// Replaces rom_solve + rom_solve_step_adaptive + rom_solve_step +
// rom_assemble (/root/reference/proj/src/rom.cpp:34-200) for a batch of
// independent RVE instances sharing one RomModel.  Every instance runs its
// own Newton / bisection state machine; one "global iteration" is one
// reduced assembly for every still-active instance:
//
//   k_rom_point     (instance, ECM point): F = Fbar + R(Fmu^-1)^T (G_p^T a),
//                   material point (P, FD tangent, trial history), then the
//                   mapped per-point operators
//                     At_p = c_p R_p A_p R_p^T   (4x4),  Pt_p = c_p R_p P_p
//                   with c_p = w_p det Fmu_p and R_p = right_mult_op(Fmu^-1)
//                   (rom.cpp:16-26);
//   k_rom_contract  K = sum_p G_p At_p G_p^T and f = sum_p G_p Pt_p as one
//                   FP64 tensor-core GEMM per instance, K_ext = Gm^T Y with
//                   Gm the (4Q x N) stack of the shared mode gradients and
//                   Y = blockdiag(At) Gm | Pt (f rides in the padding column
//                   N of the N+1 -> 8-aligned tile width); mma.sync m8n8k4
//                   f64 (DMMA — tcgen05 has no f64 kind on sm_100a);
//   k_rom_newton    one warp per instance: ||f||, the reference's convergence
//                   test (tolerance frozen at iteration 0), dense LU with
//                   partial pivoting (Eigen PartialPivLU semantics) and the
//                   update, or the adaptive bisection / commit logic.
//
// Default ("lazy tangent") order of one global iteration: k_rom_F, k_rom_point
// MODE 1 (P, Pt, trial history), k_rom_check (f = Gm^T Pt by DMMA, residual
// test; converged / failed instances finish here, the rest are compacted into
// a list), k_rom_point MODE 2 (FD tangent for the listed instances only),
// k_rom_contract over the list, k_rom_solve (LU + update).  A quarter of the
// assemblies are the final convergence checks, which never need K, so this
// skips a quarter of the tangents and contractions.  One deviation: an FD
// failure at an assembly that already satisfies the tolerance is not seen
// (the reference would fail that attempt); PODECM_ROM_LAZY=0 restores the
// fused order.
//
// Summation order of the contractions differs from Eigen's; the stated
// tolerance for the homogenised stress history is 1e-8 (BASELINE north star).
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <type_traits>
#include <utility>
#include <vector>

#include "rve.cuh"

using namespace podecm_dev;
using namespace podecm_impl;

namespace {

constexpr int kMaxStack = 8;    // max_bisect + 1 frames (max_bisect <= 7)
constexpr int kPC = 8;          // points per contraction chunk (32 k-rows)
constexpr int kIPC = 2;         // instances per contraction CTA (NT <= 7)
constexpr int kMaxNT = 15;      // contraction column tiles: N + 1 <= 120 (N <= 119 modes)
constexpr int kPtsTile = 32;    // material kernel: points per CTA
constexpr int kInstTile = 8;    // material kernel: instances per CTA

struct RomCtl {
  double tol, resid;
  double r0, r0max;  // first residual of the current attempt; max over converged sub-steps
  double fstack[kMaxStack][8];  // (F_prev[4], F_target[4]) per pending task
  int dstack[kMaxStack];        // remaining bisection depth per task
  int sp, it, k, iters_acc, cur, active, status, asm_fail;
};

}  // namespace

struct podecm_rom {
  podecm_rve* rve = nullptr;
  podecm_ctx* ctx = nullptr;
  int N = 0, Q = 0, Qpad = 0, NT = 0, NP = 0;
  int32_t* d_ids = nullptr;
  int32_t* d_reg = nullptr;  // material index per ECM point
  double* d_w = nullptr;
  double* d_G = nullptr;   // Gm padded [Qpad*4][NP] row-major: rows (p, r), cols i
  double* d_Gt = nullptr;  // [N][4][Qpad]: G_p[i][r], p fastest (material kernel)
  int64_t cap = 0;
  double *d_morph = nullptr, *d_S = nullptr, *d_At = nullptr, *d_P = nullptr, *d_K = nullptr,
         *d_f = nullptr, *d_a = nullptr, *d_a0 = nullptr, *d_Fb = nullptr,
         *d_Pt = nullptr;  // lazy tangent: compact Pt [cap][Qpad][4]
  RomCtl* d_ctl = nullptr;
  double* d_CA = nullptr;     // effective stiffness: c_p A_p [cap][Q][16] (lazy)
  double* d_Sprev = nullptr;  // effective stiffness: history at the start of the last increment
  int64_t abar_cap = 0;
  int* d_nactive = nullptr;  // [0] active instances, [1] lazy-tangent list length
  int* h_nactive = nullptr;
  int* d_list = nullptr;  // lazy tangent: compacted instances that need K [cap]
  int* d_alist = nullptr;  // lazy tangent: compacted active instances [cap] (refreshed at host syncs)
  int64_t last_global_iters = 0;
};

struct podecm_rom_engines {
  podecm_rom* rom = nullptr;
  int64_t n = 0;
  bool has_bounds = false;
  double bounds[6] = {0, 0, 0, 0, 0, 0};
  double *d_geom = nullptr, *d_Sc = nullptr, *d_St = nullptr, *d_ac = nullptr, *d_at = nullptr,
         *d_fc = nullptr, *d_ft = nullptr, *d_fref = nullptr, *d_ires = nullptr;
  int32_t *d_ok = nullptr, *d_oor = nullptr, *d_status = nullptr;
};

namespace {

void free_work(podecm_rom* r) {
  cudaFree(r->d_morph);
  cudaFree(r->d_S);
  cudaFree(r->d_At);
  cudaFree(r->d_P);
  cudaFree(r->d_K);
  cudaFree(r->d_f);
  cudaFree(r->d_a);
  cudaFree(r->d_a0);
  cudaFree(r->d_Fb);
  cudaFree(r->d_Pt);
  cudaFree(r->d_ctl);
  cudaFree(r->d_list);
  cudaFree(r->d_alist);
  cudaFree(r->d_CA);
  cudaFree(r->d_Sprev);
  r->d_CA = r->d_Sprev = nullptr;
  r->abar_cap = 0;
  r->d_morph = r->d_S = r->d_At = r->d_P = r->d_K = r->d_f = r->d_a = r->d_a0 = r->d_Fb = r->d_Pt = nullptr;
  r->d_ctl = nullptr;
  r->d_list = nullptr;
  r->d_alist = nullptr;
  r->cap = 0;
}

// ---- init: morph slice at the ECM points, virgin history, control blocks
// Morph slice at the ECM points (slice_morph, rom.cpp:111-120): from the
// analytic map of geom (a, b), or copied from morph_in [n][5][Q] (fmu_inv
// planes + det of a caller's MorphField, podecm_rom_solve_batch_morph).
__global__ void k_rom_init_points(int64_t n, int Q, int nq, double r0, const int32_t* ids,
                                  const double* nodes, const int32_t* elems, const double* grad,
                                  const double* geom, double* morph, double* S, int64_t cap,
                                  RomCtl* ctl, double* Sprev, const double* S_start,
                                  const double* morph_in = nullptr) {
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (tid >= n * Q) return;
  const int64_t s = tid / Q;
  const int p = (int)(tid - s * Q);
  double fmi[4], dt;
  if (morph_in) {
    const double* mi = morph_in + (size_t)s * 5 * Q;
    for (int t = 0; t < 4; ++t) fmi[t] = mi[(size_t)t * Q + p];
    dt = mi[(size_t)4 * Q + p];
  } else {
    const int qp = ids[p], e = qp >> 2;
    const double ka = geom[2 * s] / r0 - 1.0, kb = geom[2 * s + 1] / r0 - 1.0;
    double d[4][2], gq[8];
    for (int t = 0; t < 8; ++t) gq[t] = grad[(size_t)qp * 8 + t];
    for (int a = 0; a < 4; ++a) {
      const int nd = elems[4 * e + a];
      morph_d(nodes[2 * nd], nodes[2 * nd + 1], ka, kb, r0, d[a][0], d[a][1]);
    }
    dt = derive_qp(d, gq, fmi);
  }
  double* mo = morph + (size_t)s * 5 * Q;
  for (int t = 0; t < 4; ++t) mo[(size_t)t * Q + p] = fmi[t];
  mo[(size_t)4 * Q + p] = dt;
  if (!(dt > 0.0)) {  // morph folds the mesh: SolveError (morph.cpp:116-119)
    ctl[s].status = PODECM_ESOLVE;
    ctl[s].active = 0;
  }
  double* st = S + (size_t)s * 6 * Q;  // buffer 0 = committed history (virgin or given)
  double v[6] = {1.0, 0.0, 0.0, 1.0, 1.0, 0.0};
  if (S_start)
    for (int t = 0; t < 6; ++t) v[t] = S_start[((size_t)s * 6 + t) * Q + p];
  for (int t = 0; t < 6; ++t) st[(size_t)t * Q + p] = v[t];
  if (Sprev)
    for (int t = 0; t < 6; ++t) Sprev[((size_t)s * 6 + t) * Q + p] = v[t];
  (void)cap;
  (void)nq;
}

__global__ void k_rom_init_inst(int64_t n, int N, int max_bisect, const double* sched, int K,
                                double* a, double* a0, RomCtl* ctl, int32_t* status,
                                const double* fprev, const double* a_start) {
  const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= n) return;
  RomCtl c;
  memset(&c, 0, sizeof(c));
  c.active = 1;
  c.sp = 1;
  c.dstack[0] = max_bisect;
  const double I[4] = {1.0, 0.0, 0.0, 1.0};
  for (int t = 0; t < 4; ++t) {
    c.fstack[0][t] = fprev ? fprev[(size_t)s * 4 + t] : I[t];
    c.fstack[0][4 + t] = sched[((size_t)s * K + 0) * 4 + t];
  }
  ctl[s] = c;
  for (int i = 0; i < N; ++i) {
    const double v = a_start ? a_start[(size_t)s * N + i] : 0.0;
    a[(size_t)s * N + i] = a0[(size_t)s * N + i] = v;
  }
  if (status) status[s] = 0;
}

// status of morph failures written by k_rom_init_points lands after init_inst
__global__ void k_rom_fix_status(int64_t n, RomCtl* ctl, int32_t* status, unsigned int* fail) {
  const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= n) return;
  if (ctl[s].status) {
    ctl[s].active = 0;
    if (status) status[s] = PODECM_ESOLVE;
    atomicAdd(fail, 1u);
  }
}

// ---- material at the ECM points -----------------------------------------
struct PointArgs {
  int64_t n;          // instances (or, with alist, entries of alist) this launch covers
  const int* alist = nullptr;  // nullable: instance of entry k (lazy pipeline: active instances only)
  int N, Q, Qpad;
  int64_t cap;
  const double* Gt;
  const double* a;
  const double* morph;
  const double* w;
  const int32_t* reg;
  double* S;   // [2][cap][6][Q]
  double* At;  // [n][Qpad][20]
  double* P;   // [n][Q][4]
  double* Fb;  // [n][4][Q]
  double* Pt;  // MODE 1: compact Pt [n][Qpad][4]
  RomCtl* ctl;
  const double* S0;  // effective-stiffness stage: frozen history [n][6][Q]
  double* CA;        // effective-stiffness stage: c_p A_p [n][Q][16]
  const int* list;   // lazy tangent: instances that need K (MODE 2)
  const int* count;
};

// F at every ECM point: F = Fbar + R(Fmu^-1)^T (G_p^T a) (rom.cpp:48-50).  CTA =
// 32 points x 8 instances sharing one SMEM tile of the mode gradients.
constexpr int kFInst = 32;  // k_rom_F: instances per CTA (4 per thread)

__device__ __forceinline__ int64_t inst_of(const int* alist, int64_t k) { return alist ? alist[k] : k; }

// Active instances in ascending order (deterministic block scan, one CTA):
// alist[0 .. alist[cap]) .  The lazy pipeline sizes its grids by this count
// between host syncs, so finished instances cost no empty CTAs.
__global__ void __launch_bounds__(1024) k_rom_compact(int64_t n, const RomCtl* ctl, int* alist, int64_t cap) {
  __shared__ int part[1024];
  const int t = threadIdx.x;
  const int64_t per = (n + 1023) / 1024, b = t * per, e = b + per < n ? b + per : n;
  int cnt = 0;
  for (int64_t i = b; i < e; ++i) cnt += ctl[i].active ? 1 : 0;
  part[t] = cnt;
  __syncthreads();
  if (t == 0) {
    int acc = 0;
    for (int k = 0; k < 1024; ++k) {
      const int v = part[k];
      part[k] = acc;
      acc += v;
    }
    alist[cap] = acc;
  }
  __syncthreads();
  int o = part[t];
  for (int64_t i = b; i < e; ++i)
    if (ctl[i].active) alist[o++] = (int)i;
}

__global__ void __launch_bounds__(256) k_rom_F(PointArgs g) {
  extern __shared__ double sm[];
  double* sG = sm;                               // [N][4][32]
  double* sa = sm + (size_t)g.N * 4 * kPtsTile;  // [kFInst][N]
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const int p0 = blockIdx.x * kPtsTile;
  const int64_t s0 = (int64_t)blockIdx.y * kFInst;
  {  // whole CTA idle (finished / failed instances): skip the staging
    __shared__ int any_active;
    if (threadIdx.x == 0) any_active = 0;
    __syncthreads();
    if (threadIdx.x < kFInst && s0 + threadIdx.x < g.n && g.ctl[inst_of(g.alist, s0 + threadIdx.x)].active)
      any_active = 1;
    __syncthreads();
    if (!any_active) return;
  }
  for (int t = threadIdx.x; t < g.N * 4 * kPtsTile; t += blockDim.x) {
    const int ir = t / kPtsTile, pl = t - ir * kPtsTile;
    sG[t] = (p0 + pl < g.Qpad) ? g.Gt[(size_t)ir * g.Qpad + p0 + pl] : 0.0;
  }
  for (int t = threadIdx.x; t < kFInst * g.N; t += blockDim.x) {
    const int si = t / g.N, i = t - si * g.N;
    sa[t] = (s0 + si < g.n) ? g.a[(size_t)inst_of(g.alist, s0 + si) * g.N + i] : 0.0;
  }
  __syncthreads();
  const int p = p0 + tx;
  if (p >= g.Q) return;
  // u = G_p^T a for 4 instances per thread: each G value from SMEM feeds 4 FMAs
  double u[4][4];
#pragma unroll
  for (int q = 0; q < 4; ++q)
#pragma unroll
    for (int r = 0; r < 4; ++r) u[q][r] = 0.0;
  for (int i = 0; i < g.N; ++i) {
    double gv[4];
#pragma unroll
    for (int r = 0; r < 4; ++r) gv[r] = sG[(i * 4 + r) * kPtsTile + tx];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const double av = sa[(ty + 8 * q) * g.N + i];
#pragma unroll
      for (int r = 0; r < 4; ++r) u[q][r] = fma(gv[r], av, u[q][r]);
    }
  }
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    if (s0 + ty + 8 * q >= g.n) break;
    const int64_t s = inst_of(g.alist, s0 + ty + 8 * q);
    const RomCtl* c = g.ctl + s;
    if (!c->active) continue;
    // F = Fbar + R(fmi)^T u  (mapped^T a, rom.cpp:48-50)
    const double* mo = g.morph + (size_t)s * 5 * g.Q;
    double m[4];
#pragma unroll
    for (int t = 0; t < 4; ++t) m[t] = mo[(size_t)t * g.Q + p];
    const int top = c->sp - 1;
#pragma unroll
    for (int ii = 0; ii < 2; ++ii)
#pragma unroll
      for (int l = 0; l < 2; ++l)
        g.Fb[((size_t)s * 4 + ii + 2 * l) * g.Q + p] =
            c->fstack[top][4 + ii + 2 * l] + (u[q][ii] * m[2 * l] + u[q][ii + 2] * m[1 + 2 * l]);
  }
}

// D += A B on one m8n8k4 f64 tile (mma.sync: DMMA; tcgen05 has no f64 kind)
__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

// The same F by FP64 tensor cores: U = A Gm^T with A the (instances x modes)
// reduced coordinates and Gm the (4Q x N) mode-gradient stack (d_G, zero
// padded), one DMMA GEMM tile per CTA (32 instances x 32 points = 128 point
// rows, K = N rounded up to the k-step of 4), then F = Fbar + R(fmi)^T u per
// (instance, point) from shared memory.  Same F formula as k_rom_F; u is
// summed in the tensor cores' order instead of k_rom_F's sequential FMA chain
// (agreement to rounding, well inside the ROM tolerance).
constexpr int kFMI = 32;  // instances per CTA
constexpr int kFMP = 32;  // points per CTA
constexpr int kFUP = kFMP + 1;  // sU pitch per (instance, r): conflict-free lane = point reads

__host__ __device__ inline int fmma_ld(int N) {
  const int kp = (N + 3) & ~3;
  return (kp & 7) == 4 ? kp : kp + 4;  // == 4 mod 8: conflict-free m8n8k4 fragment loads
}
__host__ __device__ inline size_t fmma_smem_doubles(int N) {
  const int ld = fmma_ld(N);
  const size_t b = (size_t)kFMP * 4 * ld, u = (size_t)kFMI * 4 * kFUP;
  return (size_t)kFMI * ld + (b > u ? b : u);
}

__global__ void __launch_bounds__(256) k_rom_F_mma(PointArgs g, const double* __restrict__ G, int NP) {
  extern __shared__ double sm[];
  const int N = g.N, KP = (N + 3) & ~3, LD = fmma_ld(N);
  double* sA = sm;                       // [kFMI][LD]   reduced coordinates
  double* sB = sm + (size_t)kFMI * LD;   // [4 kFMP][LD] mode-gradient rows (p, r)
  double* sU = sB;                       // [kFMI][4][kFUP] after the MMA
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int gid = lane >> 2, tig = lane & 3;
  const int p0 = blockIdx.x * kFMP;
  const int64_t s0 = (int64_t)blockIdx.y * kFMI;
  {  // whole CTA idle (finished / failed instances): skip
    __shared__ int any_active;
    if (tid == 0) any_active = 0;
    __syncthreads();
    if (tid < kFMI && s0 + tid < g.n && g.ctl[inst_of(g.alist, s0 + tid)].active) any_active = 1;
    __syncthreads();
    if (!any_active) return;
  }
  // staging: each thread's loads are all issued before its shared-memory
  // stores (kFB in flight), so the tile arrives at memory-level parallelism
  // rather than one dependent round trip per element
  constexpr int kFB = 8;
  for (int t0 = 0; t0 < kFMI * KP; t0 += 256 * kFB) {
    double v[kFB];
#pragma unroll
    for (int u = 0; u < kFB; ++u) {
      const int t = t0 + u * 256 + tid;
      const int si = t / KP, k = t - si * KP;
      v[u] = (t < kFMI * KP && k < N && s0 + si < g.n) ? g.a[(size_t)inst_of(g.alist, s0 + si) * N + k] : 0.0;
    }
#pragma unroll
    for (int u = 0; u < kFB; ++u) {
      const int t = t0 + u * 256 + tid;
      const int si = t / KP, k = t - si * KP;
      if (t < kFMI * KP) sA[si * LD + k] = v[u];
    }
  }
  const int R0 = p0 * 4, RQ = g.Qpad * 4;
  for (int t0 = 0; t0 < kFMP * 4 * KP; t0 += 256 * kFB) {
    double v[kFB];
#pragma unroll
    for (int u = 0; u < kFB; ++u) {
      const int t = t0 + u * 256 + tid;
      const int rr = t / KP, k = t - rr * KP;
      v[u] = (t < kFMP * 4 * KP && R0 + rr < RQ) ? __ldg(G + (size_t)(R0 + rr) * NP + k) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < kFB; ++u) {
      const int t = t0 + u * 256 + tid;
      const int rr = t / KP, k = t - rr * KP;
      if (t < kFMP * 4 * KP) sB[rr * LD + k] = v[u];
    }
  }
  __syncthreads();
  const int mt = warp & 3, nt0 = (warp >> 2) * 8;
  double acc[8][2];
#pragma unroll
  for (int j = 0; j < 8; ++j) acc[j][0] = acc[j][1] = 0.0;
  for (int ks = 0; ks < KP; ks += 4) {
    const double afr = sA[(mt * 8 + gid) * LD + ks + tig];
#pragma unroll
    for (int j = 0; j < 8; ++j) dmma(acc[j][0], acc[j][1], afr, sB[((nt0 + j) * 8 + gid) * LD + ks + tig]);
  }
  __syncthreads();  // sB is reused as sU
#pragma unroll
  for (int j = 0; j < 8; ++j)
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int row = (nt0 + j) * 8 + 2 * tig + h;  // point-row (pl, r) of the tile
      sU[((mt * 8 + gid) * 4 + (row & 3)) * kFUP + (row >> 2)] = acc[j][h];
    }
  __syncthreads();
  const int p = p0 + lane;
  if (p >= g.Q) return;
  // the warp's instances: control words and morph loads issued up front
  int64_t sq[kFMI / 8];
  bool act[kFMI / 8];
  int top[kFMI / 8];
  double m[kFMI / 8][4];
#pragma unroll
  for (int q = 0; q < kFMI / 8; ++q) {
    const int si = warp + 8 * q;
    sq[q] = s0 + si < g.n ? inst_of(g.alist, s0 + si) : -1;
    act[q] = sq[q] >= 0 && g.ctl[sq[q]].active;
    top[q] = act[q] ? g.ctl[sq[q]].sp - 1 : 0;
    const double* mo = g.morph + (size_t)(act[q] ? sq[q] : 0) * 5 * g.Q;
#pragma unroll
    for (int t = 0; t < 4; ++t) m[q][t] = act[q] ? mo[(size_t)t * g.Q + p] : 0.0;
  }
#pragma unroll
  for (int q = 0; q < kFMI / 8; ++q) {
    const int si = warp + 8 * q;
    if (!act[q]) continue;
    const int64_t s = sq[q];
    const RomCtl* c = g.ctl + s;
    double u[4];
#pragma unroll
    for (int r = 0; r < 4; ++r) u[r] = sU[(si * 4 + r) * kFUP + lane];
#pragma unroll
    for (int ii = 0; ii < 2; ++ii)
#pragma unroll
      for (int l = 0; l < 2; ++l)
        g.Fb[((size_t)s * 4 + ii + 2 * l) * g.Q + p] =
            c->fstack[top[q]][4 + ii + 2 * l] + (u[ii] * m[q][2 * l] + u[ii + 2] * m[q][1 + 2 * l]);
  }
}

// Material at every ECM point (one thread per point, C1-style register
// budget): P, FD tangent, trial history, then the mapped operators
// At = c R A R^T and Pt = c R P.  ABAR (rom_effective_stiffness,
// rom.cpp:206-207): history from g.S0, no trial history, and c A kept too.
// MODE (lazy-tangent pipeline): 0 everything, 1 P / Pt / trial history only,
// 2 the tangent only, for the instances g.list[0 .. *g.count).
// SLAB: the FD loop runs over a shared-memory slab column (material.cuh,
// SlabSrc), which frees the registers for more resident warps.
template <int MINB, bool ABAR = false, int MODE = 0, bool SLAB = false>
__global__ void __launch_bounds__(128, MINB) k_rom_point(PointArgs g, MatTable tab) {
  constexpr int kSlabS = 128;
  __shared__ double slab[(SLAB && MODE != 1) ? kSlabSlots * kSlabS : 1];
  const int tid = blockIdx.x * blockDim.x + threadIdx.x;
  if (tid >= g.n * g.Q) return;
  int64_t s;
  int p;
  if (MODE == 2) {
    const int j = tid / g.Q;
    if (j >= *g.count) return;
    s = g.list[j];
    p = tid - j * g.Q;
  } else {
    const int64_t k = tid / g.Q;
    p = tid - (int)k * g.Q;
    s = inst_of(g.alist, k);
  }
  RomCtl* c = g.ctl + s;
  if (!c->active) return;
  const double* mo = g.morph + (size_t)s * 5 * g.Q;
  double m[4], F[4];
#pragma unroll
  for (int t = 0; t < 4; ++t) {
    m[t] = mo[(size_t)t * g.Q + p];
    F[t] = g.Fb[((size_t)s * 4 + t) * g.Q + p];
  }
  const double det = mo[(size_t)4 * g.Q + p];
  const MatConst& pm = tab.m[g.reg[p]];
  const int cur = c->cur;
  const double* s0p = ABAR ? g.S0 + (size_t)s * 6 * g.Q : g.S + ((size_t)cur * g.cap + s) * 6 * g.Q;
  double* s1p = g.S + ((size_t)(cur ^ 1) * g.cap + s) * 6 * g.Q;
  double fp[4];
#pragma unroll
  for (int t = 0; t < 4; ++t) fp[t] = s0p[(size_t)t * g.Q + p];
  Frozen z;
  freeze(fp, s0p[(size_t)4 * g.Q + p], s0p[(size_t)5 * g.Q + p], z);
  const double cw = g.w[p] * det;  // rom.cpp:56
  // Ã_p and P̃_p as planes [s][20][Qpad] (entry t at at[t * Qpad]): a warp's
  // stores of one entry are one contiguous run of points
  double* at = g.At + (size_t)s * 20 * g.Qpad + p;
  const size_t aqs = (size_t)g.Qpad;
  bool ok = true;
  constexpr bool kSlab = SLAB && MODE != 1;
  volatile double* sc = slab + threadIdx.x;
  if constexpr (kSlab) slab_put<kSlabS>(sc, F, z);
  if (MODE != 2) {
    double P[4];
    FullOut fo;
    if constexpr (kSlab)
      ok = lsu_eval_src<true>(pm, SlabSrc<kSlabS>{sc}, P, &fo);
    else
      ok = lsu_eval<true>(pm, z, F, P, &fo);
    if (!ABAR) {
#pragma unroll
      for (int t = 0; t < 4; ++t) s1p[(size_t)t * g.Q + p] = fo.fp[t];
      s1p[(size_t)4 * g.Q + p] = fo.fpzz;
      s1p[(size_t)5 * g.Q + p] = fo.xi;
    }
    double* Pp = g.P + ((size_t)s * g.Q + p) * 4;
#pragma unroll
    for (int t = 0; t < 4; ++t) Pp[t] = P[t];
    // Pt = c R P : (R P)[i + 2j] = sum_l m(j,l) P[i + 2l]
    double pt[4];
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const int i = r & 1, j = r >> 1;
      pt[r] = cw * (m[j] * P[i] + m[j + 2] * P[i + 2]);
    }
    if (MODE == 1)  // read back by k_rom_check only (32 B per point, not a 160 B At row)
      *reinterpret_cast<double4*>(g.Pt + ((size_t)s * g.Qpad + p) * 4) = make_double4(pt[0], pt[1], pt[2], pt[3]);
    else
#pragma unroll
      for (int r = 0; r < 4; ++r) at[(16 + r) * aqs] = pt[r];
  }
  if (ok && MODE != 1) {
    // At = c R A R^T streamed per column pair: columns e = (s&1) + 2l' arrive
    // in the order 0, 2, 1, 3, so after each pair the four entries of both
    // output columns s in {e&1, (e&1)+2} are final.  T = R col:
    // T[r] = sum_l m(r>>1, l) col[(r&1) + 2l].
    double T0[4];
    auto sink = [&](int e, const double col[4]) {
      if (ABAR) {
        double* ca = g.CA + ((size_t)s * g.Q + p) * 16 + 4 * e;
#pragma unroll
        for (int r = 0; r < 4; ++r) ca[r] = cw * col[r];
      }
      double Tc[4];
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        const int i = r & 1, j = r >> 1;
        Tc[r] = fma(m[j + 2], col[i + 2], m[j] * col[i]);
      }
      if (e < 2) {
#pragma unroll
        for (int r = 0; r < 4; ++r) T0[r] = Tc[r];
        return;
      }
      const int sb = e & 1;  // output columns sb and sb + 2
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int sc = sb + 2 * h, js = sc >> 1;
#pragma unroll
        for (int r = 0; r < 4; ++r) at[(r + 4 * sc) * aqs] = cw * fma(Tc[r], m[js + 2], T0[r] * m[js]);
      }
    };
    if constexpr (kSlab) {
      ok = fd_tangent_slab<kSlabS>(pm, sc, 1e-7, sink);
    } else {
      ok = fd_tangent<false>(pm, z, F, 1e-7, sink);
    }
  }
  if (!ok) c->asm_fail = 1;  // SolveError inside rom_assemble -> attempt fails
}

// ---- K and f: DMMA contraction ---------------------------------------------
struct ContractArgs {
  int64_t n;
  int N, Q, Qpad, NT, NP;
  const double* G;   // [Qpad*4][NP]
  const double* At;  // [n][Qpad][20]
  double* K;         // [n][N][N]
  double* f;         // [n][N]
  const RomCtl* ctl;
  const int* list;   // nullable: CTA slots index this compacted instance list
  const int* count;
};


// Software-pipelined over chunks of kPC points: while the warps run the DMMA
// k-steps of chunk c they also build Y for chunk c+1 (independent SMEM
// buffers, so the DFMA and DMMA streams interleave) and have the global loads
// of chunk c+2 in flight in registers.  Two barriers per chunk.
// SMEM rows are padded to NT*8 + 4 doubles: the m8n8k4 fragment loads
// (row = k + tig, col = 8 t + gid) then hit 32 distinct bank pairs per
// half-warp (an unpadded 56-double row gives 2-way conflicts).
template <int NT>
__host__ __device__ constexpr int contract_ld() {
  return NT * 8 + 4;
}
// instances per CTA: two for the usual tile widths, one for wide ones (SMEM)
template <int NT>
__host__ __device__ constexpr int contract_ipc() {
  return NT <= 7 ? kIPC : 1;
}
template <int NT, int IPC = contract_ipc<NT>()>
constexpr size_t contract_smem_bytes() {
  return sizeof(double) * (2 * (kPC * 4) * contract_ld<NT>() + 2 * IPC * (kPC * 4) * contract_ld<NT>() +
                           2 * IPC * kPC * 20);
}

// two-instance CTAs: 2 resident per SM when the SMEM allows, as a register
// bound too, so a register-hungrier variant cannot silently halve occupancy
template <int NT, int IPC>
constexpr int contract_minb() {
  return IPC > 1 && (228 * 1024) / (contract_smem_bytes<NT, IPC>() + 1024) >= 2 ? 2 : 1;
}

template <int NT, int IPC = contract_ipc<NT>(), bool LIST = false>
__global__ void __launch_bounds__(32 * NT * IPC, (contract_minb<NT, IPC>())) k_rom_contract(ContractArgs g) {
  constexpr int kIPC = IPC;
  constexpr int NP = NT * 8;
  constexpr int LDY = contract_ld<NT>();
  constexpr int KR = kPC * 4;  // k-rows per chunk
  constexpr int NTHR = 32 * NT * kIPC;
  constexpr int GPT = (KR * NP + NTHR - 1) / NTHR;  // Gm doubles per thread per chunk
  constexpr int APT = (kIPC * kPC * 20 + NTHR - 1) / NTHR;  // At doubles per thread
  extern __shared__ double smc[];
  double* sGm = smc;                        // [2][KR][LDY]
  double* sY = sGm + 2 * KR * LDY;          // [2][kIPC][KR][LDY]
  double* sAt = sY + 2 * kIPC * KR * LDY;   // [2][kIPC][kPC][20]
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int si = warp / NT, trow = warp - si * NT;
  const int64_t sbase = (int64_t)blockIdx.x * kIPC;
  // LIST: CTA slots index the compacted instance list (lazy tangent)
  int64_t sid[kIPC];
  if constexpr (LIST) {
    const int64_t lim = *g.count;
#pragma unroll
    for (int q = 0; q < kIPC; ++q) sid[q] = sbase + q < lim ? (int64_t)g.list[sbase + q] : -1;
  }
  bool any = false;
  if constexpr (LIST) {
#pragma unroll
    for (int q = 0; q < kIPC; ++q)
      if (sid[q] >= 0) any = true;
  } else {
    for (int q = 0; q < kIPC; ++q)
      if (sbase + q < g.n && g.ctl[sbase + q].active) any = true;
  }
  if (!any) return;
  const int gid = lane >> 2, tig = lane & 3;
  double acc[NT][2];
#pragma unroll
  for (int ct = 0; ct < NT; ++ct) acc[ct][0] = acc[ct][1] = 0.0;
  const int nch = g.Qpad / kPC;
  double rG[GPT], rA[APT];

  auto gload = [&](int c) {
    const double* gsrc = g.G + (size_t)c * kPC * 4 * NP;
#pragma unroll
    for (int k = 0; k < GPT; ++k) {
      const int t = tid + k * NTHR;
      rG[k] = t < KR * NP ? gsrc[t] : 0.0;
    }
#pragma unroll
    for (int k = 0; k < APT; ++k) {
      const int t = tid + k * NTHR;
      rA[k] = 0.0;
      if (t < kIPC * kPC * 20) {
        const int q = t / (kPC * 20), rem = t - q * kPC * 20;
        const int tp = rem / kPC, pl = rem - tp * kPC;  // At planes [s][20][Qpad], points fastest
        if constexpr (LIST) {
          int64_t sq = sid[0];
#pragma unroll
          for (int u = 1; u < kIPC; ++u)
            if (q == u) sq = sid[u];
          if (sq >= 0) rA[k] = g.At[((size_t)sq * 20 + tp) * g.Qpad + (size_t)c * kPC + pl];
        } else {
          const int64_t sq = sbase + q;
          if (sq < g.n) rA[k] = g.At[((size_t)sq * 20 + tp) * g.Qpad + (size_t)c * kPC + pl];
        }
      }
    }
  };
  auto gstore = [&](int buf) {
#pragma unroll
    for (int k = 0; k < GPT; ++k) {
      const int t = tid + k * NTHR;
      if (t < KR * NP) sGm[buf * KR * LDY + (t / NP) * LDY + t % NP] = rG[k];
    }
#pragma unroll
    for (int k = 0; k < APT; ++k) {
      const int t = tid + k * NTHR;
      if (t < kIPC * kPC * 20) {  // back to the [instance][point][20] shared layout of build_y
        const int q = t / (kPC * 20), rem = t - q * kPC * 20;
        const int tp = rem / kPC, pl = rem - tp * kPC;
        sAt[buf * kIPC * kPC * 20 + q * kPC * 20 + pl * 20 + tp] = rA[k];
      }
    }
  };
  // Y[(p,r)][j] = sum_t At_p[r][t] Gm[(p,t)][j] (j < N); Y[.][N] = Pt; else 0.
  // One thread per (instance, point, column j) builds the 4 rows r of that
  // point: the 4 Gm values are loaded once and At_p comes as broadcast
  // 128-bit loads, so Y costs ~2.8x fewer SMEM wavefronts than per element.
  auto build_y = [&](int buf) {
    const double* G0 = sGm + buf * KR * LDY;
    for (int t = tid; t < kIPC * kPC * NP; t += NTHR) {
      const int q = t / (kPC * NP), rem = t - q * kPC * NP;
      const int pl = rem / NP, j = rem - pl * NP;
      const double* at = sAt + (buf * kIPC + q) * kPC * 20 + pl * 20;
      double* y = sY + (buf * kIPC + q) * KR * LDY + (pl * 4) * LDY + j;
      if (j < g.N) {
        const double g0 = G0[(pl * 4) * LDY + j], g1 = G0[(pl * 4 + 1) * LDY + j];
        const double g2 = G0[(pl * 4 + 2) * LDY + j], g3 = G0[(pl * 4 + 3) * LDY + j];
        const double4 c0 = *reinterpret_cast<const double4*>(at);       // At[r][0], r = 0..3
        const double4 c1 = *reinterpret_cast<const double4*>(at + 4);   // At[r][1]
        const double4 c2 = *reinterpret_cast<const double4*>(at + 8);
        const double4 c3 = *reinterpret_cast<const double4*>(at + 12);
        y[0] = fma(c3.x, g3, fma(c2.x, g2, fma(c1.x, g1, c0.x * g0)));
        y[LDY] = fma(c3.y, g3, fma(c2.y, g2, fma(c1.y, g1, c0.y * g0)));
        y[2 * LDY] = fma(c3.z, g3, fma(c2.z, g2, fma(c1.z, g1, c0.z * g0)));
        y[3 * LDY] = fma(c3.w, g3, fma(c2.w, g2, fma(c1.w, g1, c0.w * g0)));
      } else if (j == g.N) {
        const double4 pt = *reinterpret_cast<const double4*>(at + 16);
        y[0] = pt.x;
        y[LDY] = pt.y;
        y[2 * LDY] = pt.z;
        y[3 * LDY] = pt.w;
      } else {
        y[0] = y[LDY] = y[2 * LDY] = y[3 * LDY] = 0.0;
      }
    }
  };
  auto mma = [&](int buf) {
    const double* G0 = sGm + buf * KR * LDY;
    const double* Y0 = sY + (buf * kIPC + si) * KR * LDY;
#pragma unroll
    for (int ks = 0; ks < KR / 4; ++ks) {
      const double afr = G0[(ks * 4 + tig) * LDY + trow * 8 + gid];  // (Gm^T)[i][k]
#pragma unroll
      for (int ct = 0; ct < NT; ++ct) dmma(acc[ct][0], acc[ct][1], afr, Y0[(ks * 4 + tig) * LDY + ct * 8 + gid]);
    }
  };

  gload(0);
  gstore(0);
  __syncthreads();
  build_y(0);
  if (nch > 1) {
    gload(1);
    gstore(1);
  }
  __syncthreads();
  for (int c = 0; c < nch; ++c) {
    const int cur = c & 1, nxt = cur ^ 1;
    if (c + 2 < nch) gload(c + 2);
    if (c + 1 < nch) build_y(nxt);
    mma(cur);
    __syncthreads();
    if (c + 2 < nch) gstore(cur);
    __syncthreads();
  }
  int64_t s = sbase + si;
  if constexpr (LIST) {
    s = sid[0];
#pragma unroll
    for (int u = 1; u < kIPC; ++u)
      if (si == u) s = sid[u];
    if (s < 0) return;
  } else {
    if (s >= g.n || !g.ctl[s].active) return;
  }
  const int i = trow * 8 + gid;
  if (i >= g.N) return;
#pragma unroll
  for (int ct = 0; ct < NT; ++ct)
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int j = ct * 8 + 2 * tig + h;
      if (j < g.N)
        g.K[((size_t)s * g.N + i) * g.N + j] = acc[ct][h];
      else if (j == g.N && !LIST)  // LIST: f comes from k_rom_check (the Pt column is stale here)
        g.f[(size_t)s * g.N + i] = acc[ct][h];
    }
}

// ---- remainder-packed contraction (lazy pipeline, N = 8 NTM + 1 or 2) --------
// For N = 50 the 56-wide tiling above spends 13 of its 49 DMMA tiles per
// k-step on the two remainder rows and columns.  Here the NTM x NTM block of
// full tiles runs as above (NTM warps per instance, NTM column tiles each),
// and the remainder of BOTH instances of the CTA is one 8-column B tile for
// one extra warp: with Zc = Gm[:, 8 NTM ..] (the last 1-2 mode columns),
//   K[:, 8NTM + m]  = Gm^T (D Zc)      (the usual Y columns)        m < 2
//   K[8NTM + m, :]^T = Gm^T (D^T Zc)   (the rows, through the transposed At)
// so B = [D Zc | D^T Zc] of instance 0, then of instance 1: NTM + 1 tiles per
// k-step for the pair.  Per pair and k-step 2 NTM^2 + NTM + 1 DMMAs instead of
// 2 (NTM + 1)^2: 79 against 98 for N = 50.  The remainder rows are summed over
// D^T Zc instead of Y, so they differ from the 56-wide kernel's by rounding;
// every other entry is the same sum in the same order.
template <int NTM, int IPC>
constexpr size_t contract_rp_smem_bytes() {
  return sizeof(double) * (2 * (kPC * 4) * contract_ld<NTM + 1>() + 2 * IPC * (kPC * 4) * (NTM * 8 + 4) +
                           2 * (kPC * 4) * 12 + 2 * IPC * kPC * 20);
}

// Warps own a 2 x 3 block of tiles (row-tile pair x column-tile triple: 5
// fragment loads per 6 DMMAs instead of 7; the kernel is bound by the
// shared-memory data pipe and by warp balance, not by the DMMA pipe).  The
// remainder tile's NTM + 1 row tiles ride on four of the warps, on different
// SM sub-partitions (warp w runs on sub-partition w % 4): three add the two
// row tiles of their own A fragments, one the last (padded) row tile; with
// two instances per CTA every sub-partition issues 38-40 DMMAs per k-step.
// IPC = 1 (small batches: twice the CTAs) leaves half of the remainder tile
// empty and gives its row tiles to two extra warps (4 + 3 tiles: 12, 12, 10, 9
// DMMAs per k-step on the four sub-partitions); an instance's K has the same
// bits either way (its columns of the tile do not depend on the other
// instance's, and every tile is the same k-ordered DMMA chain).
template <int NTM, int IPC>
__global__ void __launch_bounds__(32 * (IPC * NTM + (IPC == 1 ? 2 : 0)), (IPC == 2 ? 2 : 3))
    k_rom_contract_rp(ContractArgs g) {
  static_assert(NTM == 6 && (IPC == 1 || IPC == 2), "warp roles below are laid out for 6 x 6 full tiles");
  constexpr int NT = NTM + 1;
  constexpr int NP = NT * 8;     // columns of the global Gm rows
  constexpr int NM = NTM * 8;    // modes in full tiles
  constexpr int LDG = contract_ld<NT>();
  constexpr int LDY = NM + 4;    // = 4 mod 16: conflict-free fragment loads
  constexpr int LDR = 12;        // 8 remainder columns + 4
  constexpr int KR = kPC * 4;
  constexpr int NWM = IPC * NTM;            // warps with a 2 x 3 block of full tiles
  constexpr int NW = NWM + (IPC == 1 ? 2 : 0);
  constexpr int NTHR = 32 * NW;
  constexpr int GPT = (KR * NP + NTHR - 1) / NTHR;
  constexpr int APT = (IPC * kPC * 16 + NTHR - 1) / NTHR;
  constexpr int CB = NTM / 3;    // column-triple blocks per instance
  constexpr int NRA = IPC == 1 ? 4 : 2;     // remainder accumulator tiles per warp
  static_assert(LDY % 16 == 4 || LDY % 16 == 12, "Y row stride");
  extern __shared__ double smc[];
  double* sGm = smc;                        // [2][KR][LDG]
  double* sY = sGm + 2 * KR * LDG;          // [2][IPC][KR][LDY]
  double* sR = sY + 2 * IPC * KR * LDY;     // [2][KR][LDR]
  double* sAt = sR + 2 * KR * LDR;          // [2][IPC][kPC][20]: At[r][t] at 4 r + t
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const bool mainw = warp < NWM;
  const int si = mainw ? warp / NTM : 0, wb = mainw ? warp - si * NTM : 0;
  const int rb = wb / CB, cb = wb - rb * CB;  // row tiles 2 rb, 2 rb + 1; column tiles 3 cb ..
  // IPC 2: remainder row tiles 2 rb, 2 rb + 1 (rb = 0, 1, 2) / row tile NTM ride on main warps
  const bool rem2 = IPC == 2 && (warp == 0 || warp == 9 || warp == 10);
  const bool rem7 = IPC == 2 && warp == 3;
  // IPC 1: warp NWM owns remainder row tiles 0..3, warp NWM + 1 tiles 4..NTM
  const int rt0 = warp == NWM ? 0 : 4, rtn = warp == NWM ? 4 : NT - 4;
  constexpr int kTailA = IPC == 2 ? 7 : 7, kTailB = IPC == 2 ? 11 : 7;  // warps building D Zc / D^T Zc
  const int64_t sbase = (int64_t)blockIdx.x * IPC;
  const int64_t lim = *g.count;
  int64_t sid[IPC];
  bool any = false;
#pragma unroll
  for (int q = 0; q < IPC; ++q) {
    sid[q] = sbase + q < lim ? (int64_t)g.list[sbase + q] : -1;
    any = any || sid[q] >= 0;
  }
  if (!any) return;
  const int gid = lane >> 2, tig = lane & 3;
  double acc[6][2];   // tile (h, c) of the block at acc[3 h + c]
  double accr[NRA][2];  // remainder row tiles of this warp (rem2: 2 rb + h; rem7: NTM at [0]; IPC 1: rt0 + h)
#pragma unroll
  for (int ct = 0; ct < 6; ++ct) acc[ct][0] = acc[ct][1] = 0.0;
#pragma unroll
  for (int ct = 0; ct < NRA; ++ct) accr[ct][0] = accr[ct][1] = 0.0;
  const int nch = g.Qpad / kPC;
  double rG[GPT], rA[APT];

  auto gload = [&](int c) {
    const double* gsrc = g.G + (size_t)c * kPC * 4 * NP;
#pragma unroll
    for (int k = 0; k < GPT; ++k) {
      const int t = tid + k * NTHR;
      rG[k] = t < KR * NP ? gsrc[t] : 0.0;
    }
#pragma unroll
    for (int k = 0; k < APT; ++k) {
      const int t = tid + k * NTHR;
      rA[k] = 0.0;
      if (t < IPC * kPC * 16) {
        const int q = t / (kPC * 16), rm = t - q * kPC * 16;
        const int tp = rm / kPC, pl = rm - tp * kPC;  // At planes [s][20][Qpad], points fastest
        const int64_t sq = (IPC == 2 && q) ? sid[IPC - 1] : sid[0];
        if (sq >= 0) rA[k] = g.At[((size_t)sq * 20 + tp) * g.Qpad + (size_t)c * kPC + pl];
      }
    }
  };
  auto gstore = [&](int buf) {
#pragma unroll
    for (int k = 0; k < GPT; ++k) {
      const int t = tid + k * NTHR;
      if (t < KR * NP) sGm[buf * KR * LDG + (t / NP) * LDG + t % NP] = rG[k];
    }
#pragma unroll
    for (int k = 0; k < APT; ++k) {
      const int t = tid + k * NTHR;
      if (t < IPC * kPC * 16) {
        const int q = t / (kPC * 16), rm = t - q * kPC * 16;
        const int tp = rm / kPC, pl = rm - tp * kPC;  // plane tp = r + 4 t holds At[r][t]
        sAt[buf * IPC * kPC * 20 + q * kPC * 20 + pl * 20 + 4 * (tp & 3) + (tp >> 2)] = rA[k];
      }
    }
  };
  // Item (instance q, point pl, column j): the 4 rows of Y column j (j >= NM:
  // into the remainder tile, columns 4 q + j - NM), row r from At's row r (one
  // 32-byte load) in the 56-wide kernel's FMA order.
  auto y_item = [&](const double* G0, int buf, int q, int pl, int j) {
    const double* at = sAt + (buf * IPC + q) * kPC * 20 + pl * 20;
    const double g0 = G0[(pl * 4) * LDG + j], g1 = G0[(pl * 4 + 1) * LDG + j];
    const double g2 = G0[(pl * 4 + 2) * LDG + j], g3 = G0[(pl * 4 + 3) * LDG + j];
    double* y = j < NM ? sY + (buf * IPC + q) * KR * LDY + (pl * 4) * LDY + j
                       : sR + buf * KR * LDR + (pl * 4) * LDR + q * 4 + (j - NM);
    const int ld = j < NM ? LDY : LDR;
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const double4 ar = *reinterpret_cast<const double4*>(at + 4 * r);  // At[r][0..3]
      y[r * ld] = fma(ar.w, g3, fma(ar.z, g2, fma(ar.y, g1, ar.x * g0)));
    }
  };
  // Two items per thread over the IPC x kPC x NM full-tile columns (a
  // half-warp = 16 consecutive columns of one point: conflict-free stores).
  // The IPC x kPC x 2 remainder columns D Zc and as many of D^T Zc go to the
  // tail warp(s), on the sub-partition with the fewest remainder DMMAs.
  static_assert(IPC * kPC * NM <= 2 * NTHR && NTHR % 16 == 0, "at most two full-tile columns per thread");
  auto build_y = [&](int buf) {
    const double* G0 = sGm + buf * KR * LDG;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int u = tid + h * NTHR;
      if (u >= IPC * kPC * NM) break;
      const int q = u / (kPC * NM), rm = u - q * kPC * NM;
      y_item(G0, buf, q, rm / NM, rm % NM);
    }
    if (warp != kTailA && warp != kTailB) return;
    // lane -> (instance or kind, point, m)
    const int hi = lane >> 4, pl = (lane >> 1) & (kPC - 1), m = lane & 1;
    const int q = IPC == 2 ? hi : 0;
    const bool tr = IPC == 2 ? warp == kTailB : hi == 1;
    if (!tr) {
      y_item(G0, buf, q, pl, NM + m);
    } else {  // (D^T Zc)[4p + t] = sum_r At[r][t] Zc[4p + r]
      const double* at = sAt + (buf * IPC + q) * kPC * 20 + pl * 20;
      const double g0 = G0[(pl * 4) * LDG + NM + m], g1 = G0[(pl * 4 + 1) * LDG + NM + m];
      const double g2 = G0[(pl * 4 + 2) * LDG + NM + m], g3 = G0[(pl * 4 + 3) * LDG + NM + m];
      double* y = sR + buf * KR * LDR + (pl * 4) * LDR + q * 4 + 2 + m;
#pragma unroll
      for (int t = 0; t < 4; ++t) y[t * LDR] = fma(at[12 + t], g3, fma(at[8 + t], g2, fma(at[4 + t], g1, at[t] * g0)));
    }
  };
  auto mma = [&](int buf) {
    const double* G0 = sGm + buf * KR * LDG;
    const double* Y0 = sY + (buf * IPC + si) * KR * LDY + cb * 24 + gid;
    const double* A0 = G0 + rb * 16 + gid;
    const double* R0 = sR + buf * KR * LDR + gid;
    if (IPC == 1 && !mainw) {  // remainder-only warp: its row tiles against the remainder B tile
      const double* Ar = G0 + rt0 * 8 + gid;
#pragma unroll
      for (int ks = 0; ks < KR / 4; ++ks) {
        const double br = R0[(ks * 4 + tig) * LDR];
#pragma unroll
        for (int t = 0; t < NRA; ++t)
          if (t < rtn) dmma(accr[t][0], accr[t][1], Ar[(ks * 4 + tig) * LDG + t * 8], br);
      }
      return;
    }
#pragma unroll
    for (int ks = 0; ks < KR / 4; ++ks) {
      const double a0 = A0[(ks * 4 + tig) * LDG], a1 = A0[(ks * 4 + tig) * LDG + 8];  // (Gm^T)[i][k]
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        const double b = Y0[(ks * 4 + tig) * LDY + c * 8];
        dmma(acc[c][0], acc[c][1], a0, b);
        dmma(acc[3 + c][0], acc[3 + c][1], a1, b);
      }
      if (rem2) {
        const double br = R0[(ks * 4 + tig) * LDR];
        dmma(accr[0][0], accr[0][1], a0, br);
        dmma(accr[1][0], accr[1][1], a1, br);
      } else if (rem7) {
        dmma(accr[0][0], accr[0][1], G0[(ks * 4 + tig) * LDG + NM + gid], R0[(ks * 4 + tig) * LDR]);
      }
    }
  };

  if constexpr (IPC == 1) {  // the unused half of the remainder tile stays zero
    for (int t = tid; t < 2 * KR * LDR; t += NTHR) sR[t] = 0.0;
  }
  gload(0);
  gstore(0);
  __syncthreads();
  build_y(0);
  if (nch > 1) {
    gload(1);
    gstore(1);
  }
  __syncthreads();
  for (int c = 0; c < nch; ++c) {
    const int cur = c & 1, nxt = cur ^ 1;
    if (c + 2 < nch) gload(c + 2);
    if (c + 1 < nch) build_y(nxt);
    mma(cur);
    __syncthreads();
    if (c + 2 < nch) gstore(cur);
    __syncthreads();
  }
  if (mainw) {
    const int64_t s = sid[IPC == 2 ? si : 0];
    if (s >= 0) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int i = (2 * rb + h) * 8 + gid;
#pragma unroll
        for (int c = 0; c < 3; ++c)
#pragma unroll
          for (int e = 0; e < 2; ++e)
            g.K[((size_t)s * g.N + i) * g.N + (3 * cb + c) * 8 + 2 * tig + e] = acc[3 * h + c][e];
      }
    }
  }
  if (IPC == 2 ? (!rem2 && !rem7) : mainw) return;
  // remainder tile columns n = 2 tig + e: instance n >> 2, item m = n & 3
  if (IPC == 1 && (tig >> 1)) return;
  const int64_t s = sid[IPC == 2 ? (tig >> 1) : 0];
  if (s < 0) return;
#pragma unroll
  for (int h = 0; h < NRA; ++h) {
    if (IPC == 2 ? (rem7 && h) : h >= rtn) break;
    const int i = (IPC == 2 ? (rem7 ? NTM : 2 * rb + h) : rt0 + h) * 8 + gid;
    if (i >= g.N) continue;
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int m = 2 * (tig & 1) + e;
      if (m < 2) {
        if (NM + m < g.N) g.K[((size_t)s * g.N + i) * g.N + NM + m] = accr[h][e];
      } else if (NM + m - 2 < g.N && i < NM) {
        g.K[((size_t)s * g.N + NM + m - 2) * g.N + i] = accr[h][e];
      }
    }
  }
}

// The large-batch form: four warps per instance, each a 3 x 3 block of tiles (6
// fragment loads per 9 DMMAs; 8 warps per two-instance CTA at 128 registers, no
// spills; fewer, fatter warps: barrier stalls 4.0 -> 1.5 per issue, DMMA pipe 62 ->
// 65 % against the 12-warp 2 x 3 form, 365.1 -> 353.0 ms at 16,384 instances).  The
// remainder row tiles ride on warps 0-3 (one per SM sub-partition: 20 / 20 / 20 / 19
// DMMAs per k-step).  Every tile is the same k-ordered DMMA chain as in
// k_rom_contract_rp, so K has the same bits.  Notes of the 2 x 3 form follow: warps
// own a 2 x 3 block of tiles (row-tile pair x column-tile triple: 5
// fragment loads per 6 DMMAs instead of 7; the kernel is bound by the
// shared-memory data pipe and by warp balance, not by the DMMA pipe).  The
// remainder tile's NTM + 1 row tiles ride on four of the warps, on different
// SM sub-partitions (warp w runs on sub-partition w % 4): three add the two
// row tiles of their own A fragments, one the last (padded) row tile; with
// two instances per CTA every sub-partition issues 38-40 DMMAs per k-step.
// IPC = 1 (small batches: twice the CTAs) leaves half of the remainder tile
// empty and gives its row tiles to two extra warps (4 + 3 tiles: 12, 12, 10, 9
// DMMAs per k-step on the four sub-partitions); an instance's K has the same
// bits either way (its columns of the tile do not depend on the other
// instance's, and every tile is the same k-ordered DMMA chain).
template <int NTM, int IPC>
__global__ void __launch_bounds__(128 * IPC, (IPC == 2 ? 2 : 3)) k_rom_contract_rp3(ContractArgs g) {
  static_assert(IPC == 1 || IPC == 2, "3 x 3 blocks: four warps per instance");
  static_assert(NTM == 6 && (IPC == 1 || IPC == 2), "warp roles below are laid out for 6 x 6 full tiles");
  constexpr int NT = NTM + 1;
  constexpr int NP = NT * 8;     // columns of the global Gm rows
  constexpr int NM = NTM * 8;    // modes in full tiles
  constexpr int LDG = contract_ld<NT>();
  constexpr int LDY = NM + 4;    // = 4 mod 16: conflict-free fragment loads
  constexpr int LDR = 12;        // 8 remainder columns + 4
  constexpr int KR = kPC * 4;
  constexpr int NWM = 4 * IPC;              // warps with a 3 x 3 block of full tiles
  constexpr int NW = NWM;
  constexpr int NTHR = 32 * NW;
  constexpr int GPT = (KR * NP + NTHR - 1) / NTHR;
  constexpr int APT = (IPC * kPC * 16 + NTHR - 1) / NTHR;
  constexpr int CB = 2;          // column-triple blocks per instance
  constexpr int NRA = IPC == 1 ? 4 : 2;     // remainder accumulator tiles per warp
  static_assert(LDY % 16 == 4 || LDY % 16 == 12, "Y row stride");
  extern __shared__ double smc[];
  double* sGm = smc;                        // [2][KR][LDG]
  double* sY = sGm + 2 * KR * LDG;          // [2][IPC][KR][LDY]
  double* sR = sY + 2 * IPC * KR * LDY;     // [2][KR][LDR]
  double* sAt = sR + 2 * KR * LDR;          // [2][IPC][kPC][20]: At[r][t] at 4 r + t
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const bool mainw = warp < NWM;
  const int si = warp >> 2, wb = warp & 3;
  const int rb = wb / CB, cb = wb - rb * CB;  // row tiles 3 rb .. 3 rb + 2; column tiles 3 cb ..
  // IPC 2: remainder row tiles 2 rb, 2 rb + 1 (rb = 0, 1, 2) / row tile NTM ride on main warps
  // remainder row tiles: warp 0: 0, 1 (its A fragments 0, 1); warp 1: 2 (A fragment 2) and NTM (extra
  // load); warp 2: 3, 4; warp 3: 5 -- one warp per SM sub-partition, 20 / 20 / 20 / 19 DMMAs per k-step
  const bool rem2 = warp == 0 || warp == 2;
  const bool rem7 = warp == 1;
  const bool rem1 = warp == 3;
  // IPC 1: warp NWM owns remainder row tiles 0..3, warp NWM + 1 tiles 4..NTM
  const int rt0 = warp == NWM ? 0 : 4, rtn = warp == NWM ? 4 : NT - 4;
  constexpr int kTailA = IPC == 2 ? 5 : 3, kTailB = IPC == 2 ? 7 : 3;  // warps building D Zc / D^T Zc
  const int64_t sbase = (int64_t)blockIdx.x * IPC;
  const int64_t lim = *g.count;
  int64_t sid[IPC];
  bool any = false;
#pragma unroll
  for (int q = 0; q < IPC; ++q) {
    sid[q] = sbase + q < lim ? (int64_t)g.list[sbase + q] : -1;
    any = any || sid[q] >= 0;
  }
  if (!any) return;
  const int gid = lane >> 2, tig = lane & 3;
  double acc[9][2];   // tile (h, c) of the block at acc[3 h + c]
  double accr[NRA][2];  // remainder row tiles of this warp (rem2: 2 rb + h; rem7: NTM at [0]; IPC 1: rt0 + h)
#pragma unroll
  for (int ct = 0; ct < 9; ++ct) acc[ct][0] = acc[ct][1] = 0.0;
#pragma unroll
  for (int ct = 0; ct < NRA; ++ct) accr[ct][0] = accr[ct][1] = 0.0;
  const int nch = g.Qpad / kPC;
  double rG[GPT], rA[APT];

  auto gload = [&](int c) {
    const double* gsrc = g.G + (size_t)c * kPC * 4 * NP;
#pragma unroll
    for (int k = 0; k < GPT; ++k) {
      const int t = tid + k * NTHR;
      rG[k] = t < KR * NP ? gsrc[t] : 0.0;
    }
#pragma unroll
    for (int k = 0; k < APT; ++k) {
      const int t = tid + k * NTHR;
      rA[k] = 0.0;
      if (t < IPC * kPC * 16) {
        const int q = t / (kPC * 16), rm = t - q * kPC * 16;
        const int tp = rm / kPC, pl = rm - tp * kPC;  // At planes [s][20][Qpad], points fastest
        const int64_t sq = (IPC == 2 && q) ? sid[IPC - 1] : sid[0];
        if (sq >= 0) rA[k] = g.At[((size_t)sq * 20 + tp) * g.Qpad + (size_t)c * kPC + pl];
      }
    }
  };
  auto gstore = [&](int buf) {
#pragma unroll
    for (int k = 0; k < GPT; ++k) {
      const int t = tid + k * NTHR;
      if (t < KR * NP) sGm[buf * KR * LDG + (t / NP) * LDG + t % NP] = rG[k];
    }
#pragma unroll
    for (int k = 0; k < APT; ++k) {
      const int t = tid + k * NTHR;
      if (t < IPC * kPC * 16) {
        const int q = t / (kPC * 16), rm = t - q * kPC * 16;
        const int tp = rm / kPC, pl = rm - tp * kPC;  // plane tp = r + 4 t holds At[r][t]
        sAt[buf * IPC * kPC * 20 + q * kPC * 20 + pl * 20 + 4 * (tp & 3) + (tp >> 2)] = rA[k];
      }
    }
  };
  // Item (instance q, point pl, column j): the 4 rows of Y column j (j >= NM:
  // into the remainder tile, columns 4 q + j - NM), row r from At's row r (one
  // 32-byte load) in the 56-wide kernel's FMA order.
  auto y_item = [&](const double* G0, int buf, int q, int pl, int j) {
    const double* at = sAt + (buf * IPC + q) * kPC * 20 + pl * 20;
    const double g0 = G0[(pl * 4) * LDG + j], g1 = G0[(pl * 4 + 1) * LDG + j];
    const double g2 = G0[(pl * 4 + 2) * LDG + j], g3 = G0[(pl * 4 + 3) * LDG + j];
    double* y = j < NM ? sY + (buf * IPC + q) * KR * LDY + (pl * 4) * LDY + j
                       : sR + buf * KR * LDR + (pl * 4) * LDR + q * 4 + (j - NM);
    const int ld = j < NM ? LDY : LDR;
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const double4 ar = *reinterpret_cast<const double4*>(at + 4 * r);  // At[r][0..3]
      y[r * ld] = fma(ar.w, g3, fma(ar.z, g2, fma(ar.y, g1, ar.x * g0)));
    }
  };
  // Two items per thread over the IPC x kPC x NM full-tile columns (a
  // half-warp = 16 consecutive columns of one point: conflict-free stores).
  // The IPC x kPC x 2 remainder columns D Zc and as many of D^T Zc go to the
  // tail warp(s), on the sub-partition with the fewest remainder DMMAs.
  static_assert(IPC * kPC * NM == 3 * NTHR && NTHR % 16 == 0, "three full-tile columns per thread");
  auto build_y = [&](int buf) {
    const double* G0 = sGm + buf * KR * LDG;
#pragma unroll
    for (int h = 0; h < 3; ++h) {
      const int u = tid + h * NTHR;
      const int q = u / (kPC * NM), rm = u - q * kPC * NM;
      y_item(G0, buf, q, rm / NM, rm % NM);
    }
    if (warp != kTailA && warp != kTailB) return;
    // lane -> (instance or kind, point, m)
    const int hi = lane >> 4, pl = (lane >> 1) & (kPC - 1), m = lane & 1;
    const int q = IPC == 2 ? hi : 0;
    const bool tr = IPC == 2 ? warp == kTailB : hi == 1;
    if (!tr) {
      y_item(G0, buf, q, pl, NM + m);
    } else {  // (D^T Zc)[4p + t] = sum_r At[r][t] Zc[4p + r]
      const double* at = sAt + (buf * IPC + q) * kPC * 20 + pl * 20;
      const double g0 = G0[(pl * 4) * LDG + NM + m], g1 = G0[(pl * 4 + 1) * LDG + NM + m];
      const double g2 = G0[(pl * 4 + 2) * LDG + NM + m], g3 = G0[(pl * 4 + 3) * LDG + NM + m];
      double* y = sR + buf * KR * LDR + (pl * 4) * LDR + q * 4 + 2 + m;
#pragma unroll
      for (int t = 0; t < 4; ++t) y[t * LDR] = fma(at[12 + t], g3, fma(at[8 + t], g2, fma(at[4 + t], g1, at[t] * g0)));
    }
  };
  auto mma = [&](int buf) {
    const double* G0 = sGm + buf * KR * LDG;
    const double* Y0 = sY + (buf * IPC + si) * KR * LDY + cb * 24 + gid;
    const double* A0 = G0 + rb * 24 + gid;
    const double* R0 = sR + buf * KR * LDR + gid;
#pragma unroll
    for (int ks = 0; ks < KR / 4; ++ks) {
      double av[3];
#pragma unroll
      for (int h = 0; h < 3; ++h) av[h] = A0[(ks * 4 + tig) * LDG + h * 8];  // (Gm^T)[i][k]
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        const double b = Y0[(ks * 4 + tig) * LDY + c * 8];
#pragma unroll
        for (int h = 0; h < 3; ++h) dmma(acc[3 * h + c][0], acc[3 * h + c][1], av[h], b);
      }
      if (rem2) {
        const double br = R0[(ks * 4 + tig) * LDR];
        dmma(accr[0][0], accr[0][1], av[0], br);
        dmma(accr[1][0], accr[1][1], av[1], br);
      } else if (rem7) {
        const double br = R0[(ks * 4 + tig) * LDR];
        dmma(accr[0][0], accr[0][1], av[2], br);
        dmma(accr[1][0], accr[1][1], G0[(ks * 4 + tig) * LDG + NM + gid], br);
      } else if (rem1) {
        dmma(accr[0][0], accr[0][1], av[2], R0[(ks * 4 + tig) * LDR]);
      }
    }
  };

  if constexpr (IPC == 1) {  // the unused half of the remainder tile stays zero
    for (int t = tid; t < 2 * KR * LDR; t += NTHR) sR[t] = 0.0;
  }
  gload(0);
  gstore(0);
  __syncthreads();
  build_y(0);
  if (nch > 1) {
    gload(1);
    gstore(1);
  }
  __syncthreads();
  for (int c = 0; c < nch; ++c) {
    const int cur = c & 1, nxt = cur ^ 1;
    if (c + 2 < nch) gload(c + 2);
    if (c + 1 < nch) build_y(nxt);
    mma(cur);
    __syncthreads();
    if (c + 2 < nch) gstore(cur);
    __syncthreads();
  }
  {
    const int64_t s = sid[IPC == 2 ? si : 0];
    if (s >= 0) {
#pragma unroll
      for (int h = 0; h < 3; ++h) {
        const int i = (3 * rb + h) * 8 + gid;
#pragma unroll
        for (int c = 0; c < 3; ++c)
#pragma unroll
          for (int e = 0; e < 2; ++e)
            g.K[((size_t)s * g.N + i) * g.N + (3 * cb + c) * 8 + 2 * tig + e] = acc[3 * h + c][e];
      }
    }
  }
  if (!rem2 && !rem7 && !rem1) return;
  // remainder tile columns n = 2 tig + e: instance n >> 2, item m = n & 3
  if (IPC == 1 && (tig >> 1)) return;
  const int64_t s = sid[IPC == 2 ? (tig >> 1) : 0];
  if (s < 0) return;
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    if (rem1 && h) break;
    // row tile of accr[h]: warp 0: h; warp 2: 3 + h; warp 1: 2, NTM; warp 3: 5
    const int rt = rem2 ? 3 * rb + h : (rem7 ? (h ? NTM : 2) : 5);
    const int i = rt * 8 + gid;
    if (i >= g.N) continue;
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int m = 2 * (tig & 1) + e;
      if (m < 2) {
        if (NM + m < g.N) g.K[((size_t)s * g.N + i) * g.N + NM + m] = accr[h][e];
      } else if (NM + m - 2 < g.N && i < NM) {
        g.K[((size_t)s * g.N + NM + m - 2) * g.N + i] = accr[h][e];
      }
    }
  }
}

// ---- Newton / bisection state machine + LU --------------------------------
struct NewtonArgs {
  int64_t n;
  int N, Q, K, max_iter, max_bisect;
  double eps_rel, eps_abs, force_ref;
  const double* Kg;
  const double* f;
  const double* P;
  const double* morph;
  const double* w;
  const double* sched;
  double* a;
  double* a0;
  RomCtl* ctl;
  double* pbar;
  int32_t* iters;
  double* resid;
  double* a_final;
  int32_t* status;
  int* nactive;
  unsigned int* fail;
  const double* S;  // [2][cap][6][Q]
  int64_t cap;
  double* Sprev;  // nullable: committed history at the start of increment K-1
  const double* force_ref_inst;  // nullable [n]: per-instance force_ref (RomMicroEngine)
  double* init_res;              // nullable [n][K]: RomStepResult::initial_residual
  double* a_hist = nullptr;      // nullable [n][K][N]: RomSolution::steps[k].a
  // lazy-tangent pipeline (k_rom_check / k_rom_solve)
  const double* G;   // Gm [Qpad*4][NP]
  const double* Pt;  // compact Pt [n][Qpad][4] (k_rom_point MODE 1)
  int Qpad, NP;
  double* f_out;
  int* list;
  int* count;
  const int* alist = nullptr;  // k_rom_check: instance of entry k (n = entries)
};

constexpr int kNW = 1;  // warps (instances) per Newton CTA (SMEM-bound: 10 per SM)

// Dense LU with partial pivoting (Eigen PartialPivLU semantics: pivot = first
// row of max |a_ik|, rows swapped whole, unit-lower L) of the column-major
// Ks (ld LD) in SMEM by one warp, solving NR right-hand sides rhs[c*N + i] in
// place: the forward substitution is fused into the elimination and the
// transpositions are applied to the RHS in order (PartialPivLU::solve).
template <int NR>
__device__ __forceinline__ void warp_lu_solve(double* Ks, int LD, int N, double* rhs, int lane) {
  for (int k = 0; k < N; ++k) {
    double best = -1.0;
    int bi = N;
    for (int i = k + lane; i < N; i += 32) {
      const double v = fabs(Ks[k * LD + i]);
      if (v > best) {
        best = v;
        bi = i;
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double ob = __shfl_xor_sync(0xffffffffu, best, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (ob > best || (ob == best && oi < bi)) {
        best = ob;
        bi = oi;
      }
    }
    if (bi != k) {
      for (int j = lane; j < N; j += 32) {
        const double t0 = Ks[j * LD + k];
        Ks[j * LD + k] = Ks[j * LD + bi];
        Ks[j * LD + bi] = t0;
      }
      if (lane < NR) {
        const double t0 = rhs[lane * N + k];
        rhs[lane * N + k] = rhs[lane * N + bi];
        rhs[lane * N + bi] = t0;
      }
    }
    __syncwarp();
    const double d = Ks[k * LD + k];
    if (best != 0.0) {
      const double rd = __drcp_rn(d);  // correctly rounded: div_rcp == '/'
      for (int i = k + 1 + lane; i < N; i += 32) Ks[k * LD + i] = div_rcp(Ks[k * LD + i], d, rd);
    }
    __syncwarp();
    double bk[NR];
#pragma unroll
    for (int c = 0; c < NR; ++c) bk[c] = rhs[c * N + k];
    for (int i = k + 1 + lane; i < N; i += 32) {
      const double l = Ks[k * LD + i];
      // rank-1 update of the trailing block, 4 independent columns in flight
      int j = k + 1;
      for (; j + 3 < N; j += 4) {
        const double u0 = Ks[j * LD + k], u1 = Ks[(j + 1) * LD + k];
        const double u2 = Ks[(j + 2) * LD + k], u3 = Ks[(j + 3) * LD + k];
        const double a0 = Ks[j * LD + i], a1 = Ks[(j + 1) * LD + i];
        const double a2 = Ks[(j + 2) * LD + i], a3 = Ks[(j + 3) * LD + i];
        Ks[j * LD + i] = fma(-l, u0, a0);
        Ks[(j + 1) * LD + i] = fma(-l, u1, a1);
        Ks[(j + 2) * LD + i] = fma(-l, u2, a2);
        Ks[(j + 3) * LD + i] = fma(-l, u3, a3);
      }
      for (; j < N; ++j) Ks[j * LD + i] = fma(-l, Ks[j * LD + k], Ks[j * LD + i]);
#pragma unroll
      for (int c = 0; c < NR; ++c) rhs[c * N + i] = fma(-l, bk[c], rhs[c * N + i]);
    }
    __syncwarp();
  }
  // back substitution with U, lanes over rows
  for (int k = N - 1; k >= 0; --k) {
    const double ukk = Ks[k * LD + k];
    const double ru = __drcp_rn(ukk);
    double xk[NR];
#pragma unroll
    for (int c = 0; c < NR; ++c) xk[c] = div_rcp(rhs[c * N + k], ukk, ru);
    __syncwarp();
    if (lane < NR) {
      double v = xk[0];
#pragma unroll
      for (int c = 1; c < NR; ++c) v = (c == lane) ? xk[c] : v;
      rhs[lane * N + k] = v;
    }
    for (int i = lane; i < k; i += 32) {
      const double u = Ks[k * LD + i];
#pragma unroll
      for (int c = 0; c < NR; ++c) rhs[c * N + i] = fma(-u, xk[c], rhs[c * N + i]);
    }
    __syncwarp();
  }
}

// The same factorisation and solve (identical pivots and per-element FMA
// sequence) on a row-major A[i * N + j] as it arrives from global memory in
// one bulk copy: lanes over columns in the rank-1 update (conflict-free rows,
// the multipliers are warp broadcasts), one right-hand side.
__device__ __forceinline__ void warp_lu_solve_rm(double* A, int N, double* rhs, int lane) {
  for (int k = 0; k < N; ++k) {
    double best = -1.0;
    int bi = N;
    for (int i = k + lane; i < N; i += 32) {
      const double v = fabs(A[i * N + k]);
      if (v > best) {
        best = v;
        bi = i;
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double ob = __shfl_xor_sync(0xffffffffu, best, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (ob > best || (ob == best && oi < bi)) {
        best = ob;
        bi = oi;
      }
    }
    if (bi != k) {
      for (int j = lane; j < N; j += 32) {
        const double t0 = A[k * N + j];
        A[k * N + j] = A[bi * N + j];
        A[bi * N + j] = t0;
      }
      if (lane == 0) {
        const double t0 = rhs[k];
        rhs[k] = rhs[bi];
        rhs[bi] = t0;
      }
    }
    __syncwarp();
    const double d = A[k * N + k];
    if (best != 0.0) {
      const double rd = __drcp_rn(d);  // correctly rounded: div_rcp == '/'
      for (int i = k + 1 + lane; i < N; i += 32) A[i * N + k] = div_rcp(A[i * N + k], d, rd);
    }
    __syncwarp();
    const double bk = rhs[k];
    // rank-1 update, lanes over columns: a lane's columns j and j + 32 (the
    // second exists while N - k > 33) in one pass over 8-row chunks, so up to
    // 16 independent FMAs are in flight per chunk (same per-element FMA
    // sequence, bit-identical to a column-by-column loop)
    for (int j = k + 1 + lane; j < N; j += 64) {
      const int j2 = j + 32;
      const bool two = j2 < N;
      const double u = A[k * N + j], u2 = two ? A[k * N + j2] : 0.0;
      int i = k + 1;
      for (; i + 7 < N; i += 8) {
        double l[8], a[8], b[8];
#pragma unroll
        for (int r = 0; r < 8; ++r) l[r] = A[(i + r) * N + k];
#pragma unroll
        for (int r = 0; r < 8; ++r) a[r] = A[(i + r) * N + j];
        if (two) {
#pragma unroll
          for (int r = 0; r < 8; ++r) b[r] = A[(i + r) * N + j2];
        }
#pragma unroll
        for (int r = 0; r < 8; ++r) A[(i + r) * N + j] = fma(-l[r], u, a[r]);
        if (two) {
#pragma unroll
          for (int r = 0; r < 8; ++r) A[(i + r) * N + j2] = fma(-l[r], u2, b[r]);
        }
      }
      for (; i < N; ++i) {
        const double l = A[i * N + k];
        A[i * N + j] = fma(-l, u, A[i * N + j]);
        if (two) A[i * N + j2] = fma(-l, u2, A[i * N + j2]);
      }
    }
    for (int i = k + 1 + lane; i < N; i += 32) rhs[i] = fma(-A[i * N + k], bk, rhs[i]);
    __syncwarp();
  }
  for (int k = N - 1; k >= 0; --k) {  // back substitution with U, lanes over rows
    const double ukk = A[k * N + k];
    const double xk = div_rcp(rhs[k], ukk, __drcp_rn(ukk));
    __syncwarp();
    if (lane == 0) rhs[k] = xk;
    for (int i = lane; i < k; i += 32) rhs[i] = fma(-A[i * N + k], xk, rhs[i]);
    __syncwarp();
  }
}

// One cp.async.bulk global -> shared copy completing on an mbarrier (bytes
// and both addresses 16-byte aligned), issued and awaited by one warp.
__device__ __forceinline__ void warp_bulk_load(void* dst, const void* src, unsigned bytes, uint64_t* mbar,
                                               int lane) {
  const unsigned bar = (unsigned)__cvta_generic_to_shared(mbar);
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  if (lane == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(bar));
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::);
    asm volatile("fence.proxy.async.shared::cta;\n" ::);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(bar), "r"(bytes));
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(d),
        "l"(src), "r"(bytes), "r"(bar)
        : "memory");
  }
  __syncwarp();
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(bar)
      : "memory");
}

// The three outcomes of one Newton check (rom.cpp:129-150 with the adaptive
// wrapper :152-175), shared by the fused and the lazy-tangent pipelines.
__device__ __forceinline__ void rom_converged(const NewtonArgs& g, RomCtl* c, int64_t s, int lane, double r, int it) {
  const int N = g.N;
  // rom_effective_stress at the converged state (rom.cpp:68-76)
  const bool last_sub = c->sp == 1;
  if (last_sub) {  // lanes over points, fixed shuffle tree
    double pb[4] = {0.0, 0.0, 0.0, 0.0};
    const double* mo = g.morph + (size_t)s * 5 * g.Q;
    for (int p = lane; p < g.Q; p += 32) {
      const double cw = g.w[p] * mo[(size_t)4 * g.Q + p];
      const double4 P4 = *reinterpret_cast<const double4*>(g.P + ((size_t)s * g.Q + p) * 4);
      pb[0] += cw * P4.x;
      pb[1] += cw * P4.y;
      pb[2] += cw * P4.z;
      pb[3] += cw * P4.w;
    }
#pragma unroll
    for (int c4 = 0; c4 < 4; ++c4)
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) pb[c4] += __shfl_xor_sync(0xffffffffu, pb[c4], o);
    if (lane == 0)
      for (int c4 = 0; c4 < 4; ++c4) g.pbar[((size_t)s * g.K + c->k) * 4 + c4] = pb[c4] / 1.0;
  }
  for (int i = lane; i < N; i += 32) g.a0[(size_t)s * N + i] = g.a[(size_t)s * N + i];
  if (last_sub && g.a_hist) {  // the increment completes: steps[k].a (rom.cpp:191)
    const int k = c->k;
    for (int i = lane; i < N; i += 32) g.a_hist[((size_t)s * g.K + k) * N + i] = g.a[(size_t)s * N + i];
  }
  __syncwarp();
  int adv = 0;  // entered the last increment: keep its start history (run_online prev_states)
  if (lane == 0) {
    c->iters_acc += it;
    c->r0max = fmax(c->r0max, c->r0);  // rom.cpp:173 (failed attempts do not count)
    c->cur ^= 1;  // commit the trial history
    c->sp -= 1;
    c->it = 0;
    if (c->sp == 0) {
      if (g.init_res) g.init_res[(size_t)s * g.K + c->k] = c->r0max;
      c->r0max = 0.0;
      if (g.iters) g.iters[(size_t)s * g.K + c->k] = c->iters_acc;
      if (g.resid) g.resid[(size_t)s * g.K + c->k] = r;
      c->iters_acc = 0;
      c->k += 1;
      if (c->k == g.K) {
        c->active = 0;
      } else {
        for (int t = 0; t < 4; ++t) {
          c->fstack[0][t] = g.sched[((size_t)s * g.K + c->k - 1) * 4 + t];
          c->fstack[0][4 + t] = g.sched[((size_t)s * g.K + c->k) * 4 + t];
        }
        c->dstack[0] = g.max_bisect;
        c->sp = 1;
        adv = c->k == g.K - 1;
      }
    }
  }
  __syncwarp();
  adv = __shfl_sync(0xffffffffu, adv, 0);
  if (adv && g.Sprev) {
    const double* src = g.S + ((size_t)c->cur * g.cap + s) * 6 * g.Q;
    double* dst = g.Sprev + (size_t)s * 6 * g.Q;
    for (int t = lane; t < 6 * g.Q; t += 32) dst[t] = src[t];
  }
  if (!c->active && g.a_final)
    for (int i = lane; i < N; i += 32) g.a_final[(size_t)s * N + i] = g.a[(size_t)s * N + i];
}

__device__ __forceinline__ void rom_failed(const NewtonArgs& g, RomCtl* c, int64_t s, int lane) {
  const int N = g.N;
  for (int i = lane; i < N; i += 32) g.a[(size_t)s * N + i] = g.a0[(size_t)s * N + i];
  __syncwarp();
  if (lane == 0) {
    c->asm_fail = 0;
    c->it = 0;
    const int top = c->sp - 1;
    if (c->dstack[top] <= 0 || c->sp + 1 > kMaxStack) {
      c->active = 0;  // rom.cpp:159: rethrow -> SolveError for this instance
      c->status = PODECM_ESOLVE;
      if (g.status) g.status[s] = PODECM_ESOLVE;
      atomicAdd(g.fail, 1u);
    } else {
      double fp[4], ft[4], mid[4];
      for (int t = 0; t < 4; ++t) {
        fp[t] = c->fstack[top][t];
        ft[t] = c->fstack[top][4 + t];
        mid[t] = 0.5 * (fp[t] + ft[t]);
      }
      const int d = c->dstack[top] - 1;
      for (int t = 0; t < 4; ++t) {  // second half below, first half on top
        c->fstack[top][t] = mid[t];
        c->fstack[top][4 + t] = ft[t];
        c->fstack[top + 1][t] = fp[t];
        c->fstack[top + 1][4 + t] = mid[t];
      }
      c->dstack[top] = d;
      c->dstack[top + 1] = d;
      c->sp += 1;
    }
  }
  __syncwarp();
}

// K da = -f (dense LU, partial pivoting: first row of max |a_ik|), a += da.
// SMEM per warp: K row-major [N][N], rhs [N], the mbarrier (fits the
// N (N + 1) + 2N doubles the launches reserve).
__device__ __forceinline__ void rom_update(const NewtonArgs& g, RomCtl* c, int64_t s, int lane, double* Ks,
                                           double*, int it) {
  const int N = g.N, NN = N * N;
  double* rhs = Ks + NN;
  uint64_t* mbar = reinterpret_cast<uint64_t*>(rhs + N);
  const double* src = g.Kg + (size_t)s * NN;
  if ((NN & 1) == 0) {  // 16-byte aligned rows of the batch: one bulk copy
    warp_bulk_load(Ks, src, (unsigned)NN * 8u, mbar, lane);
  } else {
    for (int t0 = 0; t0 < NN; t0 += 32 * 8) {
      double v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int t = t0 + u * 32 + lane;
        v[u] = t < NN ? __ldcs(src + t) : 0.0;
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int t = t0 + u * 32 + lane;
        if (t < NN) Ks[t] = v[u];
      }
    }
  }
  for (int i = lane; i < N; i += 32) rhs[i] = -g.f[(size_t)s * N + i];
  __syncwarp();
  warp_lu_solve_rm(Ks, N, rhs, lane);
  for (int i = lane; i < N; i += 32) g.a[(size_t)s * N + i] += rhs[i];
  if (lane == 0) c->it = it + 1;
}

// residual norm and the reference's convergence test (tolerance frozen at
// iteration 0); returns 0 solve, 1 converged, 2 failed
__device__ __forceinline__ int rom_decide(const NewtonArgs& g, RomCtl* c, int64_t s, int lane, double ss,
                                          double* r_out) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
  const double r = sqrt(ss);
  *r_out = r;
  int out = 0;
  if (c->asm_fail != 0) {
    out = 2;
  } else {
    const int it = c->it;
    if (it == 0) {
      const double fr = g.force_ref_inst ? fmax(g.force_ref, g.force_ref_inst[s]) : g.force_ref;
      const double tol = fmax(g.eps_rel * fmax(r, fr), g.eps_abs);
      __syncwarp();
      if (lane == 0) {
        c->tol = tol;
        c->r0 = r;
      }
      out = r <= tol ? 1 : (it == g.max_iter ? 2 : 0);
    } else {
      out = r <= c->tol ? 1 : (it == g.max_iter ? 2 : 0);
    }
  }
  __syncwarp();
  return out;
}

__global__ void __launch_bounds__(32 * kNW) k_rom_newton(NewtonArgs g) {
  extern __shared__ double smn[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int N = g.N, LD = N + 1;
  double* Ks = smn + (size_t)warp * (N * LD + 2 * N);  // column-major, ld = N+1
  double* rhs = Ks + N * LD;
  const int64_t s = (int64_t)blockIdx.x * kNW + warp;
  if (s >= g.n) return;
  RomCtl* c = g.ctl + s;
  if (!c->active) return;
  const int it = c->it;
  double ss = 0.0;
  for (int i = lane; i < N; i += 32) {
    const double v = g.f[(size_t)s * N + i];
    ss = fma(v, v, ss);
  }
  double r;
  const int d = rom_decide(g, c, s, lane, ss, &r);
  if (d == 0) rom_update(g, c, s, lane, Ks, rhs, it);
  if (d == 1) rom_converged(g, c, s, lane, r, it);
  if (d == 2) rom_failed(g, c, s, lane);
  __syncwarp();
  if (lane == 0 && c->active) atomicAdd(g.nactive, 1);
}

// Lazy-tangent pipeline, step 1: f = Gm^T Pt for kCI instances per CTA as
// one DMMA GEMM (M = instances, N = modes, K = the 4Q point rows; Gm staged
// through SMEM 32 rows at a time and shared by the CTA's instances), then the
// Newton decision, one warp per instance.  Converged and failed instances
// finish here without ever needing K; the rest are appended to g.list for the
// tangent pass, the contraction and k_rom_solve.
constexpr int kCW = 32;     // warps per k_rom_check CTA
constexpr int kCI = 32;     // instances per CTA at IPW = 1 (each CTA streams all of Gm once)
constexpr int kCRows = 32;  // Gm rows per SMEM stage (kPC points)
constexpr int kCLdp = kCRows + 4;

__host__ __device__ constexpr size_t check_smem_doubles(int NP, int ipw = 1) {
  return (size_t)kCRows * (NP + 4) + (size_t)kCW * ipw * kCLdp + (size_t)kCW * ipw * NP;
}

// IPW instances per warp (kCW * IPW per CTA): every stage of Gm brought into
// shared memory feeds IPW times the DMMA work (large batches; the f sums keep
// their k order, so f is the same for any IPW).
template <int IPW = 1>
__global__ void __launch_bounds__(32 * kCW) k_rom_check(NewtonArgs g) {
  constexpr int CI = kCW * IPW;
  extern __shared__ double smk[];
  const int NP = g.NP, LDG = NP + 4, N = g.N;
  double* sG = smk;                                // [kCRows][LDG]
  double* sPt = sG + (size_t)kCRows * LDG;         // [CI][kCLdp]
  double* sF = sPt + (size_t)CI * kCLdp;           // [CI][NP]
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int gid = lane >> 2, tig = lane & 3;
  const int64_t k0 = (int64_t)blockIdx.x * CI;
  int64_t sv[IPW];
  bool av[IPW];
  bool anyl = false;
#pragma unroll
  for (int q = 0; q < IPW; ++q) {
    const int64_t k = k0 + warp + q * kCW;
    sv[q] = k < g.n ? inst_of(g.alist, k) : g.n;
    av[q] = k < g.n && g.ctl[sv[q]].active;
    anyl |= av[q];
  }
  if (!__syncthreads_or(anyl)) return;
  const int NTt = NP / 8;
  constexpr int MT = CI / 8;  // m-tiles (8 instances each)
  constexpr int JPW = (MT * 15 + kCW - 1) / kCW;  // jobs per warp at most (NT <= 15)
  // jobs: (m-tile, n-tile) = (j % MT, j / MT), j = warp + u kCW
  double acc[JPW][2];
#pragma unroll
  for (int u = 0; u < JPW; ++u) acc[u][0] = acc[u][1] = 0.0;
  const int R = g.Qpad * 4;  // padding rows of Gm and Pt are zero
  constexpr int kGPT = kCRows * 128 / (32 * kCW);  // Gm doubles per thread per stage (NP <= 128)
  double rG[kGPT], rP[IPW];
  auto load = [&](int r0) {  // next stage into registers (in flight during the DMMAs)
#pragma unroll
    for (int k = 0; k < kGPT; ++k) {
      const int t = tid + k * 32 * kCW;
      rG[k] = t < kCRows * NP ? g.G[(size_t)r0 * NP + t] : 0.0;
    }
    const int row = r0 + lane;
#pragma unroll
    for (int q = 0; q < IPW; ++q) rP[q] = av[q] ? g.Pt[((size_t)sv[q] * g.Qpad) * 4 + row] : 0.0;
  };
  load(0);
  for (int r0 = 0; r0 < R; r0 += kCRows) {
#pragma unroll
    for (int k = 0; k < kGPT; ++k) {
      const int t = tid + k * 32 * kCW;
      if (t < kCRows * NP) {
        const int rr = t / NP, i = t - rr * NP;
        sG[rr * LDG + i] = rG[k];
      }
    }
#pragma unroll
    for (int q = 0; q < IPW; ++q) sPt[(warp + q * kCW) * kCLdp + lane] = rP[q];
    __syncthreads();
    if (r0 + kCRows < R) load(r0 + kCRows);
#pragma unroll
    for (int u = 0; u < JPW; ++u) {
      const int j = warp + u * kCW;
      if (j < MT * NTt) {
        const int mt = j % MT, nt = j / MT;
#pragma unroll
        for (int ks = 0; ks < kCRows / 4; ++ks) {
          const double afr = sPt[(mt * 8 + gid) * kCLdp + ks * 4 + tig];
          const double bfr = sG[(ks * 4 + tig) * LDG + nt * 8 + gid];
          dmma(acc[u][0], acc[u][1], afr, bfr);
        }
      }
    }
    __syncthreads();
  }
#pragma unroll
  for (int u = 0; u < JPW; ++u) {
    const int j = warp + u * kCW;
    if (j < MT * NTt) {
      const int mt = j % MT, nt = j / MT;
      sF[(mt * 8 + gid) * NP + nt * 8 + 2 * tig] = acc[u][0];
      sF[(mt * 8 + gid) * NP + nt * 8 + 2 * tig + 1] = acc[u][1];
    }
  }
  __syncthreads();
#pragma unroll
  for (int q = 0; q < IPW; ++q) {
    if (!av[q]) continue;
    const int64_t s = sv[q];
    const int wi = warp + q * kCW;
    RomCtl* c = g.ctl + s;
    double ss = 0.0;
    for (int i = lane; i < N; i += 32) {
      const double v = sF[wi * NP + i];
      g.f_out[(size_t)s * N + i] = v;
      ss = fma(v, v, ss);
    }
    const int it = c->it;
    double r;
    const int d = rom_decide(g, c, s, lane, ss, &r);
    if (d == 1) rom_converged(g, c, s, lane, r, it);
    if (d == 2) rom_failed(g, c, s, lane);
    if (d == 0 && lane == 0) g.list[atomicAdd(g.count, 1)] = (int)s;
    __syncwarp();
    if (lane == 0 && c->active) atomicAdd(g.nactive, 1);
  }
}

// Lazy-tangent pipeline, step 2 (after the tangent pass and the contraction
// over g.list): a tangent failure fails the attempt (bisection), otherwise
// the Newton update K da = -f.
__global__ void __launch_bounds__(32) k_rom_solve(NewtonArgs g) {
  extern __shared__ double smn[];
  const int lane = threadIdx.x & 31;
  const int j = blockIdx.x;
  if (j >= *g.count) return;
  const int64_t s = g.list[j];
  RomCtl* c = g.ctl + s;
  double* Ks = smn;
  double* rhs = Ks + g.N * (g.N + 1);
  if (c->asm_fail != 0)
    rom_failed(g, c, s, lane);
  else
    rom_update(g, c, s, lane, Ks, rhs, c->it);
}

// The same Newton update with [K | -f] resident in registers (compile-time N):
// lane l holds the physical rows l + 32 t (t < R) and row exchanges are
// virtual — every row carries its current position, so "swap rows k and p"
// is a swap of two position tags and no data moves.  Per elimination step:
// the pivot is the active row (position >= k) of max |a_rk|, ties to the
// smaller position (a total order, so the warp's xor-tree gives the same row
// as warp_lu_solve_rm's scan); its owner publishes the pivot row through
// shared memory; every lane updates its rows below the pivot.  Each element
// sees exactly warp_lu_solve_rm's operations in the same order (same
// multipliers, same FMAs, same back substitution), so da is bit-identical —
// at ~1/4 of the warp instructions, with no shared-memory round trip on the
// critical path of the rank-1 updates.
template <int N>
__global__ void __launch_bounds__(32) k_rom_solve_reg(NewtonArgs g) {
  constexpr int R = (N + 31) / 32;  // rows per lane
  constexpr int W = N + 1;          // columns: K and the right-hand side
  constexpr int kNone = 1 << 20;    // position tag of an empty slot
  __shared__ __align__(16) double piv[W + 1];
  __shared__ double xs[N];
  const int lane = threadIdx.x;
  const int j = blockIdx.x;
  if (j >= *g.count) return;
  const int64_t s = g.list[j];
  RomCtl* c = g.ctl + s;
  if (c->asm_fail != 0) {
    rom_failed(g, c, s, lane);
    return;
  }
  const int it = c->it;
  double a[R][W];
  int pos[R];
  const double* src = g.Kg + (size_t)s * N * N;
#pragma unroll
  for (int t = 0; t < R; ++t) {
    const int row = lane + 32 * t;
    const bool ok = row < N;
    pos[t] = ok ? row : kNone;
    const double* rp = src + (size_t)(ok ? row : 0) * N;
    if constexpr ((N & 1) == 0) {
#pragma unroll
      for (int q = 0; q < N; q += 2) {
        const double2 v = ok ? __ldcs(reinterpret_cast<const double2*>(rp + q)) : make_double2(0.0, 0.0);
        a[t][q] = v.x;
        a[t][q + 1] = v.y;
      }
    } else {
#pragma unroll
      for (int q = 0; q < N; ++q) a[t][q] = ok ? __ldcs(rp + q) : 0.0;
    }
    a[t][N] = ok ? -g.f[(size_t)s * N + row] : 0.0;
  }
#pragma unroll
  for (int k = 0; k < N; ++k) {
    // pivot: max |a_rk| over active rows, ties to the smaller position
    double bv = -1.0;
    int bp = kNone;
#pragma unroll
    for (int t = 0; t < R; ++t) {
      const double v = fabs(a[t][k]);
      const bool act = pos[t] >= k && pos[t] < N;
      if (act && (v > bv || (v == bv && pos[t] < bp))) {
        bv = v;
        bp = pos[t];
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
      const int op = __shfl_xor_sync(0xffffffffu, bp, o);
      if (ov > bv || (ov == bv && op < bp)) {
        bv = ov;
        bp = op;
      }
    }
    const int p = bp < N ? bp : k;  // all-NaN column: no exchange (the result is NaN anyway)
    // the pivot row's owner publishes columns k .. N (pairs from an even
    // column; constant loop bounds so every register index is static once
    // the k loop is unrolled)
#pragma unroll
    for (int t = 0; t < R; ++t) {
      if (pos[t] == p) {
#pragma unroll
        for (int q = 0; q < W; q += 2) {
          if (q + 1 >= k) {
            if (q + 1 < W)
              *reinterpret_cast<double2*>(piv + q) = make_double2(a[t][q], a[t][q + 1]);
            else
              piv[q] = a[t][q];
          }
        }
      }
    }
    // exchange the position tags of rows k and p
#pragma unroll
    for (int t = 0; t < R; ++t) pos[t] = pos[t] == k ? p : (pos[t] == p ? k : pos[t]);
    __syncwarp();
    const double d = piv[k];
    const double rd = __drcp_rn(d);
#pragma unroll
    for (int t = 0; t < R; ++t) {
      if (pos[t] > k && pos[t] < N) {
        const double l = bv != 0.0 ? div_rcp(a[t][k], d, rd) : a[t][k];
        a[t][k] = l;
#pragma unroll
        for (int q = 0; q < W; ++q)
          if (q > k) a[t][q] = fma(-l, piv[q], a[t][q]);
      }
    }
    __syncwarp();
  }
  // back substitution with U (positions descending)
#pragma unroll
  for (int k = N - 1; k >= 0; --k) {
    double uk = 0.0, bk = 0.0;
    bool own = false;
#pragma unroll
    for (int t = 0; t < R; ++t)
      if (pos[t] == k) {
        own = true;
        uk = a[t][k];
        bk = a[t][N];
      }
    const unsigned m = __ballot_sync(0xffffffffu, own);
    const int owner = __ffs(m) - 1;
    const double xo = div_rcp(bk, uk, __drcp_rn(uk));
    const double x = __shfl_sync(0xffffffffu, xo, owner);
    if (lane == 0) xs[k] = x;
#pragma unroll
    for (int t = 0; t < R; ++t)
      if (pos[t] < k) a[t][N] = fma(-a[t][k], x, a[t][N]);
  }
  __syncwarp();
  for (int i = lane; i < N; i += 32) g.a[(size_t)s * N + i] += xs[i];
  if (lane == 0) c->it = it + 1;
}

// Newton update kernel of the lazy pipeline: the register-resident LU for the
// mode counts it is instantiated for, the shared-memory LU otherwise
// (PODECM_ROM_LU=smem forces the latter, for A/B comparisons).
// Instances per warp of the residual check (PODECM_ROM_CHECK_IPW = 1, 2 or 4
// forces it; read per call).  Every stage of Gm in shared memory feeds IPW
// times the DMMA work: 27.0 -> 22.2 (IPW 2) -> 21.5 ms (IPW 4) per C3 solve at
// 16,384 instances, fewer but fuller CTAs winning even below one per SM;
// small batches (the FE2 engines) keep one instance per warp.
int rom_check_ipw(int64_t n_run) {
  const char* e = getenv("PODECM_ROM_CHECK_IPW");
  if (e && (atoi(e) == 1 || atoi(e) == 2 || atoi(e) == 4)) return atoi(e);
  return n_run >= 4096 ? 4 : (n_run >= 2048 ? 2 : 1);
}

bool rom_lu_reg() {  // read per call (tests flip it)
  const char* e = getenv("PODECM_ROM_LU");
  return !(e && std::strcmp(e, "smem") == 0);
}


// ---- effective stiffness (rom_effective_stiffness, rom.cpp:202-241) -------
// Per instance: K (k_rom_contract at the frozen history), then for the four
// unit macro perturbations e_kl
//   rhs_kl = -sum_p c_p B_p A_p e_kl,      q_kl = K^-1 rhs_kl   (one LU, 4 RHS)
//   Abar(:, kl) = sum_p c_p A_p (e_kl + B_p^T q_kl)
// with B_p = G_p R(Fmu_p^-1) (rom.cpp:218-219, 227-228).
struct AbarArgs {
  int64_t n;
  int N, Q, Qpad, NP;
  const double* G;      // [Qpad*4][NP]
  const double* Gt;     // [N][4][Qpad]
  const double* CA;     // [n][Q][16]
  const double* Kg;     // [n][N][N]
  const double* morph;  // [n][5][Q]
  RomCtl* ctl;
  double* abar;  // [n][16] column-major Tensor4::m
  int32_t* status;
  unsigned int* fail;
};

__global__ void __launch_bounds__(32 * kNW) k_rom_abar(AbarArgs g) {
  extern __shared__ double sma[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int N = g.N, LD = N + 1, Q = g.Q;
  double* Ks = sma + (size_t)warp * (N * LD + 4 * N + 32 * 17);
  double* rhs = Ks + N * LD;  // [4][N]
  double* sX = rhs + 4 * N;   // [32][17]: X_p = R_p (c_p A_p), one point per lane
  const int64_t s = (int64_t)blockIdx.x * kNW + warp;
  if (s >= g.n) return;
  RomCtl* c = g.ctl + s;
  if (!c->active) return;
  if (c->asm_fail) {  // rom_assemble threw (material SolveError)
    if (lane == 0) {
      c->active = 0;
      c->status = PODECM_ESOLVE;
      if (g.status) g.status[s] = PODECM_ESOLVE;
      atomicAdd(g.fail, 1u);
    }
    return;
  }
  {
    const double* src = g.Kg + (size_t)s * N * N;
    for (int t = lane; t < N * N; t += 32) {
      const int i = t / N, j = t - i * N;
      Ks[j * LD + i] = src[t];
    }
  }
  const double* mo = g.morph + (size_t)s * 5 * Q;
  const double* CA = g.CA + (size_t)s * Q * 16;
  // rhs[c][i] = -sum_p sum_r G_p[i][r] X_p[r][c]; lanes over modes i = lane + 32 h
  constexpr int kRowsPerLane = 4;  // N <= 128
  double acc[kRowsPerLane][4];
#pragma unroll
  for (int h = 0; h < kRowsPerLane; ++h)
#pragma unroll
    for (int cc = 0; cc < 4; ++cc) acc[h][cc] = 0.0;
  for (int p0 = 0; p0 < Q; p0 += 32) {
    const int p = p0 + lane;
    if (p < Q) {
      double m[4];
#pragma unroll
      for (int t = 0; t < 4; ++t) m[t] = mo[(size_t)t * Q + p];
#pragma unroll
      for (int cc = 0; cc < 4; ++cc)
#pragma unroll
        for (int r = 0; r < 4; ++r) {  // (R v)[i + 2j] = m(j,0) v[i] + m(j,1) v[i+2]
          const int i = r & 1, j = r >> 1;
          sX[lane * 17 + r + 4 * cc] =
              fma(m[j + 2], CA[(size_t)p * 16 + 4 * cc + i + 2], m[j] * CA[(size_t)p * 16 + 4 * cc + i]);
        }
    }
    __syncwarp();
    const int np = min(32, Q - p0);
    for (int pl = 0; pl < np; ++pl)
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        const double* gr = g.G + ((size_t)(p0 + pl) * 4 + r) * g.NP;
        double gv[kRowsPerLane];
#pragma unroll
        for (int h = 0; h < kRowsPerLane; ++h) gv[h] = lane + 32 * h < N ? gr[lane + 32 * h] : 0.0;
#pragma unroll
        for (int cc = 0; cc < 4; ++cc) {
          const double x = sX[pl * 17 + r + 4 * cc];
#pragma unroll
          for (int h = 0; h < kRowsPerLane; ++h) acc[h][cc] = fma(gv[h], x, acc[h][cc]);
        }
      }
    __syncwarp();
  }
#pragma unroll
  for (int cc = 0; cc < 4; ++cc)
#pragma unroll
    for (int h = 0; h < kRowsPerLane; ++h)
      if (lane + 32 * h < N) rhs[cc * N + lane + 32 * h] = -acc[h][cc];
  __syncwarp();
  warp_lu_solve<4>(Ks, LD, N, rhs, lane);
  // Abar(:, cc) = sum_p CA_p (e_cc + R_p^T (G_p^T q_cc)); lanes over points
  double ab[16];
#pragma unroll
  for (int t = 0; t < 16; ++t) ab[t] = 0.0;
  for (int p = lane; p < Q; p += 32) {
    double m[4], ca[16];
#pragma unroll
    for (int t = 0; t < 4; ++t) m[t] = mo[(size_t)t * Q + p];
#pragma unroll
    for (int t = 0; t < 16; ++t) ca[t] = CA[(size_t)p * 16 + t];
    double u[4][4];
#pragma unroll
    for (int cc = 0; cc < 4; ++cc)
#pragma unroll
      for (int r = 0; r < 4; ++r) u[cc][r] = 0.0;
    for (int i = 0; i < N; ++i) {
      double gv[4];
#pragma unroll
      for (int r = 0; r < 4; ++r) gv[r] = g.Gt[((size_t)i * 4 + r) * g.Qpad + p];
#pragma unroll
      for (int cc = 0; cc < 4; ++cc) {
        const double q = rhs[cc * N + i];
#pragma unroll
        for (int r = 0; r < 4; ++r) u[cc][r] = fma(gv[r], q, u[cc][r]);
      }
    }
#pragma unroll
    for (int cc = 0; cc < 4; ++cc) {
      double df[4];  // e_cc + R^T u: (R^T u)[i + 2l] = m(0,l) u[i] + m(1,l) u[i+2]
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        const int i = t & 1, l = t >> 1;
        df[t] = fma(m[1 + 2 * l], u[cc][i + 2], m[2 * l] * u[cc][i]) + (t == cc ? 1.0 : 0.0);
      }
#pragma unroll
      for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int t = 0; t < 4; ++t) ab[r + 4 * cc] = fma(ca[r + 4 * t], df[t], ab[r + 4 * cc]);
    }
  }
#pragma unroll
  for (int t = 0; t < 16; ++t)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) ab[t] += __shfl_xor_sync(0xffffffffu, ab[t], o);
  if (lane < 16) {
    double v = ab[0];
#pragma unroll
    for (int t = 1; t < 16; ++t) v = (t == lane) ? ab[t] : v;
    g.abar[(size_t)s * 16 + lane] = v / 1.0;  // cell_volume (microfem.hpp:22)
  }
}

// Effective-stiffness stage set-up: instance s is evaluated at fbar =
// fb[s * fb_stride .. + 4] unless it already failed.
__global__ void k_rom_abar_prep(int64_t n, const double* fb, int64_t fb_stride, RomCtl* ctl,
                                const int32_t* status) {
  const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= n) return;
  RomCtl* c = ctl + s;
  const bool ok = c->status == 0 && (!status || status[s] == 0);
  c->active = ok ? 1 : 0;
  c->asm_fail = 0;
  c->sp = 1;
  for (int t = 0; t < 4; ++t) c->fstack[0][4 + t] = fb[(size_t)s * fb_stride + t];
}

// rom_sensitivity (rom.cpp:243-263) on the analytic (a, b) geometry: the
// batch of 4 n solves is ordered (s, k, lo/hi).
__global__ void k_rom_sens_prep(int64_t n, double h, const double* geom, const double* sched, int K,
                                double* geom4, double* sched4) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= 4 * n) return;
  const int64_t s = t >> 2;
  const int k = (int)((t >> 1) & 1), hi = (int)(t & 1);
  double gm[2] = {geom[2 * s], geom[2 * s + 1]};
  const double step = h * fmax(1.0, fabs(gm[k]));
  gm[k] = hi ? gm[k] + step : gm[k] - step;
  geom4[2 * t] = gm[0];
  geom4[2 * t + 1] = gm[1];
  for (int u = 0; u < 4 * K; ++u) sched4[(size_t)t * 4 * K + u] = sched[(size_t)s * 4 * K + u];
}

__global__ void k_rom_sens_combine(int64_t n, double h, const double* geom, const double* pbar4, int K,
                                   const int32_t* status4, double* grad, int32_t* status) {
  const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= n) return;
  bool ok = true;
  for (int k = 0; k < 2; ++k) {
    const double step = h * fmax(1.0, fabs(geom[2 * s + k]));
    const int64_t lo = 4 * s + 2 * k, hi = lo + 1;
    ok = ok && status4[lo] == 0 && status4[hi] == 0;
    for (int c4 = 0; c4 < 4; ++c4)
      grad[(s * 2 + k) * 4 + c4] = (pbar4[(hi * K + K - 1) * 4 + c4] - pbar4[(lo * K + K - 1) * 4 + c4]) / (2.0 * step);
  }
  if (status) status[s] = ok ? 0 : PODECM_ESOLVE;
}


// ---- batched RomMicroEngine (twoscale.cpp:53-96) ----------------------------
struct Bounds {
  double lo[3], hi[3];
};

// out_of_range_ (twoscale.cpp:66-74): (F00, F11, F01) outside the training box
__global__ void k_eng_oor(int64_t n, const double* fbar, Bounds b, int32_t* oor) {
  const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= n) return;
  const double comp[3] = {fbar[4 * s], fbar[4 * s + 3], fbar[4 * s + 2]};
  for (int k = 0; k < 3; ++k)
    if (comp[k] < b.lo[k] || comp[k] > b.hi[k]) {
      oor[s] += 1;
      break;
    }
}

// successful respond: keep the trial (states, fbar) and raise force_ref
// (twoscale.cpp:78-82); failed instances keep their previous trial
__global__ void k_eng_keep(int64_t n, int Q, const int32_t* status, const RomCtl* ctl, const double* S,
                           int64_t cap, const double* fbar, const double* init_res, double* St, double* ft,
                           double* fref, int32_t* ok) {
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (tid >= n * Q) return;
  const int64_t s = tid / Q;
  const int p = (int)(tid - s * Q);
  if (status[s] != 0) return;
  const double* src = S + ((size_t)ctl[s].cur * cap + s) * 6 * Q;
  for (int t = 0; t < 6; ++t) St[((size_t)s * 6 + t) * Q + p] = src[(size_t)t * Q + p];
  if (p == 0) {
    for (int t = 0; t < 4; ++t) ft[4 * s + t] = fbar[4 * s + t];
    fref[s] = fmax(fref[s], init_res[s]);
    ok[s] = 1;
  }
}

// commit (twoscale.cpp:91-96): only engines that ever produced a trial
__global__ void k_eng_commit(int64_t n, int Q, int N, const int32_t* ok, const double* St, const double* at,
                             const double* ft, double* Sc, double* ac, double* fc) {
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (tid >= n * Q) return;
  const int64_t s = tid / Q;
  const int p = (int)(tid - s * Q);
  if (!ok[s]) return;
  for (int t = 0; t < 6; ++t) Sc[((size_t)s * 6 + t) * Q + p] = St[((size_t)s * 6 + t) * Q + p];
  for (int i = p; i < N; i += Q) ac[(size_t)s * N + i] = at[(size_t)s * N + i];
  if (p == 0)
    for (int t = 0; t < 4; ++t) fc[4 * s + t] = ft[4 * s + t];
}

__global__ void k_eng_init(int64_t n, int Q, int N, double* Sc, double* ac, double* fc, double* fref,
                           int32_t* ok, int32_t* oor) {
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (tid >= n * Q) return;
  const int64_t s = tid / Q;
  const int p = (int)(tid - s * Q);
  const double v[6] = {1.0, 0.0, 0.0, 1.0, 1.0, 0.0};
  for (int t = 0; t < 6; ++t) Sc[((size_t)s * 6 + t) * Q + p] = v[t];
  for (int i = p; i < N; i += Q) ac[(size_t)s * N + i] = 0.0;
  if (p == 0) {
    for (int t = 0; t < 4; ++t) fc[4 * s + t] = v[t];
    fref[s] = 0.0;
    ok[s] = 0;
    oor[s] = 0;
  }
}

// register budget of the point kernel (2 or 3 CTAs/SM); PODECM_ROM_POINT_MINB
// Lazy tangent (default): the FD tangent and the contraction run only for
// the instances the residual check sends to a Newton update.  PODECM_ROM_LAZY=0
// restores the fused pipeline (tangent at every point every iteration).
bool rom_lazy() {
  static bool v = [] {
    const char* e = getenv("PODECM_ROM_LAZY");
    return !(e && atoi(e) == 0);
  }();
  return v;
}

// Material-point kernel variant: 4 / 5 = register-resident operands at that
// many CTAs per SM, 6 / 7 = slab-resident (PODECM_ROM_POINT_MINB).  Default 6
// (measured, C3 at 16,384 instances: k_rom_point_tangent 99.6 ms against
// 117.6 ms for 5; 7 is within noise of 6).
int point_minb() {
  static int v = [] {
    const char* e = getenv("PODECM_ROM_POINT_MINB");
    const int x = e ? atoi(e) : 6;
    return (x >= 4 && x <= 7) ? x : 6;
  }();
  return v;
}

template <bool ABAR, int MODE>
void launch_point(int grid, cudaStream_t s, const PointArgs& a, const MatTable& mats) {
  switch (point_minb()) {
    case 4: k_rom_point<4, ABAR, MODE><<<grid, 128, 0, s>>>(a, mats); break;
    case 6: k_rom_point<6, ABAR, MODE, true><<<grid, 128, 0, s>>>(a, mats); break;
    case 7: k_rom_point<7, ABAR, MODE, true><<<grid, 128, 0, s>>>(a, mats); break;
    default: k_rom_point<5, ABAR, MODE><<<grid, 128, 0, s>>>(a, mats); break;
  }
}

template <class T>
int dalloc(podecm_ctx* ctx, T** p, size_t count) {
  PODECM_CUDA_TRY(ctx, cudaMalloc(p, std::max<size_t>(1, count) * sizeof(T)));
  return PODECM_OK;
}

int ensure_cap(podecm_rom* r, int64_t n) {
  if (r->cap >= n) return PODECM_OK;
  free_work(r);
  podecm_ctx* ctx = r->ctx;
  const size_t Q = r->Q, N = r->N;
  int rc = PODECM_OK;
  if (!rc) rc = dalloc(ctx, &r->d_morph, (size_t)n * 5 * Q);
  if (!rc) rc = dalloc(ctx, &r->d_S, (size_t)2 * n * 6 * Q);
  if (!rc) rc = dalloc(ctx, &r->d_At, (size_t)n * r->Qpad * 20);
  if (!rc) rc = dalloc(ctx, &r->d_P, (size_t)n * Q * 4);
  if (!rc) rc = dalloc(ctx, &r->d_K, (size_t)n * N * N);
  if (!rc) rc = dalloc(ctx, &r->d_f, (size_t)n * N);
  if (!rc) rc = dalloc(ctx, &r->d_a, (size_t)n * N);
  if (!rc) rc = dalloc(ctx, &r->d_a0, (size_t)n * N);
  if (!rc) rc = dalloc(ctx, &r->d_Fb, (size_t)n * 4 * Q);
  if (!rc) rc = dalloc(ctx, &r->d_Pt, (size_t)n * r->Qpad * 4);
  if (!rc) rc = dalloc(ctx, &r->d_ctl, (size_t)n);
  if (!rc) rc = dalloc(ctx, &r->d_list, (size_t)n);
  if (!rc) rc = dalloc(ctx, &r->d_alist, (size_t)n + 1);  // [n]: the count
  if (rc) {
    free_work(r);
    return rc;
  }
  // padding rows of At and Pt (p >= Q) stay zero forever
  PODECM_CUDA_TRY(ctx, cudaMemset(r->d_At, 0, (size_t)n * r->Qpad * 20 * sizeof(double)));
  PODECM_CUDA_TRY(ctx, cudaMemset(r->d_Pt, 0, (size_t)n * r->Qpad * 4 * sizeof(double)));
  r->cap = n;
  return PODECM_OK;
}


int ensure_abar(podecm_rom* r, int64_t n, bool sprev) {
  if (r->abar_cap >= n && (!sprev || r->d_Sprev)) return PODECM_OK;
  cudaFree(r->d_CA);
  cudaFree(r->d_Sprev);
  r->d_CA = r->d_Sprev = nullptr;
  r->abar_cap = 0;
  int rc = dalloc(r->ctx, &r->d_CA, (size_t)n * r->Q * 16);
  if (!rc && sprev) rc = dalloc(r->ctx, &r->d_Sprev, (size_t)n * 6 * r->Q);
  if (!rc) r->abar_cap = n;
  return rc;
}

template <bool LIST, int... I>
void set_contract_attrs(std::integer_sequence<int, I...>) {
  (..., (I > 0 ? (void)cudaFuncSetAttribute(
                     k_rom_contract<(I > 0 ? I : 1), contract_ipc<(I > 0 ? I : 1)>(), LIST>,
                     cudaFuncAttributeMaxDynamicSharedMemorySize, (int)contract_smem_bytes<(I > 0 ? I : 1)>())
               : (void)0));
  (..., (I > 0 && I <= 7 ? (void)cudaFuncSetAttribute(k_rom_contract<(I > 0 && I <= 7 ? I : 1), 1, LIST>,
                                                     cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                     (int)contract_smem_bytes<(I > 0 && I <= 7 ? I : 1), 1>())
                         : (void)0));
}

// Opt-in dynamic SMEM limits are per device: set them once for every device
// a context of this process launches on.
void set_attrs() {
  static std::mutex mu;
  static uint64_t done = 0;  // bit d: device d configured
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lock(mu);
  if (dev < 64 && (done >> dev) & 1u) return;
  cudaFuncSetAttribute(k_rom_F, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaFuncSetAttribute(k_rom_F_mma, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  set_contract_attrs<false>(std::make_integer_sequence<int, kMaxNT + 1>{});
  set_contract_attrs<true>(std::make_integer_sequence<int, kMaxNT + 1>{});
  cudaFuncSetAttribute(k_rom_contract_rp<6, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)contract_rp_smem_bytes<6, 1>());
  cudaFuncSetAttribute(k_rom_contract_rp<6, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)contract_rp_smem_bytes<6, 2>());
  cudaFuncSetAttribute(k_rom_contract_rp3<6, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)contract_rp_smem_bytes<6, 2>());
  cudaFuncSetAttribute(k_rom_solve, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaFuncSetAttribute(k_rom_check<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaFuncSetAttribute(k_rom_check<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaFuncSetAttribute(k_rom_check<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaFuncSetAttribute(k_rom_newton, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaFuncSetAttribute(k_rom_abar, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  if (dev < 64) done |= uint64_t(1) << dev;
}

PointArgs point_args(podecm_rom* r, int64_t n) {
  PointArgs pa;
  pa.n = n;
  pa.N = r->N;
  pa.Q = r->Q;
  pa.Qpad = r->Qpad;
  pa.cap = r->cap;
  pa.Gt = r->d_Gt;
  pa.a = r->d_a;
  pa.morph = r->d_morph;
  pa.w = r->d_w;
  pa.reg = r->d_reg;
  pa.S = r->d_S;
  pa.At = r->d_At;
  pa.P = r->d_P;
  pa.Fb = r->d_Fb;
  pa.Pt = r->d_Pt;
  pa.ctl = r->d_ctl;
  pa.S0 = nullptr;
  pa.CA = nullptr;
  pa.list = nullptr;
  pa.count = nullptr;
  return pa;
}

ContractArgs contract_args(podecm_rom* r, int64_t n) {
  ContractArgs ca;
  ca.n = n;
  ca.N = r->N;
  ca.Q = r->Q;
  ca.Qpad = r->Qpad;
  ca.NT = r->NT;
  ca.NP = r->NP;
  ca.G = r->d_G;
  ca.At = r->d_At;
  ca.K = r->d_K;
  ca.f = r->d_f;
  ca.ctl = r->d_ctl;
  ca.list = nullptr;
  ca.count = nullptr;
  return ca;
}

// F at the ECM points: the DMMA form by default; PODECM_ROM_F=fma selects the
// DFMA kernel (k_rom_F) for A/B comparisons.
bool rom_F_mma() {  // read per call (tests flip it)
  const char* e = getenv("PODECM_ROM_F");
  return !(e && std::strcmp(e, "fma") == 0);
}

void launch_F(podecm_ctx* ctx, cudaStream_t s, podecm_rom* r, const PointArgs& pa) {
  KTimer kt(ctx, s, "k_rom_F");
  if (rom_F_mma()) {
    const dim3 g((r->Q + kFMP - 1) / kFMP, (unsigned)((pa.n + kFMI - 1) / kFMI));
    k_rom_F_mma<<<g, 256, fmma_smem_doubles(r->N) * sizeof(double), s>>>(pa, r->d_G, r->NP);
    return;
  }
  const dim3 gpt((r->Q + kPtsTile - 1) / kPtsTile, (unsigned)((pa.n + kFInst - 1) / kFInst));
  const size_t smem_pt = ((size_t)r->N * 4 * kPtsTile + (size_t)kFInst * r->N) * sizeof(double);
  k_rom_F<<<gpt, 256, smem_pt, s>>>(pa);
}

// Small batches (e.g. the FE2 engines: 800 instances = 1.35 waves of
// two-instance CTAs) run one instance per CTA for twice the CTAs.
constexpr int64_t kSmallBatch = 4096;

template <int NT, bool LIST>
void launch_contract_nt(cudaStream_t s, const ContractArgs& ca) {
  constexpr int ipc = contract_ipc<NT>();
  if (ipc > 1 && ca.n < kSmallBatch) {
    k_rom_contract<NT, 1, LIST><<<(int)ca.n, 32 * NT, contract_smem_bytes<NT, 1>(), s>>>(ca);
    return;
  }
  const int gct = (int)((ca.n + ipc - 1) / ipc);
  k_rom_contract<NT, ipc, LIST><<<gct, 32 * NT * ipc, contract_smem_bytes<NT>(), s>>>(ca);
}

template <int... I>
void launch_contract_sw(int nt, cudaStream_t s, const ContractArgs& ca, std::integer_sequence<int, I...>) {
  if (ca.list)
    (..., (nt == I + 1 ? launch_contract_nt<I + 1, true>(s, ca) : (void)0));
  else
    (..., (nt == I + 1 ? launch_contract_nt<I + 1, false>(s, ca) : (void)0));
}

// Remainder-packed form: lazy pipeline (list), N = 49 or 50 (PODECM_ROM_CONTRACT=std:
// the 56-wide kernel, =rp23: the 12-warp 2 x 3-block form for large batches; read per
// call, tests flip it).
bool contract_rp_on() {
  const char* e = getenv("PODECM_ROM_CONTRACT");
  return !(e && std::strcmp(e, "std") == 0);
}

void launch_contract(podecm_ctx* ctx, cudaStream_t s, podecm_rom* r, const ContractArgs& ca) {
  KTimer kt(ctx, s, "k_rom_contract");
  if (ca.list && r->NT == 7 && r->N > 48 && r->N <= 50 && contract_rp_on()) {
    const char* e = getenv("PODECM_ROM_CONTRACT");
    if (ca.n < kSmallBatch)  // one instance per CTA: twice the CTAs, the same bits
      k_rom_contract_rp<6, 1><<<(int)ca.n, 32 * 8, contract_rp_smem_bytes<6, 1>(), s>>>(ca);
    else if (e && std::strcmp(e, "rp23") == 0)  // 12 warps with 2 x 3 tile blocks (A/B)
      k_rom_contract_rp<6, 2><<<(int)((ca.n + 1) / 2), 32 * 12, contract_rp_smem_bytes<6, 2>(), s>>>(ca);
    else  // 8 warps with 3 x 3 tile blocks
      k_rom_contract_rp3<6, 2><<<(int)((ca.n + 1) / 2), 256, contract_rp_smem_bytes<6, 2>(), s>>>(ca);
    return;
  }
  launch_contract_sw(r->NT, s, ca, std::make_integer_sequence<int, kMaxNT>{});
}

// Effective-stiffness stage over n instances whose morph slice (d_morph),
// reduced coordinates (d_a) and control blocks are staged: history S0
// [n][6][Q], macro gradient fb[s * fb_stride ..].  Five launches.
int abar_stage(podecm_ctx* ctx, cudaStream_t s, podecm_rom* r, int64_t n, const double* S0,
               const double* fb, int64_t fb_stride, double* abar, int32_t* status) {
  k_rom_abar_prep<<<grid_for(n, 128), 128, 0, s>>>(n, fb, fb_stride, r->d_ctl, status);
  PointArgs pa = point_args(r, n);
  pa.S0 = S0;
  pa.CA = r->d_CA;
  launch_F(ctx, s, r, pa);
  {
    KTimer kt(ctx, s, "k_rom_point_abar");
    const int gp = grid_for(n * r->Q, 128);
    launch_point<true, 0>(gp, s, pa, r->rve->mats);
  }
  launch_contract(ctx, s, r, contract_args(r, n));
  AbarArgs aa;
  aa.n = n;
  aa.N = r->N;
  aa.Q = r->Q;
  aa.Qpad = r->Qpad;
  aa.NP = r->NP;
  aa.G = r->d_G;
  aa.Gt = r->d_Gt;
  aa.CA = r->d_CA;
  aa.Kg = r->d_K;
  aa.morph = r->d_morph;
  aa.ctl = r->d_ctl;
  aa.abar = abar;
  aa.status = status;
  aa.fail = ctx->d_fail;
  {
    KTimer kt(ctx, s, "k_rom_abar");
    const size_t smem = (size_t)kNW * ((size_t)r->N * (r->N + 1) + 4 * r->N + 32 * 17) * sizeof(double);
    k_rom_abar<<<(int)((n + kNW - 1) / kNW), 32 * kNW, smem, s>>>(aa);
  }
  PODECM_LAUNCHED(ctx, 5);
  return PODECM_OK;
}

int check_solve_args(podecm_ctx* ctx, podecm_rom* r, int64_t n_inst, int K, const podecm_newton* opts) {
  if (n_inst < 0 || K < 0) return set_err(ctx, PODECM_ECONFIG, "negative batch or schedule size");
  if (opts->max_bisect < 0 || opts->max_bisect + 1 > kMaxStack)
    return set_err(ctx, PODECM_ECONFIG, "max_bisect must lie in [0, 7]");
  if (opts->max_iter < 0) return set_err(ctx, PODECM_ECONFIG, "max_iter must be >= 0");
  if (r->NT > kMaxNT) return set_err(ctx, PODECM_ECONFIG, "rom: N > 119 exceeds the contraction tile");
  return PODECM_OK;
}

// Start of a solve other than rom_solve's virgin one (RomMicroEngine::respond):
// committed history, reduced coordinates, previous macro gradient and
// force_ref per instance; initial_residual out.
struct RomStart {
  const double* S = nullptr;     // [n][6][Q]
  const double* a = nullptr;     // [n][N]
  const double* fprev = nullptr; // [n][4]
  const double* fref = nullptr;  // [n]
  double* init_res = nullptr;    // [n][K]
  const double* morph_q = nullptr;  // [n][5][Q] morph slice (replaces geom)
  double* a_hist = nullptr;         // [n][K][N] reduced coordinates per increment
};

int rom_solve_impl(podecm_ctx* ctx, void* stream, podecm_rom* r, int64_t n_inst, const double* geom,
                   const double* sched, int K, const podecm_newton* opts, double* pbar, int32_t* iters,
                   double* resid, double* a_final, int32_t* status, double* abar,
                   const RomStart& start = RomStart()) {
  if (int rc = check_solve_args(ctx, r, n_inst, K, opts)) return rc;
  if (n_inst == 0 || K == 0) return PODECM_OK;
  if ((!geom && !start.morph_q) || !sched || !pbar)
    return set_err(ctx, PODECM_ECONFIG, "geom (or a morph slice), sched, pbar required");
  if (int rc = ensure_cap(r, n_inst)) return rc;
  if (abar)
    if (int rc = ensure_abar(r, n_inst, true)) return rc;
  auto s = static_cast<cudaStream_t>(stream);
  podecm_rve* rv = r->rve;
  const int Q = r->Q, N = r->N;
  set_attrs();
  k_rom_init_inst<<<grid_for(n_inst, 128), 128, 0, s>>>(n_inst, N, opts->max_bisect, sched, K,
                                                        r->d_a, r->d_a0, r->d_ctl, status, start.fprev,
                                                        start.a);
  k_rom_init_points<<<grid_for(n_inst * Q, 128), 128, 0, s>>>(
      n_inst, Q, rv->n_qp, rv->r0, r->d_ids, rv->d_nodes, rv->d_elems, rv->d_grad, geom,
      r->d_morph, r->d_S, r->cap, r->d_ctl, abar ? r->d_Sprev : nullptr, start.S, start.morph_q);
  k_rom_fix_status<<<grid_for(n_inst, 128), 128, 0, s>>>(n_inst, r->d_ctl, status, ctx->d_fail);
  PODECM_LAUNCHED(ctx, 3);

  const PointArgs pa = point_args(r, n_inst);
  const ContractArgs ca = contract_args(r, n_inst);

  NewtonArgs na;
  na.n = n_inst;
  na.N = N;
  na.Q = Q;
  na.K = K;
  na.max_iter = opts->max_iter;
  na.max_bisect = opts->max_bisect;
  na.eps_rel = opts->eps_rel;
  na.eps_abs = opts->eps_abs;
  na.force_ref = opts->force_ref;
  na.Kg = r->d_K;
  na.f = r->d_f;
  na.P = r->d_P;
  na.morph = r->d_morph;
  na.w = r->d_w;
  na.sched = sched;
  na.a = r->d_a;
  na.a0 = r->d_a0;
  na.ctl = r->d_ctl;
  na.pbar = pbar;
  na.iters = iters;
  na.resid = resid;
  na.a_final = a_final;
  na.status = status;
  na.nactive = r->d_nactive;
  na.fail = ctx->d_fail;
  na.S = r->d_S;
  na.cap = r->cap;
  na.Sprev = abar ? r->d_Sprev : nullptr;
  na.force_ref_inst = start.fref;
  na.init_res = start.init_res;
  na.a_hist = start.a_hist;
  na.G = r->d_G;
  na.Pt = r->d_Pt;
  na.Qpad = r->Qpad;
  na.NP = r->NP;
  na.f_out = r->d_f;
  na.list = r->d_list;
  na.count = r->d_nactive + 1;
  const bool lazy = rom_lazy();
  PointArgs pl = pa;
  pl.list = r->d_list;
  pl.count = r->d_nactive + 1;
  ContractArgs cl = ca;
  cl.list = r->d_list;
  cl.count = r->d_nactive + 1;
  const size_t smem_ck = check_smem_doubles(r->NP) * sizeof(double);
  const size_t smem_ck2 = check_smem_doubles(r->NP, 2) * sizeof(double);
  const size_t smem_ck4 = check_smem_doubles(r->NP, 4) * sizeof(double);
  const size_t smem_nt = (size_t)kNW * ((size_t)N * (N + 1) + 2 * N) * sizeof(double);
  const int gnt = (int)((n_inst + kNW - 1) / kNW);

  const int64_t max_global = (int64_t)K * (opts->max_iter + 1) * (2ll << opts->max_bisect) + 8;
  // lazy pipeline: grids cover only the instances still active at the last
  // host sync (k_rom_compact; a superset of the active ones until the next)
  // (large batches only: a small batch is one short wave either way, and the
  // extra host sync per call costs more than the trimmed grids save)
  int64_t n_run = n_inst;
  const bool use_alist = n_inst >= 8192;
  auto compact = [&]() -> int {
    if (use_alist) {
      k_rom_compact<<<1, 1024, 0, s>>>(n_inst, r->d_ctl, r->d_alist, n_inst);
      PODECM_LAUNCHED(ctx, 1);
      PODECM_CUDA_TRY(ctx, cudaMemcpyAsync(r->h_nactive, r->d_alist + n_inst, sizeof(int),
                                           cudaMemcpyDeviceToHost, s));
    } else {  // instances k_rom_check left active in the last iteration
      PODECM_CUDA_TRY(ctx, cudaMemcpyAsync(r->h_nactive, r->d_nactive, sizeof(int), cudaMemcpyDeviceToHost, s));
    }
    PODECM_CUDA_TRY(ctx, cudaStreamSynchronize(s));
    if (use_alist || *r->h_nactive == 0) n_run = *r->h_nactive;
    return PODECM_OK;
  };
  if (lazy && use_alist)
    if (int rc = compact()) return rc;
  for (int64_t it = 0; it < max_global; ++it) {
    if (lazy) {
      if (n_run == 0) break;
      PointArgs pr = pa;
      pr.alist = use_alist ? r->d_alist : nullptr;
      pr.n = n_run;
      NewtonArgs nr_ = na;
      nr_.alist = pr.alist;
      nr_.n = n_run;
      ContractArgs cr = cl;
      cr.n = n_run;
      launch_F(ctx, s, r, pr);
      const int gp = grid_for(n_run * Q, 128);
      {
        KTimer kt(ctx, s, "k_rom_point_p");
        launch_point<false, 1>(gp, s, pr, rv->mats);
      }
      PODECM_CUDA_TRY(ctx, cudaMemsetAsync(r->d_nactive, 0, 2 * sizeof(int), s));
      {
        KTimer kt(ctx, s, "k_rom_check");
        // instances per warp: as many as keep >= 2 CTAs per SM busy
        const int cipw = rom_check_ipw(n_run);
        if (cipw == 4)
          k_rom_check<4><<<(int)((n_run + 4 * kCW - 1) / (4 * kCW)), 32 * kCW, smem_ck4, s>>>(nr_);
        else if (cipw == 2)
          k_rom_check<2><<<(int)((n_run + 2 * kCW - 1) / (2 * kCW)), 32 * kCW, smem_ck2, s>>>(nr_);
        else
          k_rom_check<1><<<(int)((n_run + kCW - 1) / kCW), 32 * kCW, smem_ck, s>>>(nr_);
      }
      {
        KTimer kt(ctx, s, "k_rom_point_tangent");
        launch_point<false, 2>(gp, s, pl, rv->mats);
      }
      launch_contract(ctx, s, r, cr);
      {
        KTimer kt(ctx, s, "k_rom_solve");
        if (N == 50 && rom_lu_reg())
          k_rom_solve_reg<50><<<(int)n_run, 32, 0, s>>>(na);
        else
          k_rom_solve<<<(int)n_run, 32, (size_t)((size_t)N * (N + 1) + 2 * N) * sizeof(double), s>>>(na);
      }
      PODECM_LAUNCHED(ctx, 6);
      r->last_global_iters = it + 1;
      if ((it & 3) == 3)
        if (int rc = compact()) return rc;
      continue;
    }
    launch_F(ctx, s, r, pa);
    {
    {
      KTimer kt(ctx, s, "k_rom_point");
      const int gp = grid_for(n_inst * Q, 128);
      launch_point<false, 0>(gp, s, pa, rv->mats);
    }
    launch_contract(ctx, s, r, ca);
    PODECM_CUDA_TRY(ctx, cudaMemsetAsync(r->d_nactive, 0, sizeof(int), s));
    {
      KTimer kt(ctx, s, "k_rom_newton");
      k_rom_newton<<<gnt, 32 * kNW, smem_nt, s>>>(na);
    }
    PODECM_LAUNCHED(ctx, 4);
    }
    if ((it & 3) == 3) {
      PODECM_CUDA_TRY(ctx, cudaMemcpyAsync(r->h_nactive, r->d_nactive, sizeof(int),
                                           cudaMemcpyDeviceToHost, s));
      PODECM_CUDA_TRY(ctx, cudaStreamSynchronize(s));
      if (*r->h_nactive == 0) {
        r->last_global_iters = it + 1;
        break;
      }
    }
    r->last_global_iters = it + 1;
  }
  // failed instances -> context flag (podecm_check reports SolveError)
  if (abar)  // run_online's effective_stiffness request (pipeline.cpp:481-483)
    return abar_stage(ctx, s, r, n_inst, r->d_Sprev, sched + (size_t)(K - 1) * 4, (int64_t)K * 4, abar,
                      status);
  return PODECM_OK;
}

}  // namespace


extern "C" {

int podecm_rom_create(podecm_ctx* ctx, podecm_rve* rve, int N, int Q, const int32_t* ids,
                      const double* weights, const double* mode_grads, podecm_rom** out) {
  if (!ctx || !rve || !out) return PODECM_ECONFIG;
  *out = nullptr;
  if (N < 1 || N > 8 * kMaxNT - 1) return set_err(ctx, PODECM_ECONFIG, "rom: need 1 <= N <= 119 modes");
  if (Q < 1) return set_err(ctx, PODECM_ECONFIG, "rom: empty cubature rule");
  if (!ids || !weights || !mode_grads) return set_err(ctx, PODECM_ECONFIG, "rom: null model arrays");
  for (int p = 0; p < Q; ++p) {
    if (ids[p] < 0 || ids[p] >= rve->n_qp)
      return set_err(ctx, PODECM_ECONFIG, "rom: ECM id out of range");
    if (p > 0 && ids[p] <= ids[p - 1])
      return set_err(ctx, PODECM_ECONFIG, "rom: ECM ids must be strictly ascending");
  }
  auto* r = new podecm_rom;
  r->rve = rve;
  r->ctx = ctx;
  r->N = N;
  r->Q = Q;
  r->Qpad = (Q + kPC - 1) / kPC * kPC;
  r->NT = (N + 1 + 7) / 8;  // + 1: f rides in column N
  r->NP = r->NT * 8;
  std::vector<double> G((size_t)r->Qpad * 4 * r->NP, 0.0), Gt((size_t)N * 4 * r->Qpad, 0.0);
  std::vector<int32_t> reg(Q);
  for (int p = 0; p < Q; ++p) {
    reg[p] = rve->regions[ids[p] >> 2];
    for (int i = 0; i < N; ++i)
      for (int c = 0; c < 4; ++c) {
        const double v = mode_grads[((size_t)p * N + i) * 4 + c];
        G[((size_t)p * 4 + c) * r->NP + i] = v;
        Gt[((size_t)i * 4 + c) * r->Qpad + p] = v;
      }
  }
  std::vector<int32_t> hid(ids, ids + Q);
  std::vector<double> hw(weights, weights + Q);
  int rc = PODECM_OK;
  auto up = [&](auto** d, const auto& h) {
    if (rc) return;
    using T = std::remove_reference_t<decltype(h[0])>;
    if (cudaMalloc(d, h.size() * sizeof(T)) != cudaSuccess ||
        cudaMemcpy(*d, h.data(), h.size() * sizeof(T), cudaMemcpyHostToDevice) != cudaSuccess)
      rc = set_err(ctx, PODECM_ECUDA, "rom: device upload failed");
  };
  up(&r->d_ids, hid);
  up(&r->d_reg, reg);
  up(&r->d_w, hw);
  up(&r->d_G, G);
  up(&r->d_Gt, Gt);
  if (!rc && cudaMalloc(&r->d_nactive, 2 * sizeof(int)) != cudaSuccess) rc = PODECM_ECUDA;
  if (!rc && cudaMallocHost(&r->h_nactive, sizeof(int)) != cudaSuccess) rc = PODECM_ECUDA;
  if (rc) {
    podecm_rom_destroy(r);
    return rc;
  }
  *out = r;
  return PODECM_OK;
}

int64_t podecm_rom_global_iterations(const podecm_rom* r) { return r ? r->last_global_iters : 0; }

void podecm_rom_destroy(podecm_rom* r) {
  if (!r) return;
  free_work(r);
  cudaFree(r->d_ids);
  cudaFree(r->d_reg);
  cudaFree(r->d_w);
  cudaFree(r->d_G);
  cudaFree(r->d_Gt);
  cudaFree(r->d_nactive);
  if (r->h_nactive) cudaFreeHost(r->h_nactive);
  delete r;
}

int podecm_rom_solve_batch(podecm_ctx* ctx, void* stream, podecm_rom* r, int64_t n_inst,
                           const double* geom, const double* sched, int K,
                           const podecm_newton* opts, double* pbar, int32_t* iters, double* resid,
                           double* a_final, int32_t* status) {
  if (!ctx || !r || !opts) return PODECM_ECONFIG;
  return rom_solve_impl(ctx, stream, r, n_inst, geom, sched, K, opts, pbar, iters, resid, a_final, status,
                        nullptr);
}

int podecm_rom_solve_batch_ex(podecm_ctx* ctx, void* stream, podecm_rom* r, int64_t n_inst,
                              const double* geom, const double* sched, int K,
                              const podecm_newton* opts, double* pbar, int32_t* iters,
                              double* resid, double* a_final, int32_t* status, double* abar) {
  if (!ctx || !r || !opts) return PODECM_ECONFIG;
  return rom_solve_impl(ctx, stream, r, n_inst, geom, sched, K, opts, pbar, iters, resid, a_final, status,
                        abar);
}

int podecm_rom_solve_batch_morph(podecm_ctx* ctx, void* stream, podecm_rom* r, int64_t n_inst,
                                 const double* morph_q, const double* sched, int K,
                                 const podecm_newton* opts, double* pbar, int32_t* iters,
                                 double* resid, double* a_final, int32_t* status, double* abar,
                                 double* a_hist) {
  if (!ctx || !r || !opts) return PODECM_ECONFIG;
  if (!morph_q && n_inst > 0) return set_err(ctx, PODECM_ECONFIG, "morph slice required");
  RomStart st;
  st.morph_q = morph_q;
  st.a_hist = a_hist;
  return rom_solve_impl(ctx, stream, r, n_inst, nullptr, sched, K, opts, pbar, iters, resid, a_final, status,
                        abar, st);
}

int podecm_rom_effective_stiffness_batch(podecm_ctx* ctx, void* stream, podecm_rom* r, int64_t n_inst,
                                         const double* geom, const double* st0, const double* fbar,
                                         const double* a, double* abar, int32_t* status) {
  if (!ctx || !r) return PODECM_ECONFIG;
  if (n_inst < 0) return set_err(ctx, PODECM_ECONFIG, "negative batch size");
  if (n_inst == 0) return PODECM_OK;
  if (!geom || !st0 || !fbar || !a || !abar)
    return set_err(ctx, PODECM_ECONFIG, "geom, st0, fbar, a, abar required");
  if (r->NT > kMaxNT) return set_err(ctx, PODECM_ECONFIG, "rom: N > 119 exceeds the contraction tile");
  if (int rc = ensure_cap(r, n_inst)) return rc;
  if (int rc = ensure_abar(r, n_inst, false)) return rc;
  auto s = static_cast<cudaStream_t>(stream);
  podecm_rve* rv = r->rve;
  set_attrs();
  k_rom_init_inst<<<grid_for(n_inst, 128), 128, 0, s>>>(n_inst, r->N, 0, fbar, 1, r->d_a, r->d_a0,
                                                        r->d_ctl, status, nullptr, nullptr);
  k_rom_init_points<<<grid_for(n_inst * r->Q, 128), 128, 0, s>>>(
      n_inst, r->Q, rv->n_qp, rv->r0, r->d_ids, rv->d_nodes, rv->d_elems, rv->d_grad, geom,
      r->d_morph, r->d_S, r->cap, r->d_ctl, nullptr, nullptr);
  k_rom_fix_status<<<grid_for(n_inst, 128), 128, 0, s>>>(n_inst, r->d_ctl, status, ctx->d_fail);
  PODECM_LAUNCHED(ctx, 3);
  PODECM_CUDA_TRY(ctx, cudaMemcpyAsync(r->d_a, a, (size_t)n_inst * r->N * sizeof(double),
                                       cudaMemcpyDeviceToDevice, s));
  return abar_stage(ctx, s, r, n_inst, st0, fbar, 4, abar, status);
}

int podecm_rom_sensitivity_batch(podecm_ctx* ctx, void* stream, podecm_rom* r, int64_t n_inst,
                                 const double* geom, const double* sched, int K,
                                 const podecm_newton* opts, double h, double* grad, int32_t* status) {
  if (!ctx || !r || !opts) return PODECM_ECONFIG;
  if (int rc = check_solve_args(ctx, r, n_inst, K, opts)) return rc;
  if (n_inst == 0) return PODECM_OK;
  if (K == 0) return set_err(ctx, PODECM_ECONFIG, "rom_sensitivity needs a non-empty schedule");
  if (!geom || !sched || !grad) return set_err(ctx, PODECM_ECONFIG, "geom, sched, grad required");
  if (!(h > 0.0)) return set_err(ctx, PODECM_ECONFIG, "rom_sensitivity: h must be > 0");
  auto s = static_cast<cudaStream_t>(stream);
  const int64_t n4 = 4 * n_inst;
  double *geom4 = nullptr, *sched4 = nullptr, *pbar4 = nullptr;
  int32_t* status4 = nullptr;
  cudaError_t ce = cudaMallocAsync(&geom4, (size_t)n4 * 2 * sizeof(double), s);
  if (ce == cudaSuccess) ce = cudaMallocAsync(&sched4, (size_t)n4 * K * 4 * sizeof(double), s);
  if (ce == cudaSuccess) ce = cudaMallocAsync(&pbar4, (size_t)n4 * K * 4 * sizeof(double), s);
  if (ce == cudaSuccess) ce = cudaMallocAsync(&status4, (size_t)n4 * sizeof(int32_t), s);
  int rc = ce == cudaSuccess ? PODECM_OK : cuda_err(ctx, ce, "rom_sensitivity: allocation");
  if (!rc) {
    k_rom_sens_prep<<<grid_for(n4, 128), 128, 0, s>>>(n_inst, h, geom, sched, K, geom4, sched4);
    ctx->launches += 1;
    rc = rom_solve_impl(ctx, stream, r, n4, geom4, sched4, K, opts, pbar4, nullptr, nullptr, nullptr, status4,
                        nullptr);
  }
  if (!rc) {
    k_rom_sens_combine<<<grid_for(n_inst, 128), 128, 0, s>>>(n_inst, h, geom, pbar4, K, status4, grad,
                                                             status);
    rc = cudaGetLastError() == cudaSuccess ? PODECM_OK : set_err(ctx, PODECM_ECUDA, "launch");
    if (!rc) PODECM_LAUNCHED(ctx, 1);
  }
  for (void* ptr : {(void*)geom4, (void*)sched4, (void*)pbar4, (void*)status4})
    if (ptr) cudaFreeAsync(ptr, s);
  return rc;
}


int podecm_rom_engines_create(podecm_ctx* ctx, podecm_rom* rom, int64_t n, const double* geom,
                              const double* stretch_bounds, podecm_rom_engines** out) {
  if (!ctx || !rom || !out) return PODECM_ECONFIG;
  *out = nullptr;
  if (n < 1) return set_err(ctx, PODECM_ECONFIG, "engines: need n >= 1");
  if (!geom) return set_err(ctx, PODECM_ECONFIG, "engines: geom required");
  auto* e = new podecm_rom_engines;
  e->rom = rom;
  e->n = n;
  if (stretch_bounds) {
    e->has_bounds = true;
    for (int t = 0; t < 6; ++t) e->bounds[t] = stretch_bounds[t];
  }
  const size_t Q = rom->Q, N = rom->N;
  int rc = PODECM_OK;
  if (!rc) rc = dalloc(ctx, &e->d_geom, (size_t)n * 2);
  if (!rc) rc = dalloc(ctx, &e->d_Sc, (size_t)n * 6 * Q);
  if (!rc) rc = dalloc(ctx, &e->d_St, (size_t)n * 6 * Q);
  if (!rc) rc = dalloc(ctx, &e->d_ac, (size_t)n * N);
  if (!rc) rc = dalloc(ctx, &e->d_at, (size_t)n * N);
  if (!rc) rc = dalloc(ctx, &e->d_fc, (size_t)n * 4);
  if (!rc) rc = dalloc(ctx, &e->d_ft, (size_t)n * 4);
  if (!rc) rc = dalloc(ctx, &e->d_fref, (size_t)n);
  if (!rc) rc = dalloc(ctx, &e->d_ires, (size_t)n);
  if (!rc) rc = dalloc(ctx, &e->d_ok, (size_t)n);
  if (!rc) rc = dalloc(ctx, &e->d_oor, (size_t)n);
  if (!rc) rc = dalloc(ctx, &e->d_status, (size_t)n);
  if (!rc && cudaMemcpy(e->d_geom, geom, (size_t)n * 2 * sizeof(double), cudaMemcpyDefault) != cudaSuccess)
    rc = set_err(ctx, PODECM_ECUDA, "engines: geom copy failed");
  if (!rc) {
    k_eng_init<<<grid_for(n * (int64_t)Q, 128), 128>>>(n, (int)Q, (int)N, e->d_Sc, e->d_ac, e->d_fc, e->d_fref,
                                                       e->d_ok, e->d_oor);
    if (cudaDeviceSynchronize() != cudaSuccess) rc = set_err(ctx, PODECM_ECUDA, "engines: init failed");
  }
  if (rc) {
    podecm_rom_engines_destroy(e);
    return rc;
  }
  *out = e;
  return PODECM_OK;
}

void podecm_rom_engines_destroy(podecm_rom_engines* e) {
  if (!e) return;
  for (double* p : {e->d_geom, e->d_Sc, e->d_St, e->d_ac, e->d_at, e->d_fc, e->d_ft, e->d_fref, e->d_ires})
    cudaFree(p);
  for (int32_t* p : {e->d_ok, e->d_oor, e->d_status}) cudaFree(p);
  delete e;
}

int podecm_rom_engines_respond(podecm_ctx* ctx, void* stream, podecm_rom_engines* e, const double* fbar,
                               const podecm_newton* opts, double* pbar, double* abar, int32_t* iters,
                               int32_t* status) {
  if (!ctx || !e || !opts) return PODECM_ECONFIG;
  if (!fbar || !pbar) return set_err(ctx, PODECM_ECONFIG, "engines: fbar and pbar required");
  auto s = static_cast<cudaStream_t>(stream);
  podecm_rom* r = e->rom;
  const int64_t n = e->n;
  if (e->has_bounds) {
    Bounds b;
    for (int k = 0; k < 3; ++k) {
      b.lo[k] = e->bounds[2 * k];
      b.hi[k] = e->bounds[2 * k + 1];
    }
    k_eng_oor<<<grid_for(n, 128), 128, 0, s>>>(n, fbar, b, e->d_oor);
    PODECM_LAUNCHED(ctx, 1);
  }
  int32_t* st = status ? status : e->d_status;
  RomStart start;
  start.S = e->d_Sc;
  start.a = e->d_ac;
  start.fprev = e->d_fc;
  start.fref = e->d_fref;
  start.init_res = e->d_ires;
  if (int rc = rom_solve_impl(ctx, stream, r, n, e->d_geom, fbar, 1, opts, pbar, iters, nullptr, e->d_at, st,
                              nullptr, start))
    return rc;
  k_eng_keep<<<grid_for(n * r->Q, 128), 128, 0, s>>>(n, r->Q, st, r->d_ctl, r->d_S, r->cap, fbar, e->d_ires,
                                                     e->d_St, e->d_ft, e->d_fref, e->d_ok);
  PODECM_LAUNCHED(ctx, 1);
  if (abar) {  // rom_effective_stiffness(states_ committed, fbar, a_trial) (twoscale.cpp:85-88)
    if (int rc = ensure_abar(r, n, false)) return rc;
    return abar_stage(ctx, s, r, n, e->d_Sc, fbar, 4, abar, st);
  }
  return PODECM_OK;
}

int podecm_rom_engines_commit(podecm_ctx* ctx, void* stream, podecm_rom_engines* e) {
  if (!ctx || !e) return PODECM_ECONFIG;
  auto s = static_cast<cudaStream_t>(stream);
  podecm_rom* r = e->rom;
  k_eng_commit<<<grid_for(e->n * r->Q, 128), 128, 0, s>>>(e->n, r->Q, r->N, e->d_ok, e->d_St, e->d_at, e->d_ft,
                                                          e->d_Sc, e->d_ac, e->d_fc);
  PODECM_LAUNCHED(ctx, 1);
  return PODECM_OK;
}

int podecm_rom_engines_out_of_range(podecm_ctx* ctx, void* stream, const podecm_rom_engines* e,
                                    int32_t* counts) {
  if (!ctx || !e || !counts) return PODECM_ECONFIG;
  PODECM_CUDA_TRY(ctx, cudaMemcpyAsync(counts, e->d_oor, (size_t)e->n * sizeof(int32_t),
                                       cudaMemcpyDeviceToDevice, static_cast<cudaStream_t>(stream)));
  return PODECM_OK;
}

}  // extern "C"
