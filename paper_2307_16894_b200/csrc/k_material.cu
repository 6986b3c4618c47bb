// K1 — batched material-point update (BASELINE config 1) and the context
// entry points of the C-ABI.
//
// One thread per point, SoA fp64 planes: every plane access of a warp is one
// contiguous 256-byte run (fully coalesced); outputs use streaming stores so
// the 208 B/point write stream does not evict the input stream from L2.
// The kernel is FP64-issue bound (9 evaluations x ~450 DP instructions per
// point against 288 B of HBM traffic); see DESIGN.md §K1.
#include <cuda_runtime.h>

#include <cstdlib>
#include <algorithm>
#include <cstring>

#include "common.cuh"

using namespace podecm_dev;
using namespace podecm_impl;

namespace {

template <bool PAIR, int MINB>
__global__ void __launch_bounds__(128, MINB) k_material_batch(
    int64_t n, MatTable tab, int n_mats, const int32_t* __restrict__ region,
    const double* __restrict__ F, const double* __restrict__ st, double* __restrict__ P,
    double* __restrict__ A, double* __restrict__ st_out, int32_t* __restrict__ status,
    unsigned int* __restrict__ fail, double h_rel, double* __restrict__ extra) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    int r = region ? __ldg(region + i) : 0;
    r = (r < 0 || r >= n_mats) ? 0 : r;
    const MatConst& p = tab.m[r];
    double f[4], fp[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) f[k] = __ldg(F + k * n + i);
#pragma unroll
    for (int k = 0; k < 4; ++k) fp[k] = __ldg(st + k * n + i);
    Frozen z;
    freeze(fp, __ldg(st + 4 * n + i), __ldg(st + 5 * n + i), z);
    double pv[4];
    FullOut fo;
    bool ok = lsu_eval<true>(p, z, f, pv, &fo);
#pragma unroll
    for (int k = 0; k < 4; ++k) __stcs(P + k * n + i, pv[k]);
    if (extra) {
      extra[i] = fo.dgamma;
      extra[n + i] = fo.f_trial;
      extra[2 * n + i] = fo.q_trial;
      extra[3 * n + i] = fo.mises;
    }
    if (st_out) {
#pragma unroll
      for (int k = 0; k < 4; ++k) __stcs(st_out + k * n + i, fo.fp[k]);
      __stcs(st_out + 4 * n + i, fo.fpzz);
      __stcs(st_out + 5 * n + i, fo.xi);
    }
    if (ok && A) {
      // columns go straight to their planes: A[(r + 4e) * n + i]
      auto sink = [&](int e, const double col[4]) {
#pragma unroll
        for (int r = 0; r < 4; ++r) __stcs(A + (int64_t)(r + 4 * e) * n + i, col[r]);
      };
      ok = fd_tangent<PAIR>(p, z, f, h_rel, sink);
    }
    if (status) status[i] = ok ? 0 : PODECM_ESOLVE;
    if (!ok) atomicAdd(fail, 1u);
  }
}

// Slab variant: the point's operands sit in a shared-memory slab column
// (material.cuh, SlabSrc) instead of registers across the 9 evaluations.
// UNI: one material for every point (no region map, as in config 1): the
// constants are then kernel-parameter operands at fixed offsets instead of
// loads at a per-point index.
template <int MINB, bool UNI = false>
__global__ void __launch_bounds__(128, MINB) k_material_slab(
    int64_t n, MatTable tab, int n_mats, const int32_t* __restrict__ region,
    const double* __restrict__ F, const double* __restrict__ st, double* __restrict__ P,
    double* __restrict__ A, double* __restrict__ st_out, int32_t* __restrict__ status,
    unsigned int* __restrict__ fail, double h_rel, double* __restrict__ extra) {
  constexpr int S = 128;
  __shared__ double slab[kSlabSlots * S];
  volatile double* c = slab + threadIdx.x;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    int r = (!UNI && region) ? __ldg(region + i) : 0;
    r = (r < 0 || r >= n_mats) ? 0 : r;
    const MatConst& p = UNI ? tab.m[0] : tab.m[r];
    {
      double f[4], fp[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) f[k] = __ldg(F + k * n + i);
#pragma unroll
      for (int k = 0; k < 4; ++k) fp[k] = __ldg(st + k * n + i);
      slab_load<S>(c, f, fp, __ldg(st + 4 * n + i), __ldg(st + 5 * n + i));
    }
    bool ok;
    {
      double pv[4];
      FullOut fo;
      ok = lsu_eval_src<true>(p, SlabSrc<S>{c}, pv, &fo);
#pragma unroll
      for (int k = 0; k < 4; ++k) __stcs(P + k * n + i, pv[k]);
      if (extra) {
        extra[i] = fo.dgamma;
        extra[n + i] = fo.f_trial;
        extra[2 * n + i] = fo.q_trial;
        extra[3 * n + i] = fo.mises;
      }
      if (st_out) {
#pragma unroll
        for (int k = 0; k < 4; ++k) __stcs(st_out + k * n + i, fo.fp[k]);
        __stcs(st_out + 4 * n + i, fo.fpzz);
        __stcs(st_out + 5 * n + i, fo.xi);
      }
    }
    if (ok && A) {
      auto sink = [&](int e, const double col[4]) {
#pragma unroll
        for (int r = 0; r < 4; ++r) __stcs(A + (int64_t)(r + 4 * e) * n + i, col[r]);
      };
      ok = fd_tangent_slab<S>(p, c, h_rel, sink);
    }
    if (status) status[i] = ok ? 0 : PODECM_ESOLVE;
    if (!ok) atomicAdd(fail, 1u);
  }
}

// Variant table (FD pairing x register budget, register- or slab-resident
// operands); the default was chosen by measurement on B200:
// the slab kernel at 7 CTAs/SM (71 registers) runs 1.074 ms per config-1
// step against 1.146 ms for the best register-resident one (<false, 5>).
// PODECM_K1_VARIANT overrides it.
using KFn = void (*)(int64_t, MatTable, int, const int32_t*, const double*, const double*, double*,
                     double*, double*, int32_t*, unsigned int*, double, double*);
const KFn kVariants[] = {k_material_batch<true, 3>, k_material_batch<true, 4>,
                         k_material_batch<false, 4>, k_material_batch<false, 5>,
                         k_material_slab<6>,         k_material_slab<7>,
                         k_material_slab<8>};
// uniform-material forms of the slab variants 4, 5, 6
const KFn kUniVariants[] = {k_material_slab<6, true>, k_material_slab<7, true>, k_material_slab<8, true>};
constexpr int kNVariants = sizeof(kVariants) / sizeof(kVariants[0]);

constexpr int kDefaultVariant = 5;

int k1_variant() {
  static int v = [] {
    const char* e = getenv("PODECM_K1_VARIANT");
    int x = e ? atoi(e) : kDefaultVariant;
    return (x >= 0 && x < kNVariants) ? x : kDefaultVariant;
  }();
  return v;
}

}  // namespace

extern "C" {

int podecm_ctx_create(int device, podecm_ctx** out) {
  if (!out) return PODECM_ECONFIG;
  *out = nullptr;
  auto* ctx = new podecm_ctx;
  ctx->device = device;
  cudaError_t e = cudaSetDevice(device);
  if (e == cudaSuccess) e = cudaDeviceGetAttribute(&ctx->n_sm, cudaDevAttrMultiProcessorCount, device);
  if (e == cudaSuccess) e = cudaMalloc(&ctx->d_fail, sizeof(unsigned int));
  if (e == cudaSuccess) e = cudaMemset(ctx->d_fail, 0, sizeof(unsigned int));
  if (e != cudaSuccess) {
    delete ctx;
    return PODECM_ECUDA;
  }
  *out = ctx;
  return PODECM_OK;
}

void podecm_ctx_destroy(podecm_ctx* ctx) {
  if (!ctx) return;
  if (ctx->d_fail) cudaFree(ctx->d_fail);
  delete ctx;
}

const char* podecm_last_error(const podecm_ctx* ctx) {
  return ctx ? ctx->last_error.c_str() : "null context";
}

int64_t podecm_launch_count(const podecm_ctx* ctx) { return ctx ? ctx->launches.load() : 0; }

void podecm_set_timing(podecm_ctx* ctx, int on) {
  if (ctx) ctx->timing = on != 0;
}

// Synchronises the device, then returns the per-kernel-name totals (ms) and
// launch counts recorded since the last call; names are '\n'-separated.
int podecm_get_timings(podecm_ctx* ctx, char* names, int names_len, double* ms, int64_t* counts,
                       int max_items) {
  if (!ctx) return -1;
  cudaDeviceSynchronize();
  std::vector<std::string> nm;
  std::vector<double> tot;
  std::vector<int64_t> cnt;
  for (auto& r : ctx->recs) {
    float t = 0.f;
    cudaEventElapsedTime(&t, r.a, r.b);
    size_t k = 0;
    while (k < nm.size() && nm[k] != r.name) ++k;
    if (k == nm.size()) {
      nm.push_back(r.name);
      tot.push_back(0.0);
      cnt.push_back(0);
    }
    tot[k] += t;
    cnt[k] += 1;
    ctx->pool.push_back(r.a);
    ctx->pool.push_back(r.b);
  }
  ctx->recs.clear();
  std::string joined;
  const int n = (int)std::min<size_t>(nm.size(), (size_t)max_items);
  for (int k = 0; k < n; ++k) {
    joined += nm[k];
    joined += '\n';
    if (ms) ms[k] = tot[k];
    if (counts) counts[k] = cnt[k];
  }
  if (names && names_len > 0) {
    std::strncpy(names, joined.c_str(), names_len - 1);
    names[names_len - 1] = 0;
  }
  return n;
}

int podecm_check(podecm_ctx* ctx, void* stream) {
  if (!ctx) return PODECM_ECONFIG;
  unsigned int h = 0;
  auto s = static_cast<cudaStream_t>(stream);
  PODECM_CUDA_TRY(ctx, cudaMemcpyAsync(&h, ctx->d_fail, sizeof(h), cudaMemcpyDeviceToHost, s));
  PODECM_CUDA_TRY(ctx, cudaStreamSynchronize(s));
  if (h == 0) return PODECM_OK;
  PODECM_CUDA_TRY(ctx, cudaMemsetAsync(ctx->d_fail, 0, sizeof(unsigned int), s));
  PODECM_CUDA_TRY(ctx, cudaStreamSynchronize(s));
  return set_err(ctx, PODECM_ESOLVE,
                 std::to_string(h) +
                     " item(s) raised SolveError: plasticity update hit a non-positive elastic "
                     "stretch, or a cell Newton did not converge");
}

int podecm_material_batch(podecm_ctx* ctx, void* stream, int64_t n, const podecm_params* mats,
                          int n_mats, const int32_t* region, const double* F, const double* st_in,
                          double* P, double* A, double* st_out, int32_t* status, double h_rel) {
  return podecm_material_batch_ex(ctx, stream, n, mats, n_mats, region, F, st_in, P, A, st_out, status,
                                  h_rel, nullptr);
}

int podecm_material_batch_ex(podecm_ctx* ctx, void* stream, int64_t n, const podecm_params* mats,
                             int n_mats, const int32_t* region, const double* F, const double* st_in,
                             double* P, double* A, double* st_out, int32_t* status, double h_rel,
                             double* extra) {
  if (!ctx) return PODECM_ECONFIG;
  if (int rc = check_params(ctx, mats, n_mats)) return rc;
  if (n < 0) return set_err(ctx, PODECM_ECONFIG, "negative point count");
  if (n == 0) return PODECM_OK;
  if (!F || !st_in || !P) return set_err(ctx, PODECM_ECONFIG, "F, st_in and P are required");
  if (!(h_rel > 0)) return set_err(ctx, PODECM_ECONFIG, "h_rel must be positive");
  const MatTable tab = make_table(mats, n_mats);
  const int block = 128;
  const int64_t blocks = (n + block - 1) / block;
  // CTAs per SM of the grid-stride loop: 224 = 32 waves of 7 resident CTAs, so
  // config 1 (32,768 blocks) runs one point per thread and the last partial
  // wave is short (64 gave 3-or-4-point CTAs: 1.065 vs 1.053 ms per step)
  static const int64_t gmult = [] {
    const char* e = getenv("PODECM_K1_GRID_MULT");
    return (int64_t)(e ? std::max(1, atoi(e)) : 224);
  }();
  const int grid = (int)(blocks < (int64_t)ctx->n_sm * gmult ? blocks : (int64_t)ctx->n_sm * gmult);
  KTimer kt(ctx, static_cast<cudaStream_t>(stream), "k_material_batch");
  const int v = k1_variant();
  const bool uni = (!region || n_mats == 1) && v >= 4 && v <= 6;
  (uni ? kUniVariants[v - 4] : kVariants[v])<<<grid, block, 0, static_cast<cudaStream_t>(stream)>>>(
      n, tab, n_mats, region, F, st_in, P, A, st_out, status, ctx->d_fail, h_rel, extra);
  PODECM_LAUNCHED(ctx, 1);
  return PODECM_OK;
}

}  // extern "C"
