// Shared plumbing of the C-ABI implementation: context, error codes,
// launch accounting.
#pragma once

#include <cuda_runtime.h>

#include <atomic>
#include <cstdio>
#include <string>
#include <vector>

#include "../../include/podecm_cuda.h"
#include "material.cuh"

struct podecm_ctx {
  int device = 0;
  int n_sm = 148;
  std::string last_error;
  unsigned int* d_fail = nullptr;  // device-side SolveError counter
  std::atomic<int64_t> launches{0};
  // optional per-kernel event timing (podecm_set_timing)
  bool timing = false;
  struct Rec {
    const char* name;
    cudaEvent_t a, b;
  };
  std::vector<Rec> recs;
  std::vector<cudaEvent_t> pool;
};

namespace podecm_impl {

inline int set_err(podecm_ctx* ctx, int code, const std::string& msg) {
  if (ctx) ctx->last_error = msg;
  return code;
}

inline int cuda_err(podecm_ctx* ctx, cudaError_t e, const char* where) {
  return set_err(ctx, PODECM_ECUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

#define PODECM_CUDA_TRY(ctx, expr)                                  \
  do {                                                              \
    cudaError_t _e = (expr);                                        \
    if (_e != cudaSuccess) return podecm_impl::cuda_err(ctx, _e, #expr); \
  } while (0)

#define PODECM_LAUNCHED(ctx, n)                                           \
  do {                                                                    \
    cudaError_t _e = cudaGetLastError();                                  \
    if (_e != cudaSuccess) return podecm_impl::cuda_err(ctx, _e, "launch"); \
    (ctx)->launches += (n);                                               \
  } while (0)

// Reference material constants (material.hpp:15-16, material.cpp:82-104).
inline podecm_dev::MatConst make_const(const podecm_params& p) {
  podecm_dev::MatConst c;
  const double E = p.E, nu = p.nu;
  c.la = E * nu / ((1 + nu) * (1 - 2 * nu));
  c.mu = E / (2 * (1 + nu));
  c.two_mu = 2 * c.mu;
  c.three_mu = 3 * c.mu;
  c.three_mu_H = 3 * c.mu + p.H;
  c.yield0 = p.sigma_y0 + p.H * 0.0;  // SmallState{}.xi == 0 (material.cpp:137)
  c.H = p.H;
  c.rcp_3muH = 1.0 / c.three_mu_H;
  return c;
}

inline int check_params(podecm_ctx* ctx, const podecm_params* mats, int n_mats) {
  if (!mats || n_mats <= 0 || n_mats > 8)
    return set_err(ctx, PODECM_ECONFIG, "material table must hold 1..8 parameter sets");
  for (int k = 0; k < n_mats; ++k)
    if (!(mats[k].E > 0) || !(mats[k].nu > -1 && mats[k].nu < 0.5) || mats[k].H < 0)
      return set_err(ctx, PODECM_ECONFIG, "invalid material parameters");
  return PODECM_OK;
}

struct MatTable {
  podecm_dev::MatConst m[8];
};

inline MatTable make_table(const podecm_params* mats, int n_mats) {
  MatTable t{};
  for (int k = 0; k < n_mats; ++k) t.m[k] = make_const(mats[k]);
  return t;
}

inline int grid_for(int64_t n, int block) { return (int)((n + block - 1) / block); }

inline cudaEvent_t pool_event(podecm_ctx* ctx) {
  if (!ctx->pool.empty()) {
    cudaEvent_t e = ctx->pool.back();
    ctx->pool.pop_back();
    return e;
  }
  cudaEvent_t e;
  cudaEventCreate(&e);
  return e;
}

// RAII bracket that records start/stop events around one launch on `s`
// when the context's timing mode is on.
struct KTimer {
  podecm_ctx* ctx;
  cudaStream_t s;
  const char* name;
  cudaEvent_t a = nullptr;
  KTimer(podecm_ctx* c, cudaStream_t st, const char* n) : ctx(c), s(st), name(n) {
    if (ctx->timing) {
      a = pool_event(ctx);
      cudaEventRecord(a, s);
    }
  }
  ~KTimer() {
    if (a) {
      cudaEvent_t b = pool_event(ctx);
      cudaEventRecord(b, s);
      ctx->recs.push_back({name, a, b});
    }
  }
};

}  // namespace podecm_impl
