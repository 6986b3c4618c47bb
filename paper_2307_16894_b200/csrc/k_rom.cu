// K3 — batched hyper-reduced online stage (BASELINE config 3).  [in progress]
#include "rve.cuh"

using namespace podecm_impl;

struct podecm_rom {
  podecm_rve* rve = nullptr;
  int N = 0, Q = 0;
};

extern "C" {

int podecm_rom_create(podecm_ctx* ctx, podecm_rve* rve, int N, int Q, const int32_t* ids,
                      const double* weights, const double* mode_grads, podecm_rom** out) {
  (void)rve; (void)N; (void)Q; (void)ids; (void)weights; (void)mode_grads; (void)out;
  return set_err(ctx, PODECM_ECONFIG, "podecm_rom_create: not built yet");
}

void podecm_rom_destroy(podecm_rom* rom) { delete rom; }

int podecm_rom_solve_batch(podecm_ctx* ctx, void* stream, podecm_rom* rom, int64_t n_inst,
                           const double* geom, const double* sched, int K,
                           const podecm_newton* opts, double* pbar, int32_t* iters, double* resid,
                           double* a_final, int32_t* status) {
  (void)stream; (void)rom; (void)n_inst; (void)geom; (void)sched; (void)K; (void)opts;
  (void)pbar; (void)iters; (void)resid; (void)a_final; (void)status;
  return set_err(ctx, PODECM_ECONFIG, "podecm_rom_solve_batch: not built yet");
}

}  // extern "C"
