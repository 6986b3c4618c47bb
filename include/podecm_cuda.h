/*
 * podecm_cuda.h — C-ABI drop-in boundary of the B200-native (sm_100a) hot
 * path of the POD + ECM reduced-order model (arXiv 2307.16894).
 *
 * Plain pointers and sizes only; no C++, Eigen or torch types cross it.  Each
 * entry point replaces one reference interface from /root/reference/proj
 * (cited per declaration).  INTEGRATION.md shows the binding the reference
 * side would add.
 *
 * Conventions
 *   - Device pointers unless stated "host".  The ABI never frees caller
 *     memory.  Calls are stream-ordered on the caller's cudaStream_t (passed
 *     as void*; NULL = legacy default stream) and return once launched.
 *   - Return codes: 0 OK, 2 configuration/shape error (reference
 *     ConfigError), 3 solve error (reference SolveError), 4 CUDA error.
 *     Per-item failures (a material point that hits a non-positive elastic
 *     stretch, an instance whose Newton/bisection gives up) are reported in
 *     the nullable per-item status[] arrays (0 ok / 3 SolveError) and in a
 *     context-wide flag that podecm_check() collects (it synchronises the
 *     stream and returns 3 with the reference's message when any item
 *     failed).  podecm_last_error() returns the last message.
 *   - Tensor layout follows the reference (types.hpp:21-48): a 2x2 tensor is
 *     flattened column-stacked (A00, A10, A01, A11); a 4x4 tangent is the
 *     Eigen::Matrix4d storage, entry (r, c) at r + 4c with r = i + 2j,
 *     c = k + 2l.  Batched arrays are structure-of-arrays: component-major
 *     planes of length n ("[4][n]").
 *   - Material history ("state") is 6 planes: Fp00, Fp10, Fp01, Fp11, Fp_zz,
 *     xi (PlasticState, material.hpp:55-59).
 */
#ifndef PODECM_CUDA_H
#define PODECM_CUDA_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PODECM_OK 0
#define PODECM_ECONFIG 2
#define PODECM_ESOLVE 3
#define PODECM_ECUDA 4
#define PODECM_EIO 5     /* IoError (types.hpp:50-53); the reference CLI exits 2 */
#define PODECM_EFORMAT 6 /* FormatError (types.hpp:55-58); the reference CLI exits 2 */

typedef struct podecm_ctx podecm_ctx;
typedef struct podecm_rve podecm_rve;
typedef struct podecm_rom podecm_rom;

/* PlasticityParams, material.hpp:9-17 (lambda/mu derived as in :15-16). */
typedef struct podecm_params {
  double E, nu, sigma_y0, H;
} podecm_params;

/* NewtonOpts, microfem.hpp:45-56. */
typedef struct podecm_newton {
  double eps_rel, eps_abs, force_ref;
  int32_t max_iter;
  int32_t max_bisect; /* rom_solve_step_adaptive default 5, rom.hpp:66-73 */
} podecm_newton;

/* ---- context ------------------------------------------------------------ */
int podecm_ctx_create(int device, podecm_ctx** out);
void podecm_ctx_destroy(podecm_ctx* ctx);
const char* podecm_last_error(const podecm_ctx* ctx);
/* Synchronise `stream`, collect per-item failures flagged since the last
 * check; returns 0 or 3 (SolveError). */
int podecm_check(podecm_ctx* ctx, void* stream);
/* Number of kernels this context has launched (for bench accounting). */
int64_t podecm_launch_count(const podecm_ctx* ctx);
/* Optional per-kernel CUDA-event timing of every launch on its own stream
 * (bench roofline accounting).  podecm_get_timings synchronises the device
 * and returns, per kernel name ('\n'-separated in `names`), the summed ms
 * and launch count since the previous call; returns the number of names. */
void podecm_set_timing(podecm_ctx* ctx, int on);
int podecm_get_timings(podecm_ctx* ctx, char* names, int names_len, double* ms, int64_t* counts,
                       int max_items);

/* ---- (i) material point -------------------------------------------------
 * Replaces large_strain_update + large_strain_tangent per point
 * (material.hpp:69-75; material.cpp:120-181), batched over n points.
 *   mats (host)  : n_mats parameter sets; region (device, nullable) picks one
 *                  per point (default 0).
 *   F [4][n], st_in [6][n]  -> P [4][n], A [16][n] (nullable), st_out [6][n]
 *   (nullable), status [n] (nullable).  h_rel: FD step (reference 1e-7). */
int podecm_material_batch(podecm_ctx* ctx, void* stream, int64_t n, const podecm_params* mats,
                          int n_mats, const int32_t* region, const double* F, const double* st_in,
                          double* P, double* A, double* st_out, int32_t* status, double h_rel);
/* podecm_material_batch plus the remaining LargeResult fields (material.hpp:
 * 61-67): extra [4][n] = dgamma, f_trial, q_trial, mises (nullable). */
int podecm_material_batch_ex(podecm_ctx* ctx, void* stream, int64_t n, const podecm_params* mats,
                             int n_mats, const int32_t* region, const double* F, const double* st_in,
                             double* P, double* A, double* st_out, int32_t* status, double h_rel,
                             double* extra);

/* ---- RVE tables (mesh, quadrature cache, periodic dof map, CSR pattern,
 * deterministic scatter map) ----------------------------------------------
 * Replaces RveProblem::build (microfem.cpp:9-23) with build_quad_cache
 * (mesh.cpp:412-451), periodic_pairs/periodic_dof_map (mesh.cpp:307-374) and
 * the setFromTriplets pattern (microfem.cpp:125-128) for the structured
 * n_cells x n_cells bilinear Q4 unit cell of BASELINE configs 0/2/3
 * (region 1 = element centroid within r0 of the centre). */
int podecm_rve_create_q4(podecm_ctx* ctx, int n_cells, double r0, const podecm_params* mats,
                         int n_mats, podecm_rve** out);
/* Same cell with the caller's element regions (host [n_cells^2], row-major
 * elements as built here; e.g. a reference Mesh::regions) instead of the
 * centroid-within-r0 rule; r0 still parameterises the analytic morph. */
int podecm_rve_create_q4_regions(podecm_ctx* ctx, int n_cells, double r0, const int32_t* regions,
                                 const podecm_params* mats, int n_mats, podecm_rve** out);
void podecm_rve_destroy(podecm_rve* rve);
/* out[0..5] = n_nodes, n_elems, n_qp, n_red, nnz, anchor node. */
int podecm_rve_info(const podecm_rve* rve, int64_t out[6]);
/* Copy the host-side tables out (all host pointers, each nullable):
 * nodes [n_nodes][2], elems [n_elems][4], regions [n_elems],
 * grad [n_qp][4][2], w [n_qp], node_dof [n_nodes], row_ptr [n_red+1],
 * col_idx [nnz], slot_ptr [nnz+1] and slot_terms [n_triplets]: for CSR slot
 * s the triplets (qp*64 + (a*4+b)*4 + i*2 + j) that sum into it, in
 * reference triplet order. */
int podecm_rve_export(const podecm_rve* rve, double* nodes, int32_t* elems, int32_t* regions,
                      double* grad, double* w, int32_t* node_dof, int32_t* row_ptr,
                      int32_t* col_idx, int32_t* slot_ptr, int32_t* slot_terms);
int64_t podecm_rve_n_triplets(const podecm_rve* rve);

/* Analytic morph (BASELINE configs 0/2/3) of one geometry (a, b):
 * fmu_inv [4][n_qp], det [n_qp] (device) — MorphOperator::derive semantics
 * (morph.cpp:97-126) with nodal d(X) from the circle->ellipse map. */
int podecm_rve_morph(podecm_ctx* ctx, void* stream, podecm_rve* rve, int64_t n_inst,
                     const double* geom, double* fmu_inv, double* det, int32_t* status);

/* ---- (ii) batched assembly ----------------------------------------------
 * Replaces assemble (microfem.hpp:74-77; microfem.cpp:56-130) for n_inst
 * independent instances sharing the RVE tables.  Instance-major arrays:
 *   geom [n_inst][2] (a, b) of the analytic morph, or morph (nullable,
 *   overrides geom) [n_inst][5][n_qp] = fmu_inv planes + det plane;
 *   fbar [n_inst][4]; w_red [n_inst][n_red]; st0 [n_inst][6][n_qp];
 *   outputs st1 [n_inst][6][n_qp] (nullable), f [n_inst][n_red],
 *   kvals [n_inst][nnz] (nullable => no tangent, AssemblyOpts.tangent=false),
 *   p_field [n_inst][4][n_qp] (nullable), status [n_inst] (nullable).
 * The CSR values are summed per slot in the reference triplet order (no
 * atomics; bitwise reproducible). */
int podecm_assemble_batch(podecm_ctx* ctx, void* stream, podecm_rve* rve, int64_t n_inst,
                          const double* geom, const double* morph, const double* fbar,
                          const double* w_red, const double* st0, double* st1, double* f,
                          double* kvals, double* p_field, int32_t* status);

/* podecm_assemble_batch plus AssemblyOpts::store_tangent_field
 * (microfem.hpp:58-69): a_field [n_inst][16][n_qp] (plane r + 4c, the FD
 * tangent of every qp; requires kvals). */
int podecm_assemble_batch_ex(podecm_ctx* ctx, void* stream, podecm_rve* rve, int64_t n_inst,
                             const double* geom, const double* morph, const double* fbar,
                             const double* w_red, const double* st0, double* st1, double* f,
                             double* kvals, double* p_field, int32_t* status, double* a_field);

/* ---- (iii) hyper-reduced online stage ------------------------------------
 * RomModel (rom.hpp:15-30) restricted to what the online solve reads:
 * host arrays ids [Q] ascending, weights [Q], mode_grads [Q][N][4]
 * (build_rom, rom.cpp:80-109). */
int podecm_rom_create(podecm_ctx* ctx, podecm_rve* rve, int N, int Q, const int32_t* ids,
                      const double* weights, const double* mode_grads, podecm_rom** out);
void podecm_rom_destroy(podecm_rom* rom);
/* Batch-wide reduced assemblies ("global iterations") of the last solve. */
int64_t podecm_rom_global_iterations(const podecm_rom* rom);
/* Replaces rom_solve (rom.hpp:86-88; rom.cpp:177-200) with
 * rom_solve_step_adaptive (rom.cpp:152-175) for n_inst instances:
 *   geom [n_inst][2]; sched [n_inst][K][4] macro F per increment;
 *   outputs pbar [n_inst][K][4] homogenised stress history,
 *   iters [n_inst][K] (nullable), resid [n_inst][K] (nullable),
 *   a_final [n_inst][N] (nullable), status [n_inst] (nullable).
 * Default "lazy tangent" order: the FD tangent is not evaluated at an
 * iterate that already meets the Newton tolerance (the reference computes
 * and discards it, rom.cpp:132-141), so an FD failure there — which would
 * make the reference bisect — goes unseen; environment PODECM_ROM_LAZY=0
 * selects the strict order. */
int podecm_rom_solve_batch(podecm_ctx* ctx, void* stream, podecm_rom* rom, int64_t n_inst,
                           const double* geom, const double* sched, int K,
                           const podecm_newton* opts, double* pbar, int32_t* iters, double* resid,
                           double* a_final, int32_t* status);
/* podecm_rom_solve_batch plus run_online's effective-stiffness request
 * (pipeline.cpp:456-483): abar [n_inst][16] (nullable) =
 * rom_effective_stiffness at the last macro gradient sched[K-1], the final
 * reduced coordinates and the history committed at the start of the last
 * increment.  Tensor4 storage: abar[s][r + 4c], r = i + 2j, c = k + 2l. */
int podecm_rom_solve_batch_ex(podecm_ctx* ctx, void* stream, podecm_rom* rom, int64_t n_inst,
                              const double* geom, const double* sched, int K,
                              const podecm_newton* opts, double* pbar, int32_t* iters,
                              double* resid, double* a_final, int32_t* status, double* abar);
/* podecm_rom_solve_batch_ex on a caller's MorphField instead of the analytic
 * map: morph_q [n_inst][5][Q] = fmu_inv planes (flatten order) and det at
 * the ECM points (slice_morph, rom.cpp:111-120), e.g. from the reference's
 * MorphOperator::solve (the drop-in rom_solve of dropin/podecm_dropin.cpp);
 * a_hist [n_inst][K][N] (nullable) = RomSolution::steps[k].a. */
int podecm_rom_solve_batch_morph(podecm_ctx* ctx, void* stream, podecm_rom* rom, int64_t n_inst,
                                 const double* morph_q, const double* sched, int K,
                                 const podecm_newton* opts, double* pbar, int32_t* iters,
                                 double* resid, double* a_final, int32_t* status, double* abar,
                                 double* a_hist);
/* Replaces rom_effective_stiffness (rom.hpp:92-95; rom.cpp:202-241) for
 * n_inst instances: geom [n_inst][2]; st0 [n_inst][6][Q] history at the
 * ECM points (planes Fp00, Fp10, Fp01, Fp11, Fp_zz, xi); fbar [n_inst][4];
 * a [n_inst][N] -> abar [n_inst][16] (layout as above), status (nullable). */
int podecm_rom_effective_stiffness_batch(podecm_ctx* ctx, void* stream, podecm_rom* rom,
                                         int64_t n_inst, const double* geom, const double* st0,
                                         const double* fbar, const double* a, double* abar,
                                         int32_t* status);
/* Replaces rom_sensitivity (rom.hpp:100-104; rom.cpp:243-263) on the
 * analytic geometry (a, b): central differences of the final homogenised
 * stress with step h * max(1, |param|); 4 n_inst reduced solves in one batch.
 * grad [n_inst][2][4] (d pbar / d a, d pbar / d b), status (nullable). */
int podecm_rom_sensitivity_batch(podecm_ctx* ctx, void* stream, podecm_rom* rom, int64_t n_inst,
                                 const double* geom, const double* sched, int K,
                                 const podecm_newton* opts, double h, double* grad,
                                 int32_t* status);

/* ---- batched RomMicroEngine (twoscale.hpp:55-80; twoscale.cpp:53-96) ----
 * n hyper-reduced micro engines (one per macro Gauss point) sharing one
 * RomModel; each keeps its committed history, reduced coordinates, macro
 * gradient and force_ref on the device.  geom [n][2] (a, b) of every engine;
 * stretch_bounds (host, nullable) = [3][2] (lo, hi) of (F00, F11, F01). */
typedef struct podecm_rom_engines podecm_rom_engines;
int podecm_rom_engines_create(podecm_ctx* ctx, podecm_rom* rom, int64_t n, const double* geom,
                              const double* stretch_bounds, podecm_rom_engines** out);
void podecm_rom_engines_destroy(podecm_rom_engines* eng);
/* MicroEngine::respond for all engines at once: fbar [n][4] -> pbar [n][4],
 * abar [n][16] (nullable), Newton iterations [n] (nullable), status [n]
 * (nullable; 3 = SolveError of that engine's rom_solve_step_adaptive). */
int podecm_rom_engines_respond(podecm_ctx* ctx, void* stream, podecm_rom_engines* eng,
                               const double* fbar, const podecm_newton* opts, double* pbar,
                               double* abar, int32_t* iters, int32_t* status);
/* MicroEngine::commit for all engines. */
int podecm_rom_engines_commit(podecm_ctx* ctx, void* stream, podecm_rom_engines* eng);
/* RomMicroEngine::out_of_range per engine -> counts [n] (device). */
int podecm_rom_engines_out_of_range(podecm_ctx* ctx, void* stream, const podecm_rom_engines* eng,
                                    int32_t* counts);

/* ---- FE2 macro driver (twoscale.hpp:82-118) -----------
 * MacroConfig: nx x ny Quad8 plate of width x height, bottom edge clamped,
 * parabolic top traction ramped to peak and back over `steps` steps. */
typedef struct podecm_macro_cfg {
  int32_t nx, ny;
  double width, height, peak_traction;
  int32_t steps;
  podecm_newton newton; /* macro Newton (eps_rel, eps_abs, max_iter used) */
} podecm_macro_cfg;
/* out = n_nodes, n_elems, n_qp (4 per element, quadrature order), n_red. */
int podecm_macro_info(const podecm_macro_cfg* cfg, int64_t out[4]);
/* Reference positions of the macro Gauss points (host [n_qp][2]): the
 * engine factory's argument (twoscale.cpp:149-152). */
int podecm_macro_qp_positions(const podecm_macro_cfg* cfg, double* x);
/* run_twoscale (twoscale.cpp:131-242).  eng: the batched ROM micro engines
 * of the n_qp macro Gauss points (quadrature order; micro_opts for their
 * responds), or NULL for LinearElasticEngine(E, nu) at every point.  Host
 * outputs (each nullable): load_factor, compliance, iters [steps]; u_final
 * [2 n_nodes]; residual_norm; micro_evals. */
int podecm_twoscale_run(podecm_ctx* ctx, void* stream, const podecm_macro_cfg* cfg, podecm_rom_engines* eng,
                        const podecm_newton* micro_opts, double E, double nu, double* load_factor,
                        double* compliance, int32_t* iters, double* u_final, double* residual_norm,
                        int64_t* micro_evals);

/* ---- full-order Newton ------------------------------
 * solve_rve with solve_step_adaptive (microfem.cpp:142-238) for a batch of
 * instances around the batched assembly; the sparse solves are one batched
 * LU refactorisation per Newton round (symbolic analysis once per pattern). */
typedef struct podecm_fe podecm_fe;
int podecm_fe_create(podecm_ctx* ctx, podecm_rve* rve, podecm_fe** out);
void podecm_fe_destroy(podecm_fe* fe);
/* Batch-wide Newton rounds of the last solve. */
int64_t podecm_fe_global_iterations(const podecm_fe* fe);
/* geom [n][2]; sched [n][K][4] -> pbar [n][K][4] (RveSolution::steps[k].pbar),
 * iters [n][K], resid [n][K] (nullable), w_final [n][n_red] (nullable),
 * status [n] (nullable; 3 = SolveError). */
int podecm_fe_solve_batch(podecm_ctx* ctx, void* stream, podecm_fe* fe, int64_t n, const double* geom,
                          const double* sched, int K, const podecm_newton* opts, double* pbar,
                          int32_t* iters, double* resid, double* w_final, int32_t* status);
/* podecm_fe_solve_batch plus the per-increment snapshots of collect_snapshots
 * (pipeline.cpp:157-188): w_hist [n][K][n_red] converged fluctuations,
 * p_hist [n][K][4][n_qp] stress fields (each nullable). */
int podecm_fe_solve_batch_ex(podecm_ctx* ctx, void* stream, podecm_fe* fe, int64_t n, const double* geom,
                             const double* sched, int K, const podecm_newton* opts, double* pbar,
                             int32_t* iters, double* resid, double* w_final, int32_t* status,
                             double* w_hist, double* p_hist);
/* weighted_stress_field (ecm.cpp:10-18) on the analytic morph of each
 * instance: p_field [n][4][n_qp] -> W [n][n_qp][4] = P Fmu^-T det (the
 * ECM snapshot layout of podecm_ecm_select). */
int podecm_weighted_stress_field(podecm_ctx* ctx, void* stream, podecm_rve* rve, int64_t n,
                                 const double* geom, const double* p_field, double* W);
/* effective_stiffness (microfem.cpp:240-313) for n instances: geom [n][2],
 * st0 [n][6][n_qp], fbar [n][4], w [n][n_red] -> abar [n][16] (Tensor4
 * storage r + 4c), status [n] (nullable). */
int podecm_fe_effective_stiffness_batch(podecm_ctx* ctx, void* stream, podecm_fe* fe, int64_t n,
                                        const double* geom, const double* st0, const double* fbar,
                                        const double* w, double* abar, int32_t* status);

/* ---- interchange formats ----------------------------
 * PODECM1 named-array container (store.cpp:127-238) holding a RomModel
 * (rom.cpp:265-327).  Host arrays only; no context or device needed.
 * Errors: 5 IoError, 6 FormatError (message: podecm_store_last_error). */
const char* podecm_store_last_error(void);
/* FNV-1a 64-bit (store.hpp:52-54); seed 14695981039346656037 for a fresh hash. */
uint64_t podecm_fnv1a64(const void* data, uint64_t n, uint64_t seed);
/* Mesh::fingerprint (mesh.cpp:158-180) of the Q4 cell: element-kind byte 1
 * (mesh.cpp:160 maps every non-Tri6 kind to 1), no boundary tags. */
uint64_t podecm_rve_fingerprint(const podecm_rve* rve);
/* RomModel::save: modes column-major [N][n_dof] (Eigen MatX storage),
 * ids [Q], weights [Q], mode_grads [Q][N][4]. */
int podecm_rom_model_save(const char* path, uint64_t mesh_tag, int32_t kind, int32_t n_stress_modes,
                          double ecm_eps, int64_t n_dof, int32_t N, const double* modes, int32_t Q,
                          const int32_t* ids, const double* weights, const double* mode_grads);
/* RomModel::load in two calls: the shapes and scalars, then the arrays
 * (each output nullable; layouts as for podecm_rom_model_save). */
int podecm_rom_model_info(const char* path, int64_t* n_dof, int32_t* N, int32_t* Q, uint64_t* mesh_tag,
                          int32_t* kind, int32_t* n_stress_modes, double* ecm_eps);
int podecm_rom_model_read(const char* path, double* modes, int32_t* ids, double* weights,
                          double* mode_grads);

/* ---- (iv) offline POD / ECM (BASELINE config 4) -------------------------
 * Replaces pod_impl / pod_diag (podkit.cpp:43-72, 117-127):
 * C = S^T diag(g) S (n_snap x n_snap, symmetric) for the column-major
 * snapshot matrix S (n_dof x n_snap); gram_diag nullable = identity. */
int podecm_pod_gram(podecm_ctx* ctx, void* stream, const double* S, int64_t n_dof, int n_snap,
                    const double* gram_diag, double* C);
/* Eigen-decomposition of C (overwritten), keep lambda > tol_rel^2 lambda_0,
 * lambda > 0, at most max_modes; modes (column-major n_dof x kept) =
 * S v_i / sqrt(lambda_i) followed by one MGS pass in the diag(g) metric
 * (mgs_pass, podkit.cpp:75-86); evals (device, n_snap) descending;
 * *n_kept on the host.  Synchronises the stream. */
int podecm_pod_modes(podecm_ctx* ctx, void* stream, const double* S, int64_t n_dof, int n_snap,
                     double* C, const double* gram_diag, int max_modes, double tol_rel,
                     double* modes, double* evals, int* n_kept);

/* podecm_pod_modes with the MGS pass optional (mgs = 0: modes = S v_i /
 * sqrt(lambda_i) only).  The row-sharded POD runs it on each
 * rank's dof rows S_k with the all-reduced Gram sum_k S_k^T S_k, gathers the
 * rows and runs podecm_pod_mgs on the whole basis. */
int podecm_pod_modes_ex(podecm_ctx* ctx, void* stream, const double* S, int64_t n_dof, int n_snap,
                        double* C, const double* gram_diag, int max_modes, double tol_rel,
                        double* modes, double* evals, int* n_kept, int mgs);
/* mgs_pass (podkit.cpp:75-86) on k column-major modes (n_dof x k), in the
 * diag(g) metric (gram_diag nullable = identity).  Synchronises the stream. */
int podecm_pod_mgs(podecm_ctx* ctx, void* stream, double* modes, int64_t n_dof, int k, const double* gram_diag);

/* Row-sharded Gram fused with its reduce-scatter over peer memory (SURVEY
 * 8(e), the multi-GPU split of podkit.cpp:46): this rank's partial
 * S_k^T diag(g) S_k (S_k = its dof rows, column-major n_dof x n_snap) is
 * computed by the symmetric DMMA GEMM, whose epilogue stores every element
 * (i, j) straight into the receive slot of the rank owning Gram row i:
 * recv[o] + (rank * (row0[o+1] - row0[o]) + i - row0[o]) * n_snap + j, with
 * recv[o] rank o's receive buffer ([world][rows of o][n_snap]) mapped into
 * this process (podecm_ipc_open; NVLink peer stores across GPUs).  No local
 * partial is materialised and no collective library call is made.  world <=
 * 8; row0 [world + 1] (host) partitions the n_snap Gram rows. */
int podecm_pod_gram_peer(podecm_ctx* ctx, void* stream, const double* S, int64_t n_dof, int n_snap,
                         const double* gram_diag, double* const* recv, int rank, int world, const int64_t* row0);
/* The owner's side of the reduce-scatter once every rank's GEMM has
 * finished: G_rows = sum over k of recv[k] (rows x n_snap), in rank order. */
int podecm_pod_gram_reduce(podecm_ctx* ctx, void* stream, const double* recv, int world, int64_t rows, int n_snap,
                           double* G_rows);
/* count doubles from src to dst (either may be a peer mapping): the
 * all-gather of the reduced Gram rows. */
int podecm_peer_copy(podecm_ctx* ctx, void* stream, double* dst, const double* src, int64_t count);
/* Device buffers that can be exported to other processes (cudaMalloc'ed, so
 * an IPC handle maps exactly them), their CUDA IPC handles (64 bytes) and
 * the mapping of a peer's handle into this process. */
int podecm_dev_alloc(podecm_ctx* ctx, int64_t bytes, void** out);
void podecm_dev_free(void* p);
int podecm_ipc_handle(podecm_ctx* ctx, void* p, unsigned char handle[64]);
int podecm_ipc_open(podecm_ctx* ctx, const unsigned char handle[64], void** out);
void podecm_ipc_close(void* p);

/* EcmOpts (ecm.hpp:28-32) plus stop_at_count: configs 3/4 stop at
 * max_points selected points instead of throwing (documented deviation). */
typedef struct podecm_ecm_opts {
  double eps;
  int32_t volume_row;
  int32_t max_points;
  int32_t stop_at_count;
} podecm_ecm_opts;
/* Mode gradients at every quadrature point, H [n_qp][N][4] flatten order
 * (build_rom's per-point formula, rom.cpp:91-104), from full nodal modes
 * (column-major 2 n_nodes x N). */
int podecm_ecm_mode_grads(podecm_ctx* ctx, void* stream, podecm_rve* rve, const double* modes,
                          int N, double* H);
/* Weighted stress snapshots W [L][n_qp][4] (weighted_stress_field,
 * ecm.cpp:10-18) of L full nodal displacement snapshots U (column-major
 * 2 n_nodes x L): stress-only update from a virgin history at F = I + grad u
 * on the parent (identity-morph) cell. */
int podecm_ecm_stress_snapshots(podecm_ctx* ctx, void* stream, podecm_rve* rve, const double* U,
                                int64_t L, double* W, int32_t* status);
/* Greedy ECM (ecm_integrand + ecm_select, ecm.cpp:20-48, 132-204) on the
 * factored integrand J[(i L + s), q] = H_q[i] . W_s(q) (+ volume row).
 * ids / weights (host, capacity max_points or n_qp) ascending; *n_sel,
 * *resid_rel, *iterations on the host.  Returns 3 on budget exhaustion
 * (without stop_at_count) or stall, like the reference. */
int podecm_ecm_select(podecm_ctx* ctx, void* stream, podecm_rve* rve, const double* H, int N,
                      const double* W, int64_t L, const podecm_ecm_opts* opts, int32_t* ids,
                      double* weights, int* n_sel, double* resid_rel, int* iterations);

/* Candidate-sharded greedy (ecm.cpp:163-173): this rank holds
 * the candidates [q0, q0 + nq_local) of the cell (H [nq_local][N][4], W
 * [L][nq_local][4]); the exchanges run through caller-supplied host
 * callbacks (e.g. torch.distributed / NCCL), each returning 0 on success:
 *   allreduce_sum: in place elementwise sum over ranks of n host doubles;
 *   argmax: in place (score, global index) -> the global best, larger score
 *           then smaller index (index -1 = no positive score on that rank),
 *           and the owning rank;
 *   bcast: in place broadcast of n host doubles from rank root.
 * Outputs as podecm_ecm_select (global ids), identical on every rank. */
typedef struct podecm_ecm_comm {
  void* user;
  int64_t q0, nq_local;
  int (*allreduce_sum)(void* user, double* host, int64_t n);
  int (*argmax)(void* user, double* score, int64_t* index, int* owner);
  int (*bcast)(void* user, double* host, int64_t n, int root);
} podecm_ecm_comm;
int podecm_ecm_select_sharded(podecm_ctx* ctx, void* stream, podecm_rve* rve, const double* H, int N,
                              const double* W, int64_t L, const podecm_ecm_comm* comm,
                              const podecm_ecm_opts* opts, int32_t* ids, double* weights, int* n_sel,
                              double* resid_rel, int* iterations);

/* ---- diagnostics ---------------------------------------------------------
 * FP64 roofline probes (mode 0: DFMA chain, mode 1: mma.sync m8n8k4 f64);
 * *flops receives the flop count of the launch, time it on `stream`. */
int podecm_probe_fp64(podecm_ctx* ctx, void* stream, int mode, int iters, double* scratch,
                      double* flops);
/* Elementwise device arithmetic used by the material kernels (tests only):
 * which 0: a/b, 1: reciprocal-based division, 2: correctly rounded 1/b,
 * 3: 1.0/b, 4: exp(a), 5: log(a). */
int podecm_probe_math(podecm_ctx* ctx, void* stream, int which, int64_t n, const double* a,
                      const double* b, double* out);

#ifdef __cplusplus
}
#endif

#endif /* PODECM_CUDA_H */
