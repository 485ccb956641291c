/*
 * elastodyn_b200.h -- C-ABI of the B200-native Newton-step hot path.
 *
 * Drop-in boundary for the reference library `elastodyn` (C++20, CPU-only).
 * Each entry point replaces one reference interface (file:line under
 * /root/reference/proj); the reference-shaped C++ shim over this ABI is
 * include/elastodyn_b200.hpp, and INTEGRATION.md shows the binding a
 * maintainer adds.  Plain pointers and sizes only; no torch/CUDA types.
 *
 * Conventions (mirroring the reference):
 *  - every call is synchronous at return, like the reference's free functions;
 *  - host arrays are caller-owned and copied; device state belongs to ed_ctx;
 *  - errors are status codes; a reference-shaped C++ caller maps
 *    ED_ELEMENT_INVERSION -> ElementInversion (materials.hpp:16-19),
 *    ED_ZERO_DIAGONAL -> std::runtime_error (precond.cpp:15-17),
 *    ED_INVALID_ARGUMENT -> std::invalid_argument (krylov.cpp:26-28);
 *  - non-convergence is a flag in ed_linear_stats / ed_solve_result, never an
 *    error (krylov.hpp:79-83);
 *  - there is no CPU fallback: without a CUDA device ed_ctx_create fails.
 */
#ifndef ELASTODYN_B200_H
#define ELASTODYN_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum ed_status {
    ED_OK = 0,
    ED_ELEMENT_INVERSION = 1, /* J <= 0 in some element (materials.cpp:87, assembly.cpp:81-86) */
    ED_ZERO_DIAGONAL = 2,     /* build_shat: |A_ii| < 1e-300 (precond.cpp:15-17) */
    ED_INVALID_ARGUMENT = 3,  /* size / option mismatch (krylov.cpp:26-28, amg.cpp:191-193) */
    ED_CUDA_ERROR = 4,
    ED_NOT_READY = 5,         /* call order violated (e.g. solve before a tangent exists) */
    ED_UNSUPPORTED = 6        /* outside this build's scope (e.g. partially constrained nodes) */
};

typedef struct ed_ctx ed_ctx;

/* KrylovConfig, krylov.hpp:64-69 */
typedef struct {
    int32_t restart;
    int32_t max_iters;
    double rel_tol;
    double abs_tol;
} ed_krylov_config;

/* AmgOptions, amg.hpp:16-37.  use_dof_row_maps = 1 reproduces set_amg_maps
 * (driver.cpp:32-48): row_to_node/row_component taken from the DofMap. */
typedef struct {
    int32_t block_size;
    int32_t max_levels;
    int32_t coarse_max_rows;
    int32_t smoother; /* 0 = Jacobi, 1 = symmetric Gauss-Seidel (default) */
    int32_t pre_sweeps;
    int32_t post_sweeps;
    int32_t smooth_prolongator;
    int32_t use_dof_row_maps;
    double strength_theta;
    double jacobi_weight;
} ed_amg_options;

/* BlockSolverOptions, precond.hpp:167-175 (PrecondKind order, :159-165) */
typedef struct {
    int32_t precond; /* PrecondKind: 0 Nested, 1 Simple, 2 Ilu0, 3 Jacobi, 4 None (all built) */
    int32_t scale;
    ed_krylov_config outer, a, s, inner; /* outer; ScrTolerances a/s/inner (precond.hpp:83-87) */
    ed_amg_options amg_a, amg_s;
    double eps_diag;
} ed_block_solver_options;

/* LinearStats, precond.hpp:19-49 */
typedef struct {
    int64_t outer_iters, a_solves, a_iters, s_solves, s_iters, schur_applies, inner_iters;
    int32_t converged;
    int32_t pad;
    double t_solve;
} ed_linear_stats;

/* SolveResult, krylov.hpp:71-77 (history is returned through a caller buffer) */
typedef struct {
    int32_t converged;
    int32_t iterations;
    double initial_norm;
    double final_norm;
} ed_solve_result;

/* Material, materials.hpp:137-157.  kind 0: NeoHookeanIsochoric (:101-113);
 * kind 1: DispersedFiberIsochoric (:120-132, materials.cpp:8-53).
 * incompressible selects IncompressibleVolumetric (:74-85), else
 * CompressibleVolumetric(rho0, kappa) (:41-71). */
typedef struct {
    int32_t kind;
    int32_t incompressible;
    double rho0, mu, kappa;
    double k1, k2;
    double h1[9], h2[9]; /* fibre structure tensors H_i = kd I + (1-3kd) a_i (x) a_i */
} ed_material;

/* TimeScalars, assembly.hpp:62-71 */
typedef struct {
    double dt, alpha_m, alpha_f, gamma;
} ed_time_scalars;

/* Per-phase device timings of the last ed_newton_first_pass (milliseconds). */
typedef struct {
    double residual_ms, tangent_ms, planes_ms, shat_ms, amg_setup_ms, fgmres_ms, update_ms, total_ms;
    double amg_host_ms; /* host part of amg_setup_ms */
    int64_t kernel_launches;
} ed_phase_times;

/* ---- context ------------------------------------------------------------ */
int ed_ctx_create(int device, ed_ctx** out);
void ed_ctx_destroy(ed_ctx* ctx);
const char* ed_last_error(const ed_ctx* ctx);
int ed_ctx_set_threads(ed_ctx* ctx, int n_threads); /* host threads for AMG setup */
int64_t ed_kernel_launches(const ed_ctx* ctx);      /* launches issued so far by this context */

/* ---- problem definition (Mesh mesh.hpp:24-50, DofMap assembly.hpp:17-26,
 *      StabilizationParams :54-59, Loads :42-50) ------------------------- */
/* tets: 4 per element (positively oriented, as after finalize_geometry,
 * mesh.cpp:94-103); grad_n: 12 per element [a][I]; volume, tau per element. */
int ed_mesh_upload(ed_ctx* ctx, int n_nodes, int n_tets, const int32_t* tets,
                   const double* grad_n, const double* volume, const double* tau);
/* fixed: 3 bytes per node (DofMap::build, assembly.cpp:11-27).  Nodes must be
 * fully free or fully fixed (else ED_UNSUPPORTED).  Returns nv, np. */
int ed_dofs_build(ed_ctx* ctx, const uint8_t* fixed, int32_t* nv, int32_t* np);
int ed_set_material(ed_ctx* ctx, const ed_material* mat);
/* Dead tractions (assembly.cpp:173-184): one entry per (traction, facet) in
 * the reference's loop order: 3 node ids, facet_area/3, traction vector h. */
int ed_set_loads(ed_ctx* ctx, const double body_force[3], int n_facets,
                 const int32_t* facet_nodes, const double* facet_third, const double* facet_h);

/* ---- cfg-3 enablers: extensions the reference does not have,
 *      so their parity is pinned by this repo's own restatement only --------- */
/* Per-element fibre structure tensors for material kind 1: h = [n_tets][2][9]
 * (H_1, H_2 of each element, row-major), e.g. fibres in a local circumferential
 * frame.  Replaces the global constants of the reference's DispersedFiberIsochoric
 * (materials.cpp:67-80, materials.hpp:120-132); h == NULL returns to the
 * material's global h1 / h2.  With every element's entry equal to the global
 * tensors the assembly is bitwise the global-fibre one. */
int ed_set_fiber_field(ed_ctx* ctx, int n_tets, const double* h);
/* Prescribed displacement (inhomogeneous Dirichlet) for the NEXT
 * ed_step_generalized_alpha call: u = [n][3] end-of-step displacement of the n
 * listed nodes, which must be fully fixed (ED_INVALID_ARGUMENT otherwise).  The
 * reference supports homogeneous constraints only (assembly.hpp:28-30): there
 * the state at fixed nodes never changes.  Here, after the predictor
 * (timeint.cpp:57-61), the iterate at those nodes is set to u and to the
 * end-of-step rates the generalized-alpha update formulas give for it
 * (udot = (u - u_n)/(gamma dt) + (gamma-1)/gamma udot_n, v = udot, vdot alike),
 * so the stage blends (timeint.cpp:88-93) interpolate the boundary motion; the
 * Newton increments stay zero there.  One-shot: consumed by the step.  n = 0
 * clears a pending prescription. */
int ed_set_prescribed_displacement(ed_ctx* ctx, int n, const int32_t* nodes, const double* u);

/* ---- state (State, assembly.hpp:31-37): full-length host arrays ---------- */
int ed_state_upload(ed_ctx* ctx, const double* u, const double* udot, const double* p,
                    const double* pdot, const double* v, const double* vdot);
int ed_state_download(ed_ctx* ctx, double* u, double* udot, double* p, double* pdot,
                      double* v, double* vdot);

/* ---- assembly (assembly.hpp:88-94) --------------------------------------- */
/* assemble_residuals at the uploaded (stage) state; r_m (nv), r_p (np) host,
 * may be null to keep the result on the device.  On ED_ELEMENT_INVERSION,
 * *bad_element holds the smallest inverted element id. */
int ed_assemble_residuals(ed_ctx* ctx, double* r_m, double* r_p, int32_t* bad_element);
/* assemble_tangent at the uploaded state; the blocks stay on the device.
 * rk (nv, host or null = zero) is the kinematic residual whose fold-in
 * (A - A_rate) rk and (C - C_rate) rk (timeint.cpp:144-154) is formed
 * element-locally; A_rate / C_rate are never stored. */
int ed_assemble_tangent(ed_ctx* ctx, const ed_time_scalars* ts, const double* rk,
                        int32_t* bad_element);
/* Export one plane of the assembled tangent as CSR (which: 0 A, 1 B, 2 C,
 * 3 D).  Call with rowptr == null to get dims[0..2] = nrows, ncols, nnz. */
int ed_tangent_export(ed_ctx* ctx, int which, int32_t* dims, int32_t* rowptr, int32_t* col,
                      double* val);
/* Fold-in vectors (A - A_rate) rk (nv) and (C - C_rate) rk (np). */
int ed_foldin_download(ed_ctx* ctx, double* fv, double* fp);

/* ---- block system input from CSR (BlockMatrix, blocksystem.hpp:19-34) ----
 * Replaces the context's tangent with caller CSR blocks A (nv x nv), B
 * (nv x np), C (np x nv), D (np x np) with sorted columns. */
int ed_block_system_upload(ed_ctx* ctx, int nv, int np, const int32_t* a_rp,
                           const int32_t* a_c, const double* a_v, const int32_t* b_rp,
                           const int32_t* b_c, const double* b_v, const int32_t* c_rp,
                           const int32_t* c_c, const double* c_v, const int32_t* d_rp,
                           const int32_t* d_c, const double* d_v);

/* ---- solve (solve_block_system, precond.hpp:182-183 / precond.cpp:157-218) */
/* x (n = nv+np) overwritten (zero initial guess).  history (outer FGMRES
 * residual estimates, SolveResult.history) optional. */
int ed_solve_block_system(ed_ctx* ctx, const double* rhs, double* x,
                          const ed_block_solver_options* opts, ed_linear_stats* stats,
                          double* history, int32_t history_cap, int32_t* history_len);
/* Same on device pointers (rhs, x in device memory owned by the caller). */
int ed_solve_block_system_device(ed_ctx* ctx, const double* d_rhs, double* d_x,
                                 const ed_block_solver_options* opts, ed_linear_stats* stats,
                                 double* history, int32_t history_cap, int32_t* history_len);

/* ---- one Newton step: the first corrector pass of step_generalized_alpha
 * (timeint.cpp:54-176) from the uploaded state y_n, device-resident:
 * predictor, stage blend, residual, ||R||, tangent + fold-in, solve,
 * two-stage update.  The context state becomes the updated iterate.  x (host,
 * n) and history optional.  out_norm = ||R|| (timeint.cpp:110). */
int ed_newton_first_pass(ed_ctx* ctx, const ed_time_scalars* ts, const ed_block_solver_options* opts,
                         double* x, double* out_norm, ed_linear_stats* stats, double* history,
                         int32_t history_cap, int32_t* history_len, ed_phase_times* times);

/* NonlinearConfig (timeint.hpp:26-30). */
typedef struct {
    double tol_R, tol_A;
    int32_t l_max, pad;
} ed_nonlinear_config;

/* StepStats (timeint.hpp:35-45) without the vectors (res_history is an
 * out-array of the call); linear = the accumulated LinearStats. */
typedef struct {
    int32_t converged, newton_iters, n_res, pad;
    double res0, res_final, t_assembly;
} ed_step_stats;

/* One generalized-alpha time step (step_generalized_alpha, timeint.cpp:40-180)
 * from the uploaded state y_n, which becomes y_{n+1}: predictor, corrector
 * passes with the admissibility guard (element inversion, non-finite or
 * >4x-growing residual: halve the last update, up to 30 times), the Newton
 * convergence test ||R|| <= max(tol_R ||R_0||, tol_A), tangent, fold-in,
 * solve_block_system and the two-stage update -- all on the device, one
 * scalar read-back per pass.  res_history gets ||R_(l)|| per pass (up to
 * res_cap). */
int ed_step_generalized_alpha(ed_ctx* ctx, const ed_time_scalars* ts, const ed_nonlinear_config* nl,
                              const ed_block_solver_options* opts, ed_step_stats* out, ed_linear_stats* linear,
                              double* res_history, int32_t res_cap);

/* ---- debug / parity entry points ----------------------------------------- */
/* y = K x (BlockMatrix::matvec, blocksystem.hpp:27-33) on the current system
 * (unscaled), host vectors of length nv+np. */
int ed_block_matvec(ed_ctx* ctx, const double* x, double* y);
/* The same product on the solver's working copy of the current mesh system (scaled when
 * opts->scale, blocksystem.cpp:79-106), through the coupled 4x4 BSR operator the outer FGMRES
 * uses (y_coupled) and through the four BSR planes (y_planes): kernel-level parity of the two
 * storages of K. */
int ed_coupled_matvec(ed_ctx* ctx, const ed_block_solver_options* opts, const double* x,
                      double* y_coupled, double* y_planes);
/* gmres/fgmres (krylov.cpp:180-192) on the current A block (unscaled), with
 * precond 0 none, 1 Jacobi, 2 AMG(amg).  x holds the initial guess. */
int ed_gmres_a(ed_ctx* ctx, const double* b, double* x, const ed_krylov_config* cfg,
               int flexible, int precond, const ed_amg_options* amg, ed_solve_result* res,
               double* history, int32_t history_cap, int32_t* history_len);
/* AmgHierarchy::build + vcycle (amg.cpp:189-362) on the current A block
 * (which = 0) or on S_hat of the current (scaled when opts->scale) system
 * (which = 1). info[0] = n_levels, info[1] = fallback, info[2..] = rows. */
int ed_amg_vcycle(ed_ctx* ctx, int which, const ed_block_solver_options* opts,
                  const double* r, double* z, int32_t* info);
/* build_shat (precond.cpp:10-24) of the current system after the solver's
 * scaling (opts->scale) -- CSR export, two-phase like ed_tangent_export. */
int ed_shat_export(ed_ctx* ctx, const ed_block_solver_options* opts, int32_t* dims,
                   int32_t* rowptr, int32_t* col, double* val);

/* ---- device-resident benchmark helpers ----------------------------------- */
/* Coupled K x on device vectors, n_rep times (SpMV roofline). */
int ed_block_matvec_device(ed_ctx* ctx, const double* d_x, double* d_y, int n_rep, float* ms);
/* Bytes moved per coupled SpMV / per A-plane SpMV (algorithmic). */
int ed_spmv_bytes(ed_ctx* ctx, double* coupled_bytes, double* a_plane_bytes);
/* Keep / restore a device-side copy of the state (benchmark steps restart
 * from the same y_n without host traffic). */
int ed_state_save(ed_ctx* ctx);
int ed_state_restore(ed_ctx* ctx);
/* CUDA events on the context's stream: op 0 records the start event, op 1
 * records the stop event, synchronises and returns the elapsed ms. */
int ed_timer(ed_ctx* ctx, int op, float* ms);
/* Device-timed hot kernels on the current (solver-scaled) system, n_rep
 * launches each.  out[2k] = average ms per launch, out[2k+1] = algorithmic
 * bytes per launch, for k = 0 coupled K x, 1 A-plane SpMV, 2 fine-level
 * Gauss-Seidel forward sweep on A, 3 S_hat SpMV. */
int ed_bench_kernels(ed_ctx* ctx, const ed_block_solver_options* opts, int n_rep, double* out);
/* Device-timed assembly (after one ed_assemble_tangent): out[0] residual ms
 * (element kernels + tractions), out[1] its algorithmic bytes, out[2] tangent ms
 * (element kernels with the fold-in + BSR planes), out[3] its algorithmic bytes,
 * out[4] measured FP64 FMA peak GFLOP/s, out[5] elements, out[6] plane bytes,
 * out[7] K4 staging bytes. */
int ed_bench_assembly(ed_ctx* ctx, const ed_time_scalars* ts, int n_rep, double* out);
/* Live kernel accounting: while on, every sparse launch (SpMV, Gauss-Seidel
 * half sweep) is bracketed by CUDA events on its stream and attributed to
 * "kernel@level" with its algorithmic bytes.  on = 1 clears the totals. */
int ed_kernel_accounting(ed_ctx* ctx, int on);
/* Number of accounted kernel classes (resolves pending events). */
int ed_kernel_account_count(ed_ctx* ctx, int* n);
/* Class idx: name, launches, total device ms, total algorithmic bytes. */
int ed_kernel_account_get(ed_ctx* ctx, int idx, char* name, int name_cap, int64_t* launches, double* ms,
                          double* bytes);

#ifdef __cplusplus
}
#endif

#endif /* ELASTODYN_B200_H */
