// Launch interfaces of the assembly / system / Newton-pass kernels.
#pragma once

#include "ed_internal.hpp"

namespace edb {

struct AsmArgs {
    const int* tets = nullptr;
    const double* grad_n = nullptr;
    const double* volume = nullptr;
    const double* tau = nullptr;
    const int* fidx = nullptr; // node -> free index or -1
    const double* elem_h = nullptr; // [E][2][9] per-element fibre structure tensors, or null (global)
    const double *u = nullptr, *udot = nullptr, *p = nullptr, *pdot = nullptr, *v = nullptr, *vdot = nullptr;
    const double* rk = nullptr; // kinematic residual (nv) for the fold-in, or null
    const int* elem_order = nullptr;
    const int* k4slot = nullptr; // [E][16] PN block of node pair (a, b)
    double* k4 = nullptr;        // [nnzb_PN][16]
    double* r_m = nullptr;
    double* r_p = nullptr;
    double* fv = nullptr;
    double* fp = nullptr;
    int* bad_element = nullptr;
    ed_material mat{};
    ed_time_scalars ts{};
    double body_force[3] = {0.0, 0.0, 0.0};
};

void launch_residual(const AsmArgs& A, const std::vector<int>& color_ptr, cudaStream_t s);
void launch_tangent(const AsmArgs& A, const std::vector<int>& color_ptr, cudaStream_t s);
void launch_traction(const int64_t* rowptr, const int* rows, const double* vals, int nrows_with, double* r_m,
                     cudaStream_t s);
// FP64 FMA probe: returns the flops of one launch
double launch_fp64_fma(double* out, int iters, cudaStream_t s);
void launch_k4_to_plane(int plane, const int* src, const double* k4, double* val, int64_t nnzb, cudaStream_t s);
// all four planes from K4 in one pass (dst*: stored block of each K4 slot per plane, -1 none)
void launch_k4_split(const double* k4, const int* dstA, const int* dstB, const int* dstC, const int* dstD, double* A,
                     double* B, double* C, double* D, int64_t nslots, cudaStream_t s);

// ---- system kernels (kernels_system.cu) ----
// max |x_i| over [0, n) into *out (deterministic)
void absmax(Reducer& R, const double* x, int64_t n, double* out, cudaStream_t s);
// compute_block_scaling (blocksystem.cpp:53-77): w_i = |d_i|^-1/2 when
// |d_i| > eps * dmax of its block, else 1; da (nv), dd (np) -> w (nv+np)
void block_weights(const double* da, const double* dd, int nv, int np, const double* amax, const double* dmax,
                   double eps, double* w, cudaStream_t s);
// inv_da = 1/diag(A) with the build_shat zero-diagonal guard (precond.cpp:12-19)
void shat_inv_diag(const double* da, double* inv_da, int nv, double eps, int* bad_row, cudaStream_t s);

struct ShatArgs {
    // S_hat (rows = pressure nodes, 1x1 blocks, stored in level order)
    const int* s_rowptr;
    const int* s_perm;
    double* s_val;
    int s_nrows;
    // C plane (pressure rows, 1 x Bv) and D (1x1), natural row order
    const int* c_rowptr;
    const int* c_col;
    const double* c_val;
    const int* d_rowptr;
    const double* d_val;
    // B plane (velocity block rows, Bv x 1), stored in A's level order
    const int* b_rowptr;
    const int* b_inv;
    const double* b_val;
    const double* inv_da;
    // position maps
    const int64_t* cb_off;  // per pressure row
    const uint16_t* cb_pos; // per (C block, B block) pair
    const int64_t* d_off;
    const uint16_t* d_pos;  // per D block
    int Bv;
};
void launch_shat_numeric(const ShatArgs& a, cudaStream_t s);

// ---- Newton first-pass elementwise kernels (timeint.cpp:57-176) ----
struct NewtonArgs {
    const double *yn_u, *yn_udot, *yn_p, *yn_pdot, *yn_v, *yn_vdot;
    double *cur_u, *cur_udot, *cur_p, *cur_pdot, *cur_v, *cur_vdot;
    double *mid_u, *mid_udot, *mid_p, *mid_pdot, *mid_v, *mid_vdot;
    int n_nodes;
    double pf, alpha_m, alpha_f;
};
void launch_predict_blend(const NewtonArgs& a, cudaStream_t s);
// Prescribed boundary motion (extension; the reference has homogeneous constraints only,
// assembly.hpp:28-30): at the listed fully fixed nodes cur_u = u_t and the end-of-step
// rates follow the generalized-alpha update formulas, cur_udot = (u_t - u_n)/(gamma dt) + pf udot_n,
// cur_v = cur_udot, cur_vdot = (cur_v - v_n)/(gamma dt) + pf vdot_n.
void launch_prescribe(const int* nodes, const double* u_t, int n, const NewtonArgs& a, double gdt, cudaStream_t s);
// mid = blend(yn, cur) (timeint.cpp:88-93)
void launch_stage_blend(const NewtonArgs& a, cudaStream_t s);
// cur = blend(prev, cur, 0.5) with prev in the yn_* slots (timeint.cpp:131-136)
void launch_halve(const NewtonArgs& a, cudaStream_t s);
// rk[r] = mid_udot[idx] - mid_v[idx] over free rows
void launch_kinematic_residual(const int* fnode, int nfree, const double* mid_udot, const double* mid_v, double* rk,
                               cudaStream_t s);
// rhs = [-rm + fv/chi ; -rp + fp/chi]
void launch_rhs(const double* rm, const double* rp, const double* fv, const double* fp, int nv, int np, double chi,
                double* rhs, cudaStream_t s);
// two-stage update (timeint.cpp:160-176)
void launch_update(const int* fnode, int nfree, int np, const double* x, const double* rk, double chi, double am,
                   double gdt, double* u, double* udot, double* v, double* vdot, double* p, double* pdot,
                   cudaStream_t s);

} // namespace edb
