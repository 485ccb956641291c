// System-level kernels: symmetric block scaling, the S_hat numeric SpGEMM on
// a mesh-static pattern, and the elementwise parts of the Newton corrector
// pass.  Compiled with -fmad=false (reference rounding, see kernels_sparse.cu).
#include <cuda_runtime.h>

#include <algorithm>

#include "assembly.hpp"

namespace edb {

namespace {

constexpr int kRT = 256;

__global__ void __launch_bounds__(kRT) k_absmax(const double* __restrict__ x, int64_t n, double* partials,
                                                unsigned int* ticket, double* out)
{
    double m = 0.0;
    const int nb = gridDim.x;
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * kRT + threadIdx.x; i < n;
         i += static_cast<int64_t>(nb) * kRT)
        m = fmax(m, fabs(x[i]));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    __shared__ double sm[kRT / 32];
    if ((threadIdx.x & 31) == 0) sm[threadIdx.x >> 5] = m;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int w = 0; w < kRT / 32; ++w) t = fmax(t, sm[w]);
        partials[blockIdx.x] = t;
    }
    __shared__ bool last;
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned int t = atomicAdd(ticket, 1u);
        last = (t == static_cast<unsigned int>(nb) - 1);
        if (last) *ticket = 0u;
    }
    __syncthreads();
    if (last && threadIdx.x == 0) {
        __threadfence();
        double t = 0.0;
        for (int b = 0; b < nb; ++b) t = fmax(t, __ldcg(partials + b));
        *out = t;
    }
}

__global__ void k_block_weights(const double* __restrict__ da, const double* __restrict__ dd, int nv, int np,
                                const double* __restrict__ amax, const double* __restrict__ dmax, double eps,
                                double* w)
{
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < nv) {
        const double d = fabs(da[i]);
        w[i] = d > eps * *amax ? 1.0 / sqrt(d) : 1.0;
    } else if (i < static_cast<int64_t>(nv) + np) {
        const double d = fabs(dd[i - nv]);
        w[i] = d > eps * *dmax ? 1.0 / sqrt(d) : 1.0;
    }
}

__global__ void k_shat_inv_diag(const double* __restrict__ da, double* inv_da, int nv, double eps, int* bad)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= nv) return;
    const double d = da[i];
    if (fabs(d) < eps) atomicMin(bad, i);
    inv_da[i] = 1.0 / d;
}

// One thread per S_hat row p.  The row is accumulated in place in its
// output segment:
//   acc[q] = sum_{k in C row p, ascending} C[p,k] * (B[k,q] * inv_da[k])
// in the csr_matmul(C, diag(A)^-1 B) order (csr.cpp:143-164), then
// S_hat = D - acc (csr_add(D, cb, 1, -1), csr.cpp:168-198).
template <int BV>
__global__ void __launch_bounds__(kRT) k_shat(ShatArgs a)
{
    const int s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= a.s_nrows) return;
    const int p = a.s_perm ? a.s_perm[s] : s;
    double* out = a.s_val + a.s_rowptr[s];
    const int slen = a.s_rowptr[s + 1] - a.s_rowptr[s];
    for (int t = 0; t < slen; ++t) out[t] = 0.0;
    int64_t mp = a.cb_off[p];
    for (int k1 = a.c_rowptr[p]; k1 < a.c_rowptr[p + 1]; ++k1) {
        const int m = a.c_col[k1];
        const int bs = a.b_inv ? a.b_inv[m] : m;
        const int b0 = a.b_rowptr[bs];
        const int blen = a.b_rowptr[bs + 1] - b0;
#pragma unroll
        for (int c = 0; c < BV; ++c) {
            const double cv = a.c_val[static_cast<int64_t>(k1) * BV + c];
            const double id = a.inv_da[static_cast<int64_t>(m) * BV + c];
            for (int t2 = 0; t2 < blen; ++t2) {
                const double sb = a.b_val[static_cast<int64_t>(b0 + t2) * BV + c] * id; // csr_scale_rows
                const int pos = a.cb_pos[mp + t2];
                out[pos] = out[pos] + cv * sb;
            }
        }
        mp += blen;
    }
    for (int t = 0; t < slen; ++t) out[t] = -out[t];
    const int64_t dp = a.d_off[p];
    for (int k = a.d_rowptr[p]; k < a.d_rowptr[p + 1]; ++k) {
        const int pos = a.d_pos[dp + (k - a.d_rowptr[p])];
        out[pos] = a.d_val[k] + out[pos];
    }
}

__global__ void k_predict_blend(NewtonArgs a)
{
    // The yn_* and cur_* slots may alias (ed_newton_first_pass predicts in
    // place), so every y_n value is read into a register before any store.
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const int64_t n3 = 3 * static_cast<int64_t>(a.n_nodes);
    if (i < n3) {
        const double ud = a.yn_udot[i], vd = a.yn_vdot[i], u = a.yn_u[i], v = a.yn_v[i];
        // predictor: rates scaled by (gamma-1)/gamma (timeint.cpp:57-61)
        const double cud = ud * a.pf;
        const double cvd = vd * a.pf;
        a.cur_udot[i] = cud;
        a.cur_vdot[i] = cvd;
        a.cur_u[i] = u;
        a.cur_v[i] = v;
        // blends (timeint.cpp:88-93, blend at :31-36)
        a.mid_udot[i] = ud + a.alpha_m * (cud - ud);
        a.mid_vdot[i] = vd + a.alpha_m * (cvd - vd);
        a.mid_u[i] = u + a.alpha_f * (u - u);
        a.mid_v[i] = v + a.alpha_f * (v - v);
    }
    if (i < a.n_nodes) {
        const double pd = a.yn_pdot[i], p = a.yn_p[i];
        const double cpd = pd * a.pf;
        a.cur_pdot[i] = cpd;
        a.cur_p[i] = p;
        a.mid_pdot[i] = pd + a.alpha_m * (cpd - pd);
        a.mid_p[i] = p + a.alpha_f * (p - p);
    }
}

__global__ void k_prescribe(const int* __restrict__ nodes, const double* __restrict__ u_t, int n, NewtonArgs a,
                            double gdt)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= 3 * n) return;
    const int64_t idx = 3 * static_cast<int64_t>(nodes[i / 3]) + i % 3;
    const double ut = u_t[i];
    const double cud = (ut - a.yn_u[idx]) / gdt + a.pf * a.yn_udot[idx];
    a.cur_u[idx] = ut;
    a.cur_udot[idx] = cud;
    a.cur_v[idx] = cud;
    a.cur_vdot[idx] = (cud - a.yn_v[idx]) / gdt + a.pf * a.yn_vdot[idx];
}

// stage blends only (timeint.cpp:88-93): mid = blend(yn, cur)
__global__ void k_stage_blend(NewtonArgs a)
{
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const int64_t n3 = 3 * static_cast<int64_t>(a.n_nodes);
    if (i < n3) {
        a.mid_udot[i] = a.yn_udot[i] + a.alpha_m * (a.cur_udot[i] - a.yn_udot[i]);
        a.mid_vdot[i] = a.yn_vdot[i] + a.alpha_m * (a.cur_vdot[i] - a.yn_vdot[i]);
        a.mid_u[i] = a.yn_u[i] + a.alpha_f * (a.cur_u[i] - a.yn_u[i]);
        a.mid_v[i] = a.yn_v[i] + a.alpha_f * (a.cur_v[i] - a.yn_v[i]);
    }
    if (i < a.n_nodes) {
        a.mid_pdot[i] = a.yn_pdot[i] + a.alpha_m * (a.cur_pdot[i] - a.yn_pdot[i]);
        a.mid_p[i] = a.yn_p[i] + a.alpha_f * (a.cur_p[i] - a.yn_p[i]);
    }
}

// admissibility guard (timeint.cpp:131-136): cur = blend(prev, cur, 0.5);
// here the NewtonArgs' yn_* slots carry prev
__global__ void k_halve(NewtonArgs a)
{
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const int64_t n3 = 3 * static_cast<int64_t>(a.n_nodes);
    if (i < n3) {
        a.cur_udot[i] = a.yn_udot[i] + 0.5 * (a.cur_udot[i] - a.yn_udot[i]);
        a.cur_vdot[i] = a.yn_vdot[i] + 0.5 * (a.cur_vdot[i] - a.yn_vdot[i]);
        a.cur_u[i] = a.yn_u[i] + 0.5 * (a.cur_u[i] - a.yn_u[i]);
        a.cur_v[i] = a.yn_v[i] + 0.5 * (a.cur_v[i] - a.yn_v[i]);
    }
    if (i < a.n_nodes) {
        a.cur_pdot[i] = a.yn_pdot[i] + 0.5 * (a.cur_pdot[i] - a.yn_pdot[i]);
        a.cur_p[i] = a.yn_p[i] + 0.5 * (a.cur_p[i] - a.yn_p[i]);
    }
}

__global__ void k_kin_res(const int* __restrict__ fnode, int nfree, const double* __restrict__ udot,
                          const double* __restrict__ v, double* rk)
{
    const int64_t r = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (r >= 3 * static_cast<int64_t>(nfree)) return;
    const int64_t idx = 3 * static_cast<int64_t>(fnode[r / 3]) + r % 3;
    rk[r] = udot[idx] - v[idx];
}

__global__ void k_rhs(const double* __restrict__ rm, const double* __restrict__ rp, const double* __restrict__ fv,
                      const double* __restrict__ fp, int nv, int np, double chi, double* rhs)
{
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < nv)
        rhs[i] = -rm[i] + fv[i] / chi;
    else if (i < static_cast<int64_t>(nv) + np)
        rhs[i] = -rp[i - nv] + fp[i - nv] / chi;
}

__global__ void k_update(const int* __restrict__ fnode, int nfree, int np, const double* __restrict__ x,
                         const double* __restrict__ rk, double chi, double am, double gdt, double* u, double* udot,
                         double* v, double* vdot, double* p, double* pdot)
{
    const int64_t r = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const int64_t nv = 3 * static_cast<int64_t>(nfree);
    if (r < nv) {
        const int64_t idx = 3 * static_cast<int64_t>(fnode[r / 3]) + r % 3;
        const double dvd = x[r];
        const double dud = (chi / am) * dvd - rk[r] / am;
        vdot[idx] = vdot[idx] + dvd;
        v[idx] = v[idx] + gdt * dvd;
        udot[idx] = udot[idx] + dud;
        u[idx] = u[idx] + gdt * dud;
    }
    if (r < np) {
        const double dpd = x[nv + r];
        pdot[r] = pdot[r] + dpd;
        p[r] = p[r] + gdt * dpd;
    }
}

inline int g1(int64_t n) { return static_cast<int>(std::max<int64_t>(1, (n + 255) / 256)); }

} // namespace

void absmax(Reducer& R, const double* x, int64_t n, double* out, cudaStream_t s)
{
    R.ensure(1, s);
    k_absmax<<<reduce_blocks(n), kRT, 0, s>>>(x, n, R.partials.p, R.ticket.p, out);
    after_launch("k_absmax");
}

void block_weights(const double* da, const double* dd, int nv, int np, const double* amax, const double* dmax,
                   double eps, double* w, cudaStream_t s)
{
    k_block_weights<<<g1(static_cast<int64_t>(nv) + np), 256, 0, s>>>(da, dd, nv, np, amax, dmax, eps, w);
    after_launch("k_block_weights");
}

void shat_inv_diag(const double* da, double* inv_da, int nv, double eps, int* bad_row, cudaStream_t s)
{
    if (nv == 0) return;
    k_shat_inv_diag<<<g1(nv), 256, 0, s>>>(da, inv_da, nv, eps, bad_row);
    after_launch("k_shat_inv_diag");
}

void launch_shat_numeric(const ShatArgs& a, cudaStream_t s)
{
    if (a.s_nrows == 0) return;
    const int g = (a.s_nrows + kRT - 1) / kRT;
    if (a.Bv == 3)
        k_shat<3><<<g, kRT, 0, s>>>(a);
    else
        k_shat<1><<<g, kRT, 0, s>>>(a);
    after_launch("k_shat");
}

void launch_predict_blend(const NewtonArgs& a, cudaStream_t s)
{
    k_predict_blend<<<g1(3 * static_cast<int64_t>(a.n_nodes)), 256, 0, s>>>(a);
    after_launch("k_predict_blend");
}

void launch_prescribe(const int* nodes, const double* u_t, int n, const NewtonArgs& a, double gdt, cudaStream_t s)
{
    if (n == 0) return;
    k_prescribe<<<g1(3 * static_cast<int64_t>(n)), 256, 0, s>>>(nodes, u_t, n, a, gdt);
    after_launch("k_prescribe");
}

void launch_stage_blend(const NewtonArgs& a, cudaStream_t s)
{
    k_stage_blend<<<g1(3 * static_cast<int64_t>(a.n_nodes)), 256, 0, s>>>(a);
    after_launch("k_stage_blend");
}

void launch_halve(const NewtonArgs& a, cudaStream_t s)
{
    k_halve<<<g1(3 * static_cast<int64_t>(a.n_nodes)), 256, 0, s>>>(a);
    after_launch("k_halve");
}

void launch_kinematic_residual(const int* fnode, int nfree, const double* mid_udot, const double* mid_v, double* rk,
                               cudaStream_t s)
{
    if (nfree == 0) return;
    k_kin_res<<<g1(3 * static_cast<int64_t>(nfree)), 256, 0, s>>>(fnode, nfree, mid_udot, mid_v, rk);
    after_launch("k_kin_res");
}

void launch_rhs(const double* rm, const double* rp, const double* fv, const double* fp, int nv, int np, double chi,
                double* rhs, cudaStream_t s)
{
    k_rhs<<<g1(static_cast<int64_t>(nv) + np), 256, 0, s>>>(rm, rp, fv, fp, nv, np, chi, rhs);
    after_launch("k_rhs");
}

void launch_update(const int* fnode, int nfree, int np, const double* x, const double* rk, double chi, double am,
                   double gdt, double* u, double* udot, double* v, double* vdot, double* p, double* pdot,
                   cudaStream_t s)
{
    const int64_t n = std::max<int64_t>(3 * static_cast<int64_t>(nfree), np);
    k_update<<<g1(n), 256, 0, s>>>(fnode, nfree, np, x, rk, chi, am, gdt, u, udot, v, vdot, p, pdot);
    after_launch("k_update");
}


// FP64 FMA throughput probe (bench.py's assembly roofline denominator):
// 8 independent fma chains per thread, 4 resident CTAs of 256 per SM.
__global__ void __launch_bounds__(256) k_fp64_fma(double* out, int iters, double a, double b)
{
    double x[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) x[j] = threadIdx.x * 1e-3 + j;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int j = 0; j < 8; ++j) x[j] = fma(x[j], a, b);
    }
    double acc = 0.0;
#pragma unroll
    for (int j = 0; j < 8; ++j) acc += x[j];
    if (acc == 1.2345e300) out[0] = acc; // keep the chains live
}

double launch_fp64_fma(double* out, int iters, cudaStream_t s)
{
    int dev = 0, sms = 0;
    ED_CUDA(cudaGetDevice(&dev));
    ED_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    const int blocks = sms * 8;
    k_fp64_fma<<<blocks, 256, 0, s>>>(out, iters, 0.999999, 1e-7);
    after_launch("k_fp64_fma");
    return 2.0 * 8.0 * static_cast<double>(iters) * blocks * 256;
}

} // namespace edb
