// Krylov vector layer for sm_100a (FP64): fused axpy/dot/norm kernels with
// warp-shuffle + single-pass grid reductions (the last CTA to finish sums
// the per-CTA partials in a fixed order), so every reduction is
// deterministic for a given length.  Compiled with -fmad=false so the
// elementwise updates round exactly like the reference's host loops
// (krylov.cpp:78-159, csr.cpp:213-227).
#include <cuda_runtime.h>

#include <algorithm>

#include "ed_internal.hpp"

namespace edb {

namespace {

constexpr int kRT = 256;        // reduction CTA size
constexpr int kMaxRBlocks = 4 * 148;
constexpr int kGroup = 8;       // vectors per CTA in multi-dot

__device__ __forceinline__ double warp_sum(double v)
{
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = v + __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// Reduce NV values across the CTA; thread 0 stores them to partials[k*nb + blockIdx.x].
template <int NV>
__device__ __forceinline__ void cta_store(double (&v)[NV], double* partials, int nb, int bx)
{
    __shared__ double sm[NV][kRT / 32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int k = 0; k < NV; ++k) {
        const double s = warp_sum(v[k]);
        if (lane == 0) sm[k][warp] = s;
    }
    __syncthreads();
    if (threadIdx.x < NV) {
        double s = 0.0;
#pragma unroll
        for (int w = 0; w < kRT / 32; ++w) s = s + sm[threadIdx.x][w];
        partials[static_cast<int64_t>(threadIdx.x) * nb + bx] = s;
    }
}

// Returns true in exactly one CTA (the last to arrive); resets the ticket.
__device__ __forceinline__ bool last_cta(unsigned int* ticket, unsigned int total)
{
    __shared__ bool last;
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned int t = atomicAdd(ticket, 1u);
        last = (t == total - 1);
        if (last) *ticket = 0u;
    }
    __syncthreads();
    if (last) __threadfence();
    return last;
}

__device__ __forceinline__ double sum_partials(const double* p, int nb)
{
    double s = 0.0;
    for (int b = 0; b < nb; ++b) s = s + __ldcg(p + b);
    return s;
}

// out = x.y (or sqrt when SQRT)
template <bool SQRT>
__global__ void __launch_bounds__(kRT) k_dot(const double* __restrict__ x, const double* __restrict__ y, int64_t n,
                                             double* partials, unsigned int* ticket, double* out)
{
    double v[1] = {0.0};
    const int nb = gridDim.x;
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * kRT + threadIdx.x; i < n;
         i += static_cast<int64_t>(nb) * kRT)
        v[0] = v[0] + x[i] * y[i];
    cta_store<1>(v, partials, nb, blockIdx.x);
    if (last_cta(ticket, nb) && threadIdx.x == 0) {
        const double s = sum_partials(partials, nb);
        *out = SQRT ? sqrt(s) : s;
    }
}

// MGS step: w -= hprev*vprev (when hprev); out = vnext . w  (w.w if !vnext)
__global__ void __launch_bounds__(kRT) k_mgs(double* w, const double* __restrict__ vprev,
                                             const double* __restrict__ hprev, const double* __restrict__ vnext,
                                             int64_t n, double* partials, unsigned int* ticket, double* out)
{
    double v[1] = {0.0};
    const int nb = gridDim.x;
    const double h = hprev ? *hprev : 0.0;
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * kRT + threadIdx.x; i < n;
         i += static_cast<int64_t>(nb) * kRT) {
        double wi = w[i];
        if (hprev) {
            wi = wi - h * vprev[i]; // krylov.cpp:85
            w[i] = wi;
        }
        v[0] = v[0] + (vnext ? vnext[i] * wi : wi * wi);
    }
    cta_store<1>(v, partials, nb, blockIdx.x);
    if (last_cta(ticket, nb) && threadIdx.x == 0) *out = sum_partials(partials, nb);
}

// corr[i] = V_i . w for i < k; grid (nb, ceil(k/kGroup)).
__global__ void __launch_bounds__(kRT) k_multi_dot(const double* const* __restrict__ V, int k,
                                                   const double* __restrict__ w, int64_t n, double* partials,
                                                   unsigned int* ticket, double* corr)
{
    const int nb = gridDim.x;
    const int g0 = blockIdx.y * kGroup;
    double v[kGroup];
#pragma unroll
    for (int q = 0; q < kGroup; ++q) v[q] = 0.0;
    const double* vp[kGroup];
#pragma unroll
    for (int q = 0; q < kGroup; ++q) vp[q] = (g0 + q < k) ? V[g0 + q] : nullptr;
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * kRT + threadIdx.x; i < n;
         i += static_cast<int64_t>(nb) * kRT) {
        const double wi = w[i];
#pragma unroll
        for (int q = 0; q < kGroup; ++q)
            if (vp[q]) v[q] = v[q] + vp[q][i] * wi;
    }
    // partial layout: [vector][block]
    cta_store<kGroup>(v, partials + static_cast<int64_t>(g0) * nb, nb, blockIdx.x);
    if (last_cta(ticket, nb * gridDim.y)) {
        for (int q = threadIdx.x; q < k; q += blockDim.x)
            corr[q] = sum_partials(partials + static_cast<int64_t>(q) * nb, nb);
    }
}

// krylov.cpp:87-105 decision: sc[0] = |w|^2 in; sc[1] = flag; sc[2] = wnorm
__global__ void k_reorth_decide(double* sc, double* h, const double* corr, int k)
{
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    const double wnorm = sqrt(sc[0]);
    double loss = 0.0;
    for (int i = 0; i < k; ++i) loss = fmax(loss, fabs(corr[i]));
    const bool flag = wnorm > 0.0 && loss / wnorm > 1e-8;
    if (flag)
        for (int i = 0; i < k; ++i) h[i] = h[i] + corr[i];
    sc[1] = flag ? 1.0 : 0.0;
    sc[2] = wnorm;
}

// if flag: w -= sum_i corr_i V_i (i ascending per element), sc[2] = |w|
__global__ void __launch_bounds__(kRT) k_reorth_apply(double* w, const double* const* __restrict__ V,
                                                      const double* __restrict__ corr, int k, int64_t n, double* sc,
                                                      double* partials, unsigned int* ticket)
{
    if (sc[1] == 0.0) return; // uniform across the grid: no CTA touches the ticket
    double v[1] = {0.0};
    const int nb = gridDim.x;
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * kRT + threadIdx.x; i < n;
         i += static_cast<int64_t>(nb) * kRT) {
        double wi = w[i];
        for (int q = 0; q < k; ++q) wi = wi - corr[q] * V[q][i];
        w[i] = wi;
        v[0] = v[0] + wi * wi;
    }
    cta_store<1>(v, partials, nb, blockIdx.x);
    if (last_cta(ticket, nb) && threadIdx.x == 0) {
        const double s = sum_partials(partials, nb);
        sc[0] = s;
        sc[2] = sqrt(s);
    }
}

// x += sum_i y[i] V_i   (vec_axpy sequence, krylov.cpp:148/152)
__global__ void k_multi_axpy(double* x, const double* const* __restrict__ V, const double* __restrict__ y, int k,
                             int64_t n)
{
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        double xi = x[i];
        for (int q = 0; q < k; ++q) xi = xi + y[q] * V[q][i];
        x[i] = xi;
    }
}

__global__ void k_fill(double* x, double v, int64_t n)
{
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        x[i] = v;
}

__global__ void k_sub_from(double* r, const double* __restrict__ b, int64_t n)
{
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        r[i] = b[i] - r[i];
}

__global__ void k_mul(double* x, const double* __restrict__ w, int64_t n)
{
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        x[i] = x[i] * w[i];
}

__global__ void k_add(double* x, const double* __restrict__ y, int64_t n)
{
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        x[i] = x[i] + y[i];
}

__global__ void k_div_scalar(double* y, const double* __restrict__ x, const double* __restrict__ d,
                             const double* __restrict__ guard, int64_t n)
{
    if (guard && !(*guard > 1e-300)) return;
    const double s = *d;
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        y[i] = x[i] / s; // krylov.cpp:58,109 divide (not multiply by the inverse)
}

inline int ew_grid(int64_t n)
{
    const int64_t g = (n + 255) / 256;
    return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(g, 148 * 8)));
}

} // namespace

int reduce_blocks(int64_t n)
{
    const int64_t nb = (n + kRT * 4 - 1) / (kRT * 4);
    return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(nb, kMaxRBlocks)));
}

void Reducer::ensure(int vals, cudaStream_t s)
{
    const int need_vals = std::max(vals, kGroup);
    if (max_vals >= need_vals && partials.p) return;
    max_blocks = kMaxRBlocks;
    max_vals = std::max(need_vals, 2 * max_vals);
    partials.alloc(static_cast<size_t>(max_vals + kGroup) * max_blocks);
    if (!ticket.p) {
        ticket.alloc(1);
        ticket.zero(s);
    }
}

void dot(Reducer& R, const double* x, const double* y, int64_t n, double* out, cudaStream_t s)
{
    R.ensure(1, s);
    acct_vec("k_dot", 16.0 * n);
    k_dot<false><<<reduce_blocks(n), kRT, 0, s>>>(x, y, n, R.partials.p, R.ticket.p, out);
    after_launch("k_dot");
}

void norm2(Reducer& R, const double* x, int64_t n, double* out, cudaStream_t s)
{
    R.ensure(1, s);
    acct_vec("k_norm", 8.0 * n);
    k_dot<true><<<reduce_blocks(n), kRT, 0, s>>>(x, x, n, R.partials.p, R.ticket.p, out);
    after_launch("k_norm");
}

void mgs_axpy_dot(Reducer& R, double* w, const double* vprev, const double* hprev, const double* vnext,
                  int64_t n, double* hout, cudaStream_t s)
{
    R.ensure(1, s);
    acct_vec("k_mgs", 32.0 * n);
    k_mgs<<<reduce_blocks(n), kRT, 0, s>>>(w, vprev, hprev, vnext, n, R.partials.p, R.ticket.p, hout);
    after_launch("k_mgs");
}

void multi_dot(Reducer& R, const double* const* dV, int k, const double* w, int64_t n, double* corr,
               cudaStream_t s)
{
    if (k <= 0) return;
    const int groups = (k + kGroup - 1) / kGroup;
    R.ensure(groups * kGroup, s);
    dim3 grid(reduce_blocks(n), groups);
    acct_vec("k_multi_dot", 8.0 * n * (k + 1));
    k_multi_dot<<<grid, kRT, 0, s>>>(dV, k, w, n, R.partials.p, R.ticket.p, corr);
    after_launch("k_multi_dot");
}

void reorth_decide(double* sc, double* h, const double* corr, int k, cudaStream_t s)
{
    k_reorth_decide<<<1, 32, 0, s>>>(sc, h, corr, k);
    after_launch("k_reorth_decide");
}

void reorth_apply(Reducer& R, double* w, const double* const* dV, const double* corr, int k, int64_t n,
                  double* sc, cudaStream_t s)
{
    R.ensure(1, s);
    acct_vec("k_reorth_apply", 8.0 * n * (k + 2));
    k_reorth_apply<<<reduce_blocks(n), kRT, 0, s>>>(w, dV, corr, k, n, sc, R.partials.p, R.ticket.p);
    after_launch("k_reorth_apply");
}

void multi_axpy(double* x, const double* const* dV, const double* y, int k, int64_t n, cudaStream_t s)
{
    if (n == 0 || k == 0) return;
    acct_vec("k_multi_axpy", 8.0 * n * (k + 2));
    k_multi_axpy<<<ew_grid(n), 256, 0, s>>>(x, dV, y, k, n);
    after_launch("k_multi_axpy");
}

void vec_fill(double* x, double v, int64_t n, cudaStream_t s)
{
    if (n == 0) return;
    acct_vec("k_fill", 8.0 * n);
    k_fill<<<ew_grid(n), 256, 0, s>>>(x, v, n);
    after_launch("k_fill");
}

void vec_copy(double* y, const double* x, int64_t n, cudaStream_t s)
{
    if (n == 0 || y == x) return;
    acct_vec("copy", 16.0 * n);
    ED_CUDA(cudaMemcpyAsync(y, x, n * sizeof(double), cudaMemcpyDeviceToDevice, s));
}

void vec_sub_from(double* r, const double* b, int64_t n, cudaStream_t s)
{
    if (n == 0) return;
    acct_vec("k_sub_from", 24.0 * n);
    k_sub_from<<<ew_grid(n), 256, 0, s>>>(r, b, n);
    after_launch("k_sub_from");
}

void vec_mul(double* x, const double* w, int64_t n, cudaStream_t s)
{
    if (n == 0) return;
    acct_vec("k_mul", 24.0 * n);
    k_mul<<<ew_grid(n), 256, 0, s>>>(x, w, n);
    after_launch("k_mul");
}

void vec_add(double* x, const double* y, int64_t n, cudaStream_t s)
{
    if (n == 0) return;
    acct_vec("k_add", 24.0 * n);
    k_add<<<ew_grid(n), 256, 0, s>>>(x, y, n);
    after_launch("k_add");
}

void vec_div_scalar(double* y, const double* x, const double* d, const double* guard, int64_t n,
                    cudaStream_t s)
{
    if (n == 0) return;
    acct_vec("k_div_scalar", 16.0 * n);
    k_div_scalar<<<ew_grid(n), 256, 0, s>>>(y, x, d, guard, n);
    after_launch("k_div_scalar");
}

} // namespace edb
