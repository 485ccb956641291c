// SELL-32 block sparse kernels for sm_100a (FP64, CUDA cores; HBM-bound).
//
// Compiled with -fmad=false: every lane sums its row in the reference's
// column order with separately rounded multiply and add, exactly like the
// host loops of csr.cpp:11-27 and amg.cpp:311-322 (built without FMA), so the
// SpMV and Gauss-Seidel results are bitwise identical to the reference for
// identical inputs.  Bandwidth comes from the layout (one lane per block row,
// entry-major slots -> 256-B coalesced warp loads of values and indices) and
// from the x gathers hitting L2 (stencil neighbours are a few planes away).
#include <cuda_runtime.h>

#include <cstdio>

#include "ed_internal.hpp"

namespace edb {

namespace {

constexpr int kThreads = 256;

inline int grid_for_lanes(int64_t lanes) { return static_cast<int>((lanes + kThreads - 1) / kThreads); }

template <int RB, int CB, int MODE>
__global__ void __launch_bounds__(kThreads)
    k_spmv(const int64_t* __restrict__ soff, const int* __restrict__ perm, const int* __restrict__ rlen,
           const int* __restrict__ col, const double* __restrict__ val, int nslices,
           const double* __restrict__ x, double* y, const double* b)
{
    const int64_t gid = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const int sl = static_cast<int>(gid >> 5);
    const int lane = static_cast<int>(gid & 31);
    if (sl >= nslices) return;
    const int row = perm[gid];
    if (row < 0) return;
    const int len = rlen[gid];
    const int64_t base = soff[sl];
    double acc[RB];
#pragma unroll
    for (int r = 0; r < RB; ++r) acc[r] = 0.0;
#pragma unroll 4
    for (int t = 0; t < len; ++t) {
        const int64_t slot = base + t;
        const int c = __ldg(col + slot * kLanes + lane);
        const double* vp = val + slot * (RB * CB * kLanes) + lane;
        double xv[CB];
#pragma unroll
        for (int d = 0; d < CB; ++d) xv[d] = __ldg(x + static_cast<int64_t>(c) * CB + d);
#pragma unroll
        for (int r = 0; r < RB; ++r)
#pragma unroll
            for (int d = 0; d < CB; ++d) acc[r] = acc[r] + __ldg(vp + (r * CB + d) * kLanes) * xv[d];
    }
#pragma unroll
    for (int r = 0; r < RB; ++r) {
        const int64_t i = static_cast<int64_t>(row) * RB + r;
        if (MODE == 0) y[i] = acc[r];
        if (MODE == 1) y[i] = b[i] - acc[r];
        if (MODE == 2) y[i] = y[i] + acc[r];
    }
}

// y = (M1 x1) + sgn * (M2 x2), both on the same row layout.
template <int RB, int CB1, int CB2>
__global__ void __launch_bounds__(kThreads)
    k_spmv2(const int64_t* __restrict__ soff1, const int* __restrict__ perm, const int* __restrict__ rlen1,
            const int* __restrict__ col1, const double* __restrict__ val1, const int64_t* __restrict__ soff2,
            const int* __restrict__ rlen2, const int* __restrict__ col2, const double* __restrict__ val2,
            int nslices, const double* __restrict__ x1, const double* __restrict__ x2, double* y, double sgn)
{
    const int64_t gid = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const int sl = static_cast<int>(gid >> 5);
    const int lane = static_cast<int>(gid & 31);
    if (sl >= nslices) return;
    const int row = perm[gid];
    if (row < 0) return;
    double a1[RB], a2[RB];
#pragma unroll
    for (int r = 0; r < RB; ++r) a1[r] = a2[r] = 0.0;
    {
        const int len = rlen1[gid];
        const int64_t base = soff1[sl];
#pragma unroll 4
        for (int t = 0; t < len; ++t) {
            const int64_t slot = base + t;
            const int c = __ldg(col1 + slot * kLanes + lane);
            const double* vp = val1 + slot * (RB * CB1 * kLanes) + lane;
            double xv[CB1];
#pragma unroll
            for (int d = 0; d < CB1; ++d) xv[d] = __ldg(x1 + static_cast<int64_t>(c) * CB1 + d);
#pragma unroll
            for (int r = 0; r < RB; ++r)
#pragma unroll
                for (int d = 0; d < CB1; ++d) a1[r] = a1[r] + __ldg(vp + (r * CB1 + d) * kLanes) * xv[d];
        }
    }
    {
        const int len = rlen2[gid];
        const int64_t base = soff2[sl];
#pragma unroll 4
        for (int t = 0; t < len; ++t) {
            const int64_t slot = base + t;
            const int c = __ldg(col2 + slot * kLanes + lane);
            const double* vp = val2 + slot * (RB * CB2 * kLanes) + lane;
            double xv[CB2];
#pragma unroll
            for (int d = 0; d < CB2; ++d) xv[d] = __ldg(x2 + static_cast<int64_t>(c) * CB2 + d);
#pragma unroll
            for (int r = 0; r < RB; ++r)
#pragma unroll
                for (int d = 0; d < CB2; ++d) a2[r] = a2[r] + __ldg(vp + (r * CB2 + d) * kLanes) * xv[d];
        }
    }
#pragma unroll
    for (int r = 0; r < RB; ++r) {
        const int64_t i = static_cast<int64_t>(row) * RB + r;
        // y = acc1 + 1.0*acc2 (matvec_add) or acc1 - acc2 (Schur: D x - C z)
        y[i] = sgn > 0.0 ? a1[r] + a2[r] : a1[r] - a2[r];
    }
}

// One level of an in-place Gauss-Seidel half sweep (amg.cpp:311-322): rows
// of a level are independent; inside a block row the B scalar rows run in
// sweep order, each summing its off-diagonal columns in ascending order.
template <int B, bool FWD>
__global__ void __launch_bounds__(kThreads)
    k_sgs_level(const int64_t* __restrict__ soff, const int* __restrict__ perm, const int* __restrict__ rlen,
                const int* __restrict__ col, const double* __restrict__ val, int s0, int s1,
                const double* __restrict__ bvec, double* z, const double* __restrict__ invd)
{
    const int64_t gid = static_cast<int64_t>(s0) * kLanes + static_cast<int64_t>(blockIdx.x) * blockDim.x +
                        threadIdx.x;
    const int sl = static_cast<int>(gid >> 5);
    const int lane = static_cast<int>(gid & 31);
    if (sl >= s1) return;
    const int row = perm[gid];
    if (row < 0) return;
    const int len = rlen[gid];
    const int64_t base = soff[sl];
#pragma unroll
    for (int ci = 0; ci < B; ++ci) {
        const int cc = FWD ? ci : B - 1 - ci;
        const int64_t i = static_cast<int64_t>(row) * B + cc;
        double acc = bvec[i];
        for (int t = 0; t < len; ++t) {
            const int64_t slot = base + t;
            const int c = col[slot * kLanes + lane];
            const double* vp = val + slot * (B * B * kLanes) + lane + (cc * B) * kLanes;
#pragma unroll
            for (int d = 0; d < B; ++d) {
                if (c == row && d == cc) continue;
                acc = acc - vp[d * kLanes] * z[static_cast<int64_t>(c) * B + d];
            }
        }
        z[i] = acc * invd[i];
    }
}

template <int RB, int CB>
__global__ void __launch_bounds__(kThreads)
    k_scale(const int64_t* __restrict__ soff, const int* __restrict__ perm, const int* __restrict__ rlen,
            const int* __restrict__ col, double* val, int nslices, const double* __restrict__ wr,
            const double* __restrict__ wc)
{
    const int64_t gid = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const int sl = static_cast<int>(gid >> 5);
    const int lane = static_cast<int>(gid & 31);
    if (sl >= nslices) return;
    const int row = perm[gid];
    if (row < 0) return;
    const int len = rlen[gid];
    const int64_t base = soff[sl];
    for (int t = 0; t < len; ++t) {
        const int64_t slot = base + t;
        const int c = col[slot * kLanes + lane];
        double* vp = val + slot * (RB * CB * kLanes) + lane;
#pragma unroll
        for (int r = 0; r < RB; ++r)
#pragma unroll
            for (int d = 0; d < CB; ++d) {
                // blocksystem.cpp:85: val *= wrow[r] * wcol[c]
                const double f = wr[static_cast<int64_t>(row) * RB + r] * wc[static_cast<int64_t>(c) * CB + d];
                vp[(r * CB + d) * kLanes] = vp[(r * CB + d) * kLanes] * f;
            }
    }
}

template <int B>
__global__ void __launch_bounds__(kThreads)
    k_diag(const int64_t* __restrict__ soff, const int* __restrict__ perm, const int* __restrict__ rlen,
           const int* __restrict__ col, const double* __restrict__ val, int nslices, double* d)
{
    const int64_t gid = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const int sl = static_cast<int>(gid >> 5);
    const int lane = static_cast<int>(gid & 31);
    if (sl >= nslices) return;
    const int row = perm[gid];
    if (row < 0) return;
    const int len = rlen[gid];
    const int64_t base = soff[sl];
    double dv[B];
#pragma unroll
    for (int r = 0; r < B; ++r) dv[r] = 0.0;
    for (int t = 0; t < len; ++t) {
        const int64_t slot = base + t;
        if (col[slot * kLanes + lane] == row) {
            const double* vp = val + slot * (B * B * kLanes) + lane;
#pragma unroll
            for (int r = 0; r < B; ++r) dv[r] = vp[(r * B + r) * kLanes];
        }
    }
#pragma unroll
    for (int r = 0; r < B; ++r) d[static_cast<int64_t>(row) * B + r] = dv[r];
}

__global__ void k_inv_diag(const double* __restrict__ d, double* invd, int64_t n)
{
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < n) invd[i] = d[i] != 0.0 ? 1.0 / d[i] : 1.0;
}

__global__ void k_jacobi(double* z, const double* __restrict__ b, const double* __restrict__ t,
                         const double* __restrict__ invd, double w, int64_t n)
{
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < n) z[i] = z[i] + w * invd[i] * (b[i] - t[i]);
}

// z = Pinv r, one warp per row.
__global__ void k_dense_gemv(const double* __restrict__ P, const double* __restrict__ r, double* z, int n)
{
    const int row = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
    const int lane = threadIdx.x & 31;
    if (row >= n) return;
    double s = 0.0;
    for (int j = lane; j < n; j += 32) s = s + P[static_cast<int64_t>(row) * n + j] * r[j];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s = s + __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) z[row] = s;
}

template <int RB, int CB>
void launch_spmv(const Sell& M, const double* x, double* y, const double* b, int mode, cudaStream_t s)
{
    const SellStruct& S = *M.st;
    if (S.nslices == 0) return;
    const int g = grid_for_lanes(static_cast<int64_t>(S.nslices) * kLanes);
    if (mode == 0)
        k_spmv<RB, CB, 0><<<g, kThreads, 0, s>>>(S.slice_off.p, S.perm.p, S.rowlen.p, S.col.p, M.val.p,
                                                 S.nslices, x, y, b);
    else if (mode == 1)
        k_spmv<RB, CB, 1><<<g, kThreads, 0, s>>>(S.slice_off.p, S.perm.p, S.rowlen.p, S.col.p, M.val.p,
                                                 S.nslices, x, y, b);
    else
        k_spmv<RB, CB, 2><<<g, kThreads, 0, s>>>(S.slice_off.p, S.perm.p, S.rowlen.p, S.col.p, M.val.p,
                                                 S.nslices, x, y, b);
    after_launch("k_spmv");
}

template <int RB, int CB1, int CB2>
void launch_spmv2(const Sell& M1, const double* x1, const Sell& M2, const double* x2, double* y, double sgn,
                  cudaStream_t s)
{
    const SellStruct& S1 = *M1.st;
    const SellStruct& S2 = *M2.st;
    if (S1.nslices == 0) return;
    const int g = grid_for_lanes(static_cast<int64_t>(S1.nslices) * kLanes);
    k_spmv2<RB, CB1, CB2><<<g, kThreads, 0, s>>>(S1.slice_off.p, S1.perm.p, S1.rowlen.p, S1.col.p, M1.val.p,
                                                 S2.slice_off.p, S2.rowlen.p, S2.col.p, M2.val.p, S1.nslices,
                                                 x1, x2, y, sgn);
    after_launch("k_spmv2");
}

template <int B>
void launch_sgs(const Sell& A, const double* b, double* z, const double* invd, bool fwd, cudaStream_t s)
{
    const SellStruct& S = *A.st;
    const int nl = S.nlev();
    for (int li = 0; li < nl; ++li) {
        const int L = fwd ? li : nl - 1 - li;
        const int s0 = S.lev_slice[L], s1 = S.lev_slice[L + 1];
        if (s1 <= s0) continue;
        const int g = grid_for_lanes(static_cast<int64_t>(s1 - s0) * kLanes);
        if (fwd)
            k_sgs_level<B, true><<<g, kThreads, 0, s>>>(S.slice_off.p, S.perm.p, S.rowlen.p, S.col.p, A.val.p,
                                                       s0, s1, b, z, invd);
        else
            k_sgs_level<B, false><<<g, kThreads, 0, s>>>(S.slice_off.p, S.perm.p, S.rowlen.p, S.col.p, A.val.p,
                                                        s0, s1, b, z, invd);
        after_launch("k_sgs_level");
    }
}

} // namespace

void spmv(const Sell& M, const double* x, double* y, const double* b, int mode, cudaStream_t s)
{
    const int RB = M.st->Rb, CB = M.st->Cb;
    if (RB == 1 && CB == 1) return launch_spmv<1, 1>(M, x, y, b, mode, s);
    if (RB == 3 && CB == 3) return launch_spmv<3, 3>(M, x, y, b, mode, s);
    if (RB == 3 && CB == 1) return launch_spmv<3, 1>(M, x, y, b, mode, s);
    if (RB == 1 && CB == 3) return launch_spmv<1, 3>(M, x, y, b, mode, s);
    throw Error(ED_UNSUPPORTED, "spmv: unsupported block shape");
}

void spmv2(const Sell& M1, const double* x1, const Sell& M2, const double* x2, double* y, double sgn,
           cudaStream_t s)
{
    const int RB = M1.st->Rb, C1 = M1.st->Cb, C2 = M2.st->Cb;
    if (M2.st->Rb != RB || M2.st->nslices != M1.st->nslices)
        throw Error(ED_INVALID_ARGUMENT, "spmv2: row layouts differ");
    if (RB == 3 && C1 == 3 && C2 == 1) return launch_spmv2<3, 3, 1>(M1, x1, M2, x2, y, sgn, s);
    if (RB == 1 && C1 == 3 && C2 == 1) return launch_spmv2<1, 3, 1>(M1, x1, M2, x2, y, sgn, s);
    if (RB == 1 && C1 == 1 && C2 == 3) return launch_spmv2<1, 1, 3>(M1, x1, M2, x2, y, sgn, s);
    if (RB == 1 && C1 == 1 && C2 == 1) return launch_spmv2<1, 1, 1>(M1, x1, M2, x2, y, sgn, s);
    throw Error(ED_UNSUPPORTED, "spmv2: unsupported block shape");
}

void sgs_sweep(const Sell& A, const double* b, double* z, const double* invd, bool forward, cudaStream_t s)
{
    const int B = A.st->Rb;
    if (A.st->Cb != B) throw Error(ED_INVALID_ARGUMENT, "sgs: non-square blocks");
    if (B == 1) return launch_sgs<1>(A, b, z, invd, forward, s);
    if (B == 3) return launch_sgs<3>(A, b, z, invd, forward, s);
    throw Error(ED_UNSUPPORTED, "sgs: unsupported block size");
}

void jacobi_update(double* z, const double* b, const double* t, const double* invd, double w, int64_t n,
                   cudaStream_t s)
{
    if (n == 0) return;
    k_jacobi<<<static_cast<int>((n + kThreads - 1) / kThreads), kThreads, 0, s>>>(z, b, t, invd, w, n);
    after_launch("k_jacobi");
}

void sell_scale(Sell& M, const double* wr, const double* wc, cudaStream_t s)
{
    const SellStruct& S = *M.st;
    if (S.nslices == 0) return;
    const int g = grid_for_lanes(static_cast<int64_t>(S.nslices) * kLanes);
#define ED_SCALE(R, C)                                                                                      \
    if (S.Rb == R && S.Cb == C) {                                                                           \
        k_scale<R, C><<<g, kThreads, 0, s>>>(S.slice_off.p, S.perm.p, S.rowlen.p, S.col.p, M.val.p, S.nslices, \
                                             wr, wc);                                                       \
        after_launch("k_scale");                                                                            \
        return;                                                                                             \
    }
    ED_SCALE(1, 1)
    ED_SCALE(3, 3)
    ED_SCALE(3, 1)
    ED_SCALE(1, 3)
#undef ED_SCALE
    throw Error(ED_UNSUPPORTED, "scale: unsupported block shape");
}

void sell_diag(const Sell& M, double* d, cudaStream_t s)
{
    const SellStruct& S = *M.st;
    if (S.Rb != S.Cb) throw Error(ED_INVALID_ARGUMENT, "diag: non-square blocks");
    if (S.nslices == 0) return;
    const int g = grid_for_lanes(static_cast<int64_t>(S.nslices) * kLanes);
    if (S.Rb == 1)
        k_diag<1><<<g, kThreads, 0, s>>>(S.slice_off.p, S.perm.p, S.rowlen.p, S.col.p, M.val.p, S.nslices, d);
    else
        k_diag<3><<<g, kThreads, 0, s>>>(S.slice_off.p, S.perm.p, S.rowlen.p, S.col.p, M.val.p, S.nslices, d);
    after_launch("k_diag");
}

void inv_diag_from(const double* d, double* invd, int64_t n, cudaStream_t s)
{
    if (n == 0) return;
    k_inv_diag<<<static_cast<int>((n + kThreads - 1) / kThreads), kThreads, 0, s>>>(d, invd, n);
    after_launch("k_inv_diag");
}

void dense_gemv(const double* P, const double* r, double* z, int n, cudaStream_t s)
{
    if (n == 0) return;
    const int rows_per_block = kThreads / 32;
    k_dense_gemv<<<(n + rows_per_block - 1) / rows_per_block, kThreads, 0, s>>>(P, r, z, n);
    after_launch("k_dense_gemv");
}

} // namespace edb
