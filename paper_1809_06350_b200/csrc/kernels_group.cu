// Level-group Gauss-Seidel half sweeps (amg.cpp:311-322) for sm_100a.
//
// The in-place sweep is sequential; its exact semantics are kept by level
// scheduling (rows of one dependency level are independent).  Narrow, deep
// schedules (a coarse AMG level: ~36 block rows per level, ~500 levels) are
// bound by the number of dependent steps, so consecutive narrow levels are
// merged into a *group* G whose in-group lower triangle T_G = (D + L)_GG is
// inverted once per hierarchy build:
//
//     forward sweep, rows of G:  T_G z_G = b_G - (A - T_G)_G z      (z: current)
//                                z_G     = T_G^-1 s_G
//
// s_G uses the new values of earlier groups and the old values of everything
// at or after G exactly as the sequential sweep does, and T_G^-1 s_G equals
// the sequential substitution inside the group up to roundoff.  A half sweep
// is ONE persistent kernel whose CTAs cross a grid barrier between the two
// phases of a group step (phase A: the sparse sums s_G; phase B: the dense
// triangular GEMV z_G = T_G^-1 s_G), so the dependency chain is the number of
// groups, not the number of levels.  Wide levels form single-level groups
// whose rows are updated in place in phase A (in-block scalar order as the
// reference) with one barrier per level.
//
// T_G^-1 (lower triangular in the group's processing order, packed by rows)
// is built by k_group_tinv: one warp per (group, 32 columns) runs the forward
// substitution T x = e_j for its 32 columns at once.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>

#include "ed_internal.hpp"

namespace edb {

namespace {

constexpr int kGT = 256; // threads per CTA of the sweep kernel

struct GrpArgs {
    const int* rowptr;
    const int* col;
    const int* perm; // stored -> original (null: identity)
    const int* inv;  // original -> stored (null: identity)
    const int* dpos;
    const double* val;
    const int4* grp;              // {r0, r1, m (0: single level), pad}
    const long long* toff;        // packed T^-1 offset of each group (doubles)
    const unsigned char* bcode;   // per block: 0 other group, 1 in-group lower, 2 in-group upper, 3 diagonal
    const int* gptr;              // [nbr+1] in-group blocks of each stored row (multi-level groups)
    const int* gblk;
    int ngrp;
};

__device__ __forceinline__ unsigned int g_ld_acquire(const unsigned int* p)
{
    unsigned int v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ void g_red_release(unsigned int* p, unsigned int v)
{
    asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// all CTAs of the (co-resident) grid; `target` counts arrivals so far
__device__ __forceinline__ void grid_barrier(unsigned int* ctr, unsigned int& target)
{
    __syncthreads();
    target += gridDim.x;
    if (threadIdx.x == 0) {
        g_red_release(ctr, 1u);
        while (g_ld_acquire(ctr) < target) {
        }
    }
    __syncthreads();
}

template <int L>
__device__ __forceinline__ double lane_sum(double v)
{
#pragma unroll
    for (int o = L / 2; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o, L);
    return v;
}

// local index (processing order) of scalar (stored row sr, component c) in group [r0, r1)
template <int B, bool FWD>
__device__ __forceinline__ int local_of(int sr, int c, int r0, int r1)
{
    return FWD ? (sr - r0) * B + c : (r1 - 1 - sr) * B + (B - 1 - c);
}

// Single-level group: the whole Gauss-Seidel update of stored row sr (lanes
// of a group of L split its blocks; current z everywhere; the leader solves
// the diagonal block in sweep order).
template <int B, int L, bool FWD>
__device__ __forceinline__ void row_update(const GrpArgs& a, const double* __restrict__ bvec,
                                           const double* __restrict__ invd, double* z, int sr, int lane)
{
    const int row = a.perm ? a.perm[sr] : sr;
    const int kb = a.rowptr[sr], ke = a.rowptr[sr + 1];
    double acc[B];
#pragma unroll
    for (int r = 0; r < B; ++r) acc[r] = 0.0;
    for (int k = kb + lane; k < ke; k += L) {
        const int c = __ldg(a.col + k);
        if (c == row) continue;
        const double* vp = a.val + static_cast<int64_t>(k) * (B * B);
        double zv[B];
#pragma unroll
        for (int d = 0; d < B; ++d) zv[d] = __ldcg(z + static_cast<int64_t>(c) * B + d);
#pragma unroll
        for (int d = 0; d < B; ++d)
#pragma unroll
            for (int r = 0; r < B; ++r) acc[r] = fma(__ldg(vp + r * B + d), zv[d], acc[r]);
    }
#pragma unroll
    for (int r = 0; r < B; ++r) acc[r] = lane_sum<L>(acc[r]);
    if (lane == 0) {
        const int dp = a.dpos[sr];
        double zs[B], D[B * B];
#pragma unroll
        for (int d = 0; d < B; ++d) zs[d] = __ldcg(z + static_cast<int64_t>(row) * B + d);
#pragma unroll
        for (int e = 0; e < B * B; ++e) D[e] = dp >= 0 ? __ldg(a.val + static_cast<int64_t>(dp) * (B * B) + e) : 0.0;
#pragma unroll
        for (int ci = 0; ci < B; ++ci) {
            const int c = FWD ? ci : B - 1 - ci;
            const int64_t i = static_cast<int64_t>(row) * B + c;
            double v = __ldg(bvec + i) - acc[c];
#pragma unroll
            for (int d = 0; d < B; ++d)
                if (d != c) v -= D[c * B + d] * zs[d];
            zs[c] = v * __ldg(invd + i);
        }
#pragma unroll
        for (int d = 0; d < B; ++d) z[static_cast<int64_t>(row) * B + d] = zs[d];
    }
}

// Multi-level group, phase A: s_i = b_i - sum of the row's entries that are
// not in T_G (every block of another group; in-group blocks on the far side
// of the sweep; the diagonal block's entries after i in sweep order), all
// with the current z.
template <int B, int L, bool FWD>
__device__ __forceinline__ void row_rhs(const GrpArgs& a, const double* __restrict__ bvec, const double* z,
                                        double* sbuf, int sr, int r0, int r1, int lane)
{
    const int row = a.perm ? a.perm[sr] : sr;
    const int kb = a.rowptr[sr], ke = a.rowptr[sr + 1];
    double acc[B];
#pragma unroll
    for (int r = 0; r < B; ++r) acc[r] = 0.0;
    for (int k = kb + lane; k < ke; k += L) {
        const int code = a.bcode[k];
        const int c = __ldg(a.col + k);
        const double* vp = a.val + static_cast<int64_t>(k) * (B * B);
        double zv[B];
#pragma unroll
        for (int d = 0; d < B; ++d) zv[d] = __ldcg(z + static_cast<int64_t>(c) * B + d);
        if (code == 3) {
#pragma unroll
            for (int r = 0; r < B; ++r)
#pragma unroll
                for (int d = 0; d < B; ++d)
                    if (FWD ? d > r : d < r) acc[r] = fma(__ldg(vp + r * B + d), zv[d], acc[r]);
        } else if (code == 0 || code == (FWD ? 2 : 1)) {
#pragma unroll
            for (int d = 0; d < B; ++d)
#pragma unroll
                for (int r = 0; r < B; ++r) acc[r] = fma(__ldg(vp + r * B + d), zv[d], acc[r]);
        }
    }
#pragma unroll
    for (int r = 0; r < B; ++r) acc[r] = lane_sum<L>(acc[r]);
    if (lane == 0) {
#pragma unroll
        for (int c = 0; c < B; ++c)
            sbuf[local_of<B, FWD>(sr, c, r0, r1)] = __ldg(bvec + static_cast<int64_t>(row) * B + c) - acc[c];
    }
}

// One half sweep: persistent grid, groups in sweep order.
template <int B, int L, bool FWD>
__global__ void __launch_bounds__(kGT) k_group_sweep(GrpArgs a, const double* __restrict__ bvec, double* z,
                                                     const double* __restrict__ invd, const double* __restrict__ X,
                                                     double* sbuf, unsigned int* bar)
{
    constexpr int GPC = kGT / L; // lane groups per CTA
    const int lg = threadIdx.x / L, lane = threadIdx.x % L;
    const int warp = threadIdx.x / 32, wl = threadIdx.x % 32;
    unsigned int target = 0;
    for (int t = 0; t < a.ngrp; ++t) {
        const int g = FWD ? t : a.ngrp - 1 - t;
        const int4 gi = a.grp[g];
        const int r0 = gi.x, r1 = gi.y, m = gi.z;
        const int nr = r1 - r0;
        // rows dealt round-robin over CTAs first (a level's rows spread over the whole GPU)
        if (m == 0) {
            for (int q = blockIdx.x + lg * gridDim.x; q < nr; q += GPC * gridDim.x) {
                const int sr = FWD ? r0 + q : r1 - 1 - q;
                row_update<B, L, FWD>(a, bvec, invd, z, sr, lane);
            }
            grid_barrier(bar, target);
            continue;
        }
        for (int q = blockIdx.x + lg * gridDim.x; q < nr; q += GPC * gridDim.x)
            row_rhs<B, L, FWD>(a, bvec, z, sbuf, r0 + q, r0, r1, lane);
        grid_barrier(bar, target);
        // phase B: z_G = T^-1 s_G, one warp per scalar row of the group
        const double* Xg = X + a.toff[g];
        for (int i = blockIdx.x + warp * gridDim.x; i < m; i += (kGT / 32) * gridDim.x) {
            const double* xr = Xg + static_cast<int64_t>(i) * (i + 1) / 2;
            double acc = 0.0;
#pragma unroll 4
            for (int j = wl; j <= i; j += 32) acc = fma(__ldg(xr + j), __ldcg(sbuf + j), acc);
            acc = lane_sum<32>(acc);
            if (wl == 0) {
                const int p = i / B, c = i % B;
                const int sr = FWD ? r0 + p : r1 - 1 - p;
                const int cc = FWD ? c : B - 1 - c;
                const int row = a.perm ? a.perm[sr] : sr;
                z[static_cast<int64_t>(row) * B + cc] = acc;
            }
        }
        grid_barrier(bar, target);
    }
}

// T_G^-1 for both directions: one warp per (group, 32 columns [j0, j0+32)),
// forward substitution over the group's scalar rows in processing order:
//   x_i = invd_i * (e_ij - sum_{k before i in G} a_ik x_k)
template <int B, bool FWD>
__global__ void __launch_bounds__(128) k_group_tinv(GrpArgs a, const double* __restrict__ invd,
                                                     const int2* __restrict__ chunks, int nchunks, double* X)
{
    const int w = (blockIdx.x * blockDim.x + threadIdx.x) / 32;
    const int lane = threadIdx.x % 32;
    if (w >= nchunks) return;
    const int g = chunks[w].x, j0 = chunks[w].y;
    const int4 gi = a.grp[g];
    const int r0 = gi.x, r1 = gi.y, m = gi.z;
    double* Xg = X + a.toff[g];
    const int j = j0 + lane;
    for (int i = j0; i < m; ++i) {
        const int p = i / B, cl = i % B;
        const int sr = FWD ? r0 + p : r1 - 1 - p;
        const int cr = FWD ? cl : B - 1 - cl;
        const int row = a.perm ? a.perm[sr] : sr;
        double acc = (i == j) ? 1.0 : 0.0;
        for (int q = a.gptr[sr]; q < a.gptr[sr + 1]; ++q) {
            const int k = a.gblk[q];
            const int code = a.bcode[k];
            const int c = a.col[k];
            const int sc = a.inv ? a.inv[c] : c;
            const double* vp = a.val + static_cast<int64_t>(k) * (B * B) + cr * B;
            if (code == 3) {
#pragma unroll
                for (int d = 0; d < B; ++d) {
                    if (!(FWD ? d < cr : d > cr)) continue;
                    const int kl = local_of<B, FWD>(sr, d, r0, r1);
                    if (j <= kl) acc -= vp[d] * Xg[static_cast<int64_t>(kl) * (kl + 1) / 2 + j];
                }
            } else if (code == (FWD ? 1 : 2)) {
#pragma unroll
                for (int d = 0; d < B; ++d) {
                    const int kl = local_of<B, FWD>(sc, d, r0, r1);
                    if (j <= kl) acc -= vp[d] * Xg[static_cast<int64_t>(kl) * (kl + 1) / 2 + j];
                }
            }
        }
        if (j <= i) Xg[static_cast<int64_t>(i) * (i + 1) / 2 + j] = acc * invd[static_cast<int64_t>(row) * B + cr];
    }
}

GrpArgs gargs_of(const Bsr& A)
{
    const BsrStruct& S = *A.st;
    return GrpArgs{S.rowptr.p, S.col.p,      S.perm.p,     S.inv.p,    S.dpos.p, A.val.p,
                   S.grp.p,    S.grp_toff.p, S.bcode.p,    S.gptr.p,   S.gblk.p, S.ngrp};
}

int sweep_grid()
{
    // co-resident CTAs of the persistent sweep (the grid barrier needs all of
    // them resident), per device
    static int grid[64] = {};
    int dev = 0;
    ED_CUDA(cudaGetDevice(&dev));
    int& g = grid[dev & 63];
    if (!g) {
        int sms = 0, occ = 0;
        ED_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
        ED_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_group_sweep<3, 32, true>, kGT, 0));
        static const int per_sm = std::getenv("ED_SWEEP_CTAS") ? std::atoi(std::getenv("ED_SWEEP_CTAS")) : 1;
        g = sms * std::max(1, std::min(occ, per_sm));
    }
    return g;
}

#define ED_GLANES(L, ...)                                     \
    switch (L) {                                              \
    case 2: { constexpr int LL = 2; __VA_ARGS__; break; }   \
    case 4: { constexpr int LL = 4; __VA_ARGS__; break; }   \
    case 8: { constexpr int LL = 8; __VA_ARGS__; break; }   \
    case 16: { constexpr int LL = 16; __VA_ARGS__; break; } \
    default: { constexpr int LL = 32; __VA_ARGS__; break; } \
    }

template <int B>
void launch_group(const Bsr& A, const double* b, double* z, const double* invd, bool fwd, cudaStream_t s,
                  const double* X)
{
    const BsrStruct& S = *A.st;
    const GrpArgs a = gargs_of(A);
    ED_CUDA(cudaMemsetAsync(S.gbar.p, 0, sizeof(unsigned int), s));
    const int grid = sweep_grid();
    const double* Xd = X ? X + (fwd ? 0 : S.grp_tinv) : nullptr;
    ED_GLANES(S.Ls, {
        if (fwd)
            k_group_sweep<B, LL, true><<<grid, kGT, 0, s>>>(a, b, z, invd, Xd, S.gsbuf.p, S.gbar.p);
        else
            k_group_sweep<B, LL, false><<<grid, kGT, 0, s>>>(a, b, z, invd, Xd, S.gsbuf.p, S.gbar.p);
    })
    after_launch("k_group_sweep");
}

} // namespace

void group_prepare(const Bsr& A, const double* invd, DevArray<double>& X, cudaStream_t s)
{
    const BsrStruct& S = *A.st;
    if (S.grp_tinv == 0) {
        X.release();
        return;
    }
    X.alloc(2 * static_cast<size_t>(S.grp_tinv));
    const GrpArgs a = gargs_of(A);
    const int blocks = (S.ntchunk * 32 + 127) / 128;
    if (S.Rb == 3) {
        k_group_tinv<3, true><<<blocks, 128, 0, s>>>(a, invd, S.tchunk.p, S.ntchunk, X.p);
        k_group_tinv<3, false><<<blocks, 128, 0, s>>>(a, invd, S.tchunk.p, S.ntchunk, X.p + S.grp_tinv);
    } else {
        k_group_tinv<1, true><<<blocks, 128, 0, s>>>(a, invd, S.tchunk.p, S.ntchunk, X.p);
        k_group_tinv<1, false><<<blocks, 128, 0, s>>>(a, invd, S.tchunk.p, S.ntchunk, X.p + S.grp_tinv);
    }
    after_launch("k_group_tinv");
}

void sgs_group(const Bsr& A, const double* b, double* z, const double* invd, bool fwd, cudaStream_t s,
               const double* X)
{
    if (A.st->grp_tinv > 0 && !X) throw Error(ED_INVALID_ARGUMENT, "group sweep needs the operator's T^-1 (group_prepare)");
    if (A.st->Rb == 3) return launch_group<3>(A, b, z, invd, fwd, s, X);
    if (A.st->Rb == 1) return launch_group<1>(A, b, z, invd, fwd, s, X);
    throw Error(ED_UNSUPPORTED, "group sweep: unsupported block size");
}

} // namespace edb
