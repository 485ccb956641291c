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
// is built by k_group_tinv: one CTA per (group, 32 columns) runs the forward
// substitution T x = e_j for its 32 columns at once.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>

#include "ed_internal.hpp"

namespace edb {

namespace {

constexpr int kGT = 256; // threads per CTA of the sweep kernel
constexpr int kGroupMaxRows = 1024;

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

// Grid barrier over all (co-resident) CTAs, split in two so that loads of the
// next step's z-independent data can be issued between arrive and wait (a
// release would otherwise wait for them).  `target` counts arrivals so far.
__device__ __forceinline__ void bar_arrive(unsigned int* ctr)
{
    __syncthreads();
    if (threadIdx.x == 0) g_red_release(ctr, 1u);
}

__device__ __forceinline__ void bar_wait(unsigned int* ctr, unsigned int& target)
{
    target += gridDim.x;
    if (threadIdx.x == 0) {
        // bounded spin: a grid whose CTAs are not all resident would wait
        // forever; trap after ~10 s instead of hanging the device
        const long long t0 = clock64();
        while (g_ld_acquire(ctr) < target) {
            if (clock64() - t0 > 20000000000LL) __trap();
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

// Row sums over a whole CTA (L = kGT lanes per row: dense-row coarse levels with hundreds of blocks
// per row): warp shuffles, then the eight warp partials through shared memory, summed by thread 0
// in warp order.  All threads of the CTA call it.
template <int B>
__device__ __forceinline__ void cta_sum(double (&acc)[B])
{
    __shared__ double red[kGT / 32][B];
#pragma unroll
    for (int r = 0; r < B; ++r) acc[r] = lane_sum<32>(acc[r]);
    if ((threadIdx.x & 31) == 0) {
#pragma unroll
        for (int r = 0; r < B; ++r) red[threadIdx.x / 32][r] = acc[r];
    }
    __syncthreads();
    if (threadIdx.x == 0) {
#pragma unroll
        for (int r = 0; r < B; ++r) {
            double t = red[0][r];
#pragma unroll
            for (int w = 1; w < kGT / 32; ++w) t += red[w][r];
            acc[r] = t;
        }
    }
    __syncthreads();
}

// local index (processing order) of scalar (stored row sr, component c) in group [r0, r1)
template <int B, bool FWD>
__device__ __forceinline__ int local_of(int sr, int c, int r0, int r1)
{
    return FWD ? (sr - r0) * B + c : (r1 - 1 - sr) * B + (B - 1 - c);
}

// Everything of one row a lane needs that does not depend on z: its first PF
// blocks (column, in-group code, values) and, for the group leader, b, inv_diag
// and the diagonal block.  Loaded for the NEXT group before the grid barrier,
// so after the barrier only the z gathers sit on the critical path.
template <int B, int PF>
struct GRow {
    int row, kb, ke;
    bool valid;
    int c[PF];
    int code[PF];
    double v[PF][B * B];
    double b[B], id[B], D[B * B], zs[B];
};

template <int B, int L, int PF>
__device__ __forceinline__ void grow_load(const GrpArgs& a, const double* __restrict__ bvec,
                                          const double* __restrict__ invd, const double* z, int sr, bool valid,
                                          int lane, GRow<B, PF>& P)
{
    P.valid = valid;
    P.row = valid ? (a.perm ? a.perm[sr] : sr) : 0;
    P.kb = valid ? a.rowptr[sr] + lane : 0;
    P.ke = valid ? a.rowptr[sr + 1] : 0;
#pragma unroll
    for (int q = 0; q < PF; ++q) {
        const int k = P.kb + q * L;
        const bool in = k < P.ke;
        P.c[q] = in ? __ldg(a.col + k) : -1;
        P.code[q] = in ? a.bcode[k] : -1;
#pragma unroll
        for (int e = 0; e < B * B; ++e) P.v[q][e] = in ? __ldg(a.val + static_cast<int64_t>(k) * (B * B) + e) : 0.0;
    }
    if (valid && lane == 0) {
        const int dp = a.dpos[sr];
#pragma unroll
        for (int d = 0; d < B; ++d) {
            const int64_t i = static_cast<int64_t>(P.row) * B + d;
            P.b[d] = __ldg(bvec + i);
            P.id[d] = __ldg(invd + i);
            P.zs[d] = __ldcg(z + i); // only this row writes z[row] during the sweep
        }
#pragma unroll
        for (int e = 0; e < B * B; ++e) P.D[e] = dp >= 0 ? __ldg(a.val + static_cast<int64_t>(dp) * (B * B) + e) : 0.0;
    }
}

// does the block's scalar (r, d) enter the sum (everything not in T_G)?
template <bool FWD, bool MULTI>
__device__ __forceinline__ bool takes(int code, int r, int d)
{
    if (!MULTI) return code != 3;                         // single level: all off-diagonal blocks
    if (code == 3) return FWD ? d > r : d < r;             // diagonal block: the far side of the sweep
    return code == 0 || code == (FWD ? 2 : 1);             // other groups; in-group blocks not yet swept
}

// Row sums over the z-dependent part.  MULTI = false: the full Gauss-Seidel
// update of the row (single-level group; the leader solves the diagonal block
// in sweep order and writes z).  MULTI = true: s_i = b_i - (A - T_G)_i z into
// the group's local buffer (phase A).
template <int B, int L, int PF, bool FWD, bool MULTI>
__device__ __forceinline__ void grow_finish(const GrpArgs& a, double* z, double* sbuf, int sr, int r0, int r1,
                                            int lane, const GRow<B, PF>& P)
{
    double acc[B];
#pragma unroll
    for (int r = 0; r < B; ++r) acc[r] = 0.0;
    double zv[PF][B];
#pragma unroll
    for (int q = 0; q < PF; ++q) {
        const int64_t cc = P.c[q] >= 0 ? P.c[q] : 0;
#pragma unroll
        for (int d = 0; d < B; ++d) zv[q][d] = __ldcg(z + cc * B + d);
    }
#pragma unroll
    for (int q = 0; q < PF; ++q) {
        if (P.c[q] < 0) continue;
#pragma unroll
        for (int d = 0; d < B; ++d)
#pragma unroll
            for (int r = 0; r < B; ++r)
                if (takes<FWD, MULTI>(P.code[q], r, d)) acc[r] = fma(P.v[q][r * B + d], zv[q][d], acc[r]);
    }
    // long rows (dense-row coarse levels: hundreds of blocks per lane): the
    // rest in batches of NB blocks per lane, all of a batch's loads in flight
    constexpr int NB = B == 3 ? 4 : 8;
    for (int k0 = P.kb + PF * L; k0 < P.ke; k0 += NB * L) {
        int cb[NB], codeb[NB];
        double vb[NB][B * B], zb[NB][B];
#pragma unroll
        for (int p = 0; p < NB; ++p) {
            const int k = k0 + p * L;
            const bool in = k < P.ke;
            cb[p] = in ? __ldg(a.col + k) : 0;
            codeb[p] = in ? a.bcode[k] : -1;
#pragma unroll
            for (int e = 0; e < B * B; ++e) vb[p][e] = in ? __ldg(a.val + static_cast<int64_t>(k) * (B * B) + e) : 0.0;
        }
#pragma unroll
        for (int p = 0; p < NB; ++p)
#pragma unroll
            for (int d = 0; d < B; ++d) zb[p][d] = __ldcg(z + static_cast<int64_t>(cb[p]) * B + d);
#pragma unroll
        for (int p = 0; p < NB; ++p)
#pragma unroll
            for (int d = 0; d < B; ++d)
#pragma unroll
                for (int r = 0; r < B; ++r)
                    if (codeb[p] >= 0 && takes<FWD, MULTI>(codeb[p], r, d)) acc[r] = fma(vb[p][r * B + d], zb[p][d], acc[r]);
    }
#pragma unroll
    if (L > 32) {
        cta_sum<B>(acc);
    } else {
#pragma unroll
        for (int r = 0; r < B; ++r) acc[r] = lane_sum<(L > 32 ? 32 : L)>(acc[r]);
    }
    if (!P.valid || lane != 0) return;
    if (MULTI) {
#pragma unroll
        for (int c = 0; c < B; ++c) sbuf[local_of<B, FWD>(sr, c, r0, r1)] = P.b[c] - acc[c];
        return;
    }
    double zs[B];
#pragma unroll
    for (int d = 0; d < B; ++d) zs[d] = P.zs[d];
#pragma unroll
    for (int ci = 0; ci < B; ++ci) {
        const int c = FWD ? ci : B - 1 - ci;
        double v = P.b[c] - acc[c];
#pragma unroll
        for (int d = 0; d < B; ++d)
            if (d != c) v -= P.D[c * B + d] * zs[d];
        zs[c] = v * P.id[c];
    }
#pragma unroll
    for (int d = 0; d < B; ++d) z[static_cast<int64_t>(P.row) * B + d] = zs[d];
}

// One half sweep: persistent grid, groups in sweep order.  Rows of a group are
// dealt round-robin over the CTAs first (lane group lg of CTA b takes row
// b + lg * grid), so a level's rows spread over the whole GPU; trip counts
// are CTA-uniform, so every lane reaches the shuffles.
template <int B, int L, bool FWD>
__global__ void __launch_bounds__(kGT, 1) k_group_sweep(GrpArgs a, const double* __restrict__ bvec, double* z,
                                                     const double* __restrict__ invd, const double* __restrict__ X,
                                                     double* sbuf, unsigned int* bar)
{
    constexpr int PF = B == 3 ? 3 : 4;  // blocks per lane prefetched ahead of the barrier
    constexpr int XQ = kGroupMaxRows / 32; // T^-1 row entries per lane prefetched ahead of phase B
    constexpr int GPC = kGT / L;         // lane groups per CTA
    const int lg = threadIdx.x / L, lane = threadIdx.x % L;
    const int warp = threadIdx.x / 32, wl = threadIdx.x % 32;
    const int stride = GPC * gridDim.x;
    unsigned int target = 0;
    GRow<B, PF> P;
    auto sr_of = [&](int r0, int r1, int q) { return FWD ? r0 + q : r1 - 1 - q; };
    {
        const int4 gi = a.grp[FWD ? 0 : a.ngrp - 1];
        const int q = blockIdx.x + lg * gridDim.x;
        grow_load<B, L, PF>(a, bvec, invd, z, sr_of(gi.x, gi.y, q), q < gi.y - gi.x, lane, P);
    }
    for (int t = 0; t < a.ngrp; ++t) {
        const int g = FWD ? t : a.ngrp - 1 - t;
        const int4 gi = a.grp[g];
        const int r0 = gi.x, r1 = gi.y, m = gi.z;
        const int nr = r1 - r0;
        if (m == 0) {
            for (int q0 = 0; q0 < nr; q0 += stride) {
                const int q = q0 + blockIdx.x + lg * gridDim.x;
                if (q0 > 0) grow_load<B, L, PF>(a, bvec, invd, z, sr_of(r0, r1, q), q < nr, lane, P);
                grow_finish<B, L, PF, FWD, false>(a, z, sbuf, sr_of(r0, r1, q), r0, r1, lane, P);
            }
        } else {
            for (int q0 = 0; q0 < nr; q0 += stride) {
                const int q = q0 + blockIdx.x + lg * gridDim.x;
                if (q0 > 0) grow_load<B, L, PF>(a, bvec, invd, z, sr_of(r0, r1, q), q < nr, lane, P);
                grow_finish<B, L, PF, FWD, true>(a, z, sbuf, sr_of(r0, r1, q), r0, r1, lane, P);
            }
            bar_arrive(bar);
            // this warp's first phase-B row of T^-1 into registers during the barrier
            const double* Xg = X + a.toff[g];
            const int i0 = blockIdx.x + warp * gridDim.x;
            double xv[XQ];
            const double* xr0 = Xg + static_cast<int64_t>(i0) * (i0 + 1) / 2;
#pragma unroll
            for (int q = 0; q < XQ; ++q) {
                const int j = wl + 32 * q;
                xv[q] = (i0 < m && j <= i0) ? __ldg(xr0 + j) : 0.0;
            }
            bar_wait(bar, target);
            // phase B: z_G = T^-1 s_G, one warp per scalar row of the group
            for (int i = i0; i < m; i += (kGT / 32) * gridDim.x) {
                const double* xr = Xg + static_cast<int64_t>(i) * (i + 1) / 2;
                double acc = 0.0;
                if (i == i0) {
#pragma unroll
                    for (int q = 0; q < XQ; ++q) {
                        const int j = wl + 32 * q;
                        if (j <= i) acc = fma(xv[q], __ldcg(sbuf + j), acc);
                    }
                    for (int j = wl + 32 * XQ; j <= i; j += 32) acc = fma(__ldg(xr + j), __ldcg(sbuf + j), acc);
                } else {
#pragma unroll 4
                    for (int j = wl; j <= i; j += 32) acc = fma(__ldg(xr + j), __ldcg(sbuf + j), acc);
                }
                acc = lane_sum<32>(acc);
                if (wl == 0) {
                    const int p = i / B, c = i % B;
                    const int sr = sr_of(r0, r1, p);
                    const int cc = FWD ? c : B - 1 - c;
                    const int row = a.perm ? a.perm[sr] : sr;
                    z[static_cast<int64_t>(row) * B + cc] = acc;
                }
            }
        }
        bar_arrive(bar);
        // the next group's rows: everything z-independent, during the barrier
        if (t + 1 < a.ngrp) {
            const int4 gn = a.grp[FWD ? t + 1 : a.ngrp - 2 - t];
            const int q = blockIdx.x + lg * gridDim.x;
            grow_load<B, L, PF>(a, bvec, invd, z, sr_of(gn.x, gn.y, q), q < gn.y - gn.x, lane, P);
        }
        bar_wait(bar, target);
    }
}

// T_G^-1 for both directions: forward substitution over the group's scalar rows in processing order,
//   x_i = invd_i * (e_ij - sum_{k before i in G} a_ik x_k),
// for 32 columns [j0, j0+32) per warp (lane = column).  One scalar row step:
template <int B, bool FWD>
__device__ __forceinline__ void tinv_row(const GrpArgs& a, const double* __restrict__ invd, double* Xg, int r0, int r1,
                                         int i, int j, int lane)
{
    const int p = i / B, cl = i % B;
    const int sr = FWD ? r0 + p : r1 - 1 - p;
    const int cr = FWD ? cl : B - 1 - cl;
    const int row = a.perm ? a.perm[sr] : sr;
    double acc = (i == j) ? 1.0 : 0.0;
    // The row's in-group blocks: the index chain (block -> code, column -> stored row) is
    // resolved for 32 blocks at once, one per lane, then the blocks are applied in order
    // (the same subtraction order as a lane-serial loop) with their operands broadcast.
    const int q0 = a.gptr[sr], q1 = a.gptr[sr + 1];
    for (int qb = q0; qb < q1; qb += 32) {
        int mk = 0, mcode = 0, msc = 0;
        if (qb + lane < q1) {
            mk = a.gblk[qb + lane];
            mcode = a.bcode[mk];
            const int c = a.col[mk];
            msc = a.inv ? a.inv[c] : c;
        }
        const int nb = min(32, q1 - qb);
        for (int e = 0; e < nb; ++e) {
            const int k = __shfl_sync(0xffffffffu, mk, e);
            const int code = __shfl_sync(0xffffffffu, mcode, e);
            const int sc = __shfl_sync(0xffffffffu, msc, e);
            const double* vp = a.val + static_cast<int64_t>(k) * (B * B) + cr * B;
            if (code == 3) {
#pragma unroll
                for (int d = 0; d < B; ++d) {
                    if (!(FWD ? d < cr : d > cr)) continue;
                    const int kl = local_of<B, FWD>(sr, d, r0, r1);
                    if (j <= kl) acc -= vp[d] * Xg[static_cast<int64_t>(kl) * (kl + 1) / 2 + j];
                }
            } else if (code == (FWD ? 1 : 2)) {
                double xs[B];
#pragma unroll
                for (int d = 0; d < B; ++d) {
                    const int kl = local_of<B, FWD>(sc, d, r0, r1);
                    xs[d] = j <= kl ? Xg[static_cast<int64_t>(kl) * (kl + 1) / 2 + j] : 0.0;
                }
#pragma unroll
                for (int d = 0; d < B; ++d) {
                    const int kl = local_of<B, FWD>(sc, d, r0, r1);
                    if (j <= kl) acc -= vp[d] * xs[d];
                }
            }
        }
    }
    if (j <= i) Xg[static_cast<int64_t>(i) * (i + 1) / 2 + j] = acc * invd[static_cast<int64_t>(row) * B + cr];
}

// One CTA of kTinvWarps warps per (group, 32 columns): the block rows of one dependency level are
// independent (their in-group couplings reach earlier levels only), so the warps split them and
// meet at a CTA barrier per level -- the sequential depth is the group's levels (~9) times B, not
// its scalar rows (~1000).  The B scalar rows of a block row stay with one warp, in sweep order.
constexpr int kTinvWarps = 8;

template <int B, bool FWD>
__global__ void __launch_bounds__(32 * kTinvWarps) k_group_tinv(GrpArgs a, const double* __restrict__ invd,
                                                                const int2* __restrict__ chunks,
                                                                const int* __restrict__ lev_ptr, int nlev, double* X)
{
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const int g = chunks[blockIdx.x].x, j0 = chunks[blockIdx.x].y;
    const int4 gi = a.grp[g];
    const int r0 = gi.x, r1 = gi.y;
    double* Xg = X + a.toff[g];
    const int j = j0 + lane;
    // the level that holds stored row r0 (levels are contiguous stored-row ranges; groups are whole levels)
    int lo = 0, hi = nlev;
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (lev_ptr[mid] <= r0) lo = mid;
        else hi = mid - 1;
    }
    int l_first = lo, l_last = lo;
    while (l_last + 1 < nlev && lev_ptr[l_last + 1] < r1) ++l_last;
    const int pmin = j0 / B; // block rows (processing order) before it only hold columns left of j0: nothing to do
    for (int li = 0; li <= l_last - l_first; ++li) {
        const int l = FWD ? l_first + li : l_last - li;
        const int a0 = lev_ptr[l], a1 = lev_ptr[l + 1]; // stored rows of the level
        // processing-order positions of the level's block rows
        const int p0 = FWD ? a0 - r0 : r1 - a1, p1 = FWD ? a1 - r0 : r1 - a0;
        for (int pp = max(p0, pmin) + warp; pp < p1; pp += kTinvWarps)
#pragma unroll 1
            for (int cl = 0; cl < B; ++cl) tinv_row<B, FWD>(a, invd, Xg, r0, r1, pp * B + cl, j, lane);
        __syncthreads();
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
        // ED_SWEEP_GRID=n: fewer CTAs (cheaper barrier, less bandwidth)
        if (std::getenv("ED_SWEEP_GRID")) g = std::min(g, std::max(1, std::atoi(std::getenv("ED_SWEEP_GRID"))));
    }
    return g;
}

#define ED_GLANES(L, ...)                                     \
    switch (L) {                                              \
    case 2: { constexpr int LL = 2; __VA_ARGS__; break; }   \
    case 4: { constexpr int LL = 4; __VA_ARGS__; break; }   \
    case 8: { constexpr int LL = 8; __VA_ARGS__; break; }   \
    case 16: { constexpr int LL = 16; __VA_ARGS__; break; } \
    case 256: { constexpr int LL = 256; __VA_ARGS__; break; } \
    default: { constexpr int LL = 32; __VA_ARGS__; break; } \
    }

template <int B>
void launch_group(const Bsr& A, const double* b, double* z, const double* invd, bool fwd, cudaStream_t s,
                  const double* X)
{
    const BsrStruct& S = *A.st;
    const GrpArgs a = gargs_of(A);
    ED_CUDA(cudaMemsetAsync(S.gbar.p, 0, sizeof(unsigned int), s));
    const double* Xd = X ? X + (fwd ? 0 : S.grp_tinv) : nullptr;
    ED_GLANES(S.Ls, {
        if (fwd)
            k_group_sweep<B, LL, true><<<sweep_grid(), kGT, 0, s>>>(a, b, z, invd, Xd, S.gsbuf.p, S.gbar.p);
        else
            k_group_sweep<B, LL, false><<<sweep_grid(), kGT, 0, s>>>(a, b, z, invd, Xd, S.gsbuf.p, S.gbar.p);
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
    const int nlev = S.nlev();
    if (S.Rb == 3) {
        k_group_tinv<3, true><<<S.ntchunk, 32 * kTinvWarps, 0, s>>>(a, invd, S.tchunk.p, S.d_lev_ptr.p, nlev, X.p);
        k_group_tinv<3, false><<<S.ntchunk, 32 * kTinvWarps, 0, s>>>(a, invd, S.tchunk.p, S.d_lev_ptr.p, nlev,
                                                                     X.p + S.grp_tinv);
    } else {
        k_group_tinv<1, true><<<S.ntchunk, 32 * kTinvWarps, 0, s>>>(a, invd, S.tchunk.p, S.d_lev_ptr.p, nlev, X.p);
        k_group_tinv<1, false><<<S.ntchunk, 32 * kTinvWarps, 0, s>>>(a, invd, S.tchunk.p, S.d_lev_ptr.p, nlev,
                                                                     X.p + S.grp_tinv);
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
