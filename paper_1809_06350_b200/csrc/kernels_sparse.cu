// Block-sparse kernels for sm_100a (FP64 CUDA cores; HBM/L2-latency bound).
//
// Every block row is owned by a group of L lanes (L = 2..32, sized to the
// row length) that split the row's blocks round-robin -- consecutive lanes
// read consecutive 72-B blocks, so a group's loads coalesce -- and combine
// their partial sums with warp shuffles.  Gauss-Seidel keeps the reference's
// exact sequential semantics (amg.cpp:311-322): rows are level-scheduled (a
// row only reads new values of rows on earlier levels), and inside a 3x3
// diagonal block the three scalar rows are solved in sweep order by the
// group leader.  A whole half sweep is ONE persistent dataflow kernel
// (k_sgs_tag): warps take work items in level order from a ticket counter,
// prefetch their rows' matrix data, and wait only on the tagged values of the
// neighbours that precede each row, so there is no launch, no grid-wide
// barrier and no level counter per dependency level.
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <string>
#include <vector>

#include "ed_internal.hpp"

namespace edb {

namespace cg = cooperative_groups;

namespace {

constexpr int kThreads = 256;

struct BsrArgs {
    const int* rowptr;
    const int* col;
    const int* perm; // null: identity
    const int* dpos;
    const double* val;
    int nbr;
};

inline BsrArgs args_of(const Bsr& M)
{
    const BsrStruct& S = *M.st;
    return BsrArgs{S.rowptr.p, S.col.p, S.perm.p, S.dpos.p, M.val.p, S.nbr};
}

template <int L>
__device__ __forceinline__ double group_sum(double v)
{
#pragma unroll
    for (int o = L / 2; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o, L);
    return v;
}

template <int RB, int CB, int L, int MODE>
__global__ void __launch_bounds__(kThreads) k_spmv(BsrArgs m, const double* __restrict__ x, double* y,
                                                   const double* __restrict__ b)
{
    const int64_t gid = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const int s = static_cast<int>(gid / L);
    const int lane = static_cast<int>(gid % L);
    const bool valid = s < m.nbr;
    double acc[RB];
#pragma unroll
    for (int r = 0; r < RB; ++r) acc[r] = 0.0;
    if (valid) {
        const int k1 = m.rowptr[s + 1];
#pragma unroll 2
        for (int k = m.rowptr[s] + lane; k < k1; k += L) {
            const int c = __ldg(m.col + k);
            const double* vp = m.val + static_cast<int64_t>(k) * (RB * CB);
            double xv[CB];
#pragma unroll
            for (int d = 0; d < CB; ++d) xv[d] = __ldg(x + static_cast<int64_t>(c) * CB + d);
#pragma unroll
            for (int r = 0; r < RB; ++r)
#pragma unroll
                for (int d = 0; d < CB; ++d) acc[r] = fma(__ldg(vp + r * CB + d), xv[d], acc[r]);
        }
    }
#pragma unroll
    for (int r = 0; r < RB; ++r) acc[r] = group_sum<L>(acc[r]);
    if (valid && lane == 0) {
        const int row = m.perm ? m.perm[s] : s;
#pragma unroll
        for (int r = 0; r < RB; ++r) {
            const int64_t i = static_cast<int64_t>(row) * RB + r;
            if (MODE == 0) y[i] = acc[r];
            if (MODE == 1) y[i] = b[i] - acc[r];
            if (MODE == 2) y[i] = y[i] + acc[r];
        }
    }
}

// y = (M1 x1) + sgn (M2 x2); M1, M2 share the stored row order.
template <int RB, int CB1, int CB2, int L>
__global__ void __launch_bounds__(kThreads) k_spmv2(BsrArgs m1, BsrArgs m2, const double* __restrict__ x1,
                                                    const double* __restrict__ x2, double* y, double sgn)
{
    const int64_t gid = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const int s = static_cast<int>(gid / L);
    const int lane = static_cast<int>(gid % L);
    const bool valid = s < m1.nbr;
    double a1[RB], a2[RB];
#pragma unroll
    for (int r = 0; r < RB; ++r) a1[r] = a2[r] = 0.0;
    if (valid) {
        int k1 = m1.rowptr[s + 1];
#pragma unroll 2
        for (int k = m1.rowptr[s] + lane; k < k1; k += L) {
            const int c = __ldg(m1.col + k);
            const double* vp = m1.val + static_cast<int64_t>(k) * (RB * CB1);
#pragma unroll
            for (int d = 0; d < CB1; ++d) {
                const double xv = __ldg(x1 + static_cast<int64_t>(c) * CB1 + d);
#pragma unroll
                for (int r = 0; r < RB; ++r) a1[r] = fma(__ldg(vp + r * CB1 + d), xv, a1[r]);
            }
        }
        k1 = m2.rowptr[s + 1];
#pragma unroll 2
        for (int k = m2.rowptr[s] + lane; k < k1; k += L) {
            const int c = __ldg(m2.col + k);
            const double* vp = m2.val + static_cast<int64_t>(k) * (RB * CB2);
#pragma unroll
            for (int d = 0; d < CB2; ++d) {
                const double xv = __ldg(x2 + static_cast<int64_t>(c) * CB2 + d);
#pragma unroll
                for (int r = 0; r < RB; ++r) a2[r] = fma(__ldg(vp + r * CB2 + d), xv, a2[r]);
            }
        }
    }
#pragma unroll
    for (int r = 0; r < RB; ++r) {
        a1[r] = group_sum<L>(a1[r]);
        a2[r] = group_sum<L>(a2[r]);
    }
    if (valid && lane == 0) {
        const int row = m1.perm ? m1.perm[s] : s;
#pragma unroll
        for (int r = 0; r < RB; ++r) y[static_cast<int64_t>(row) * RB + r] = a1[r] + sgn * a2[r];
    }
}

// Row work of one Gauss-Seidel update (amg.cpp:311-322) for stored row s
// by a group of L lanes.  Everything that does not depend on z (the lane's
// first PF blocks, b, inv_diag, the diagonal block, the row's own old z) is
// loaded by prefetch_row() BEFORE the dependency wait; finish_row() then only
// gathers off-diagonal z values.
template <int B, int PF>
struct RowPref {
    int row, kb, ke;
    int c[PF];
    double v[PF][B * B];
    double b[B], id[B], D[B * B], zs[B];
};

template <int B, int L, int PF>
__device__ __forceinline__ void prefetch_row(const BsrArgs& m, const double* __restrict__ bvec,
                                             const double* __restrict__ invd, const double* z, int s, bool valid,
                                             int lane, RowPref<B, PF>& P)
{
    P.row = valid ? (m.perm ? m.perm[s] : s) : 0;
    P.kb = valid ? m.rowptr[s] + lane : 0;
    P.ke = valid ? m.rowptr[s + 1] : 0;
#pragma unroll
    for (int q = 0; q < PF; ++q) {
        const int k = P.kb + q * L;
        P.c[q] = k < P.ke ? __ldg(m.col + k) : -1;
        if (k < P.ke) {
#pragma unroll
            for (int e = 0; e < B * B; ++e) P.v[q][e] = __ldg(m.val + static_cast<int64_t>(k) * (B * B) + e);
        }
    }
    if (valid && lane == 0) {
        const int dp = m.dpos[s];
#pragma unroll
        for (int d = 0; d < B; ++d) {
            const int64_t i = static_cast<int64_t>(P.row) * B + d;
            P.b[d] = bvec[i];
            P.id[d] = invd[i];
            P.zs[d] = __ldcg(z + i); // only this row's owner writes z[row]
        }
#pragma unroll
        for (int e = 0; e < B * B; ++e) P.D[e] = dp >= 0 ? __ldg(m.val + static_cast<int64_t>(dp) * (B * B) + e) : 0.0;
    }
}

template <int B, int L, int PF, bool FWD, bool CG>
__device__ __forceinline__ void finish_row(const BsrArgs& m, double* z, bool valid, int lane, const RowPref<B, PF>& P)
{
    double acc[B];
#pragma unroll
    for (int r = 0; r < B; ++r) acc[r] = 0.0;
    // all z gathers of the prefetched blocks in flight at once (branch-free),
    // then the products of the blocks that count (off-diagonal, present)
    double zv[PF][B];
#pragma unroll
    for (int q = 0; q < PF; ++q) {
        const int64_t cc = P.c[q] >= 0 ? P.c[q] : 0;
#pragma unroll
        for (int d = 0; d < B; ++d) zv[q][d] = CG ? __ldcg(z + cc * B + d) : z[cc * B + d];
    }
#pragma unroll
    for (int q = 0; q < PF; ++q) {
        const bool use = P.c[q] >= 0 && P.c[q] != P.row;
#pragma unroll
        for (int d = 0; d < B; ++d)
#pragma unroll
            for (int r = 0; r < B; ++r) acc[r] = use ? fma(P.v[q][r * B + d], zv[q][d], acc[r]) : acc[r];
    }
    // long rows: the rest in batches of NB blocks per lane, all loads of a batch in flight
    constexpr int NB = B == 3 ? 2 : 8;
    for (int k0 = P.kb + PF * L; k0 < P.ke; k0 += NB * L) {
        int cb[NB];
        double vb[NB][B * B], zb[NB][B];
#pragma unroll
        for (int p = 0; p < NB; ++p) {
            const int k = k0 + p * L;
            const bool in = k < P.ke;
            cb[p] = in ? __ldg(m.col + k) : -1;
#pragma unroll
            for (int e = 0; e < B * B; ++e) vb[p][e] = in ? __ldg(m.val + static_cast<int64_t>(k) * (B * B) + e) : 0.0;
        }
#pragma unroll
        for (int p = 0; p < NB; ++p) {
            const int64_t cc = cb[p] >= 0 ? cb[p] : 0;
#pragma unroll
            for (int d = 0; d < B; ++d) zb[p][d] = CG ? __ldcg(z + cc * B + d) : z[cc * B + d];
        }
#pragma unroll
        for (int p = 0; p < NB; ++p) {
            if (cb[p] < 0 || cb[p] == P.row) continue;
#pragma unroll
            for (int d = 0; d < B; ++d)
#pragma unroll
                for (int r = 0; r < B; ++r) acc[r] = fma(vb[p][r * B + d], zb[p][d], acc[r]);
        }
    }
#pragma unroll
    for (int r = 0; r < B; ++r) acc[r] = group_sum<L>(acc[r]);
    if (valid && lane == 0) {
        double zs[B];
#pragma unroll
        for (int d = 0; d < B; ++d) zs[d] = P.zs[d];
#pragma unroll
        for (int ci = 0; ci < B; ++ci) {
            const int c = FWD ? ci : B - 1 - ci;
            double a = P.b[c] - acc[c];
#pragma unroll
            for (int d = 0; d < B; ++d)
                if (d != c) a -= P.D[c * B + d] * zs[d];
            zs[c] = a * P.id[c];
        }
#pragma unroll
        for (int d = 0; d < B; ++d) z[static_cast<int64_t>(P.row) * B + d] = zs[d];
    }
}

// ---- tagged dataflow sweep ------------------------------------------------
// A z entry is published as two 8-byte words {low half, epoch} {high half,
// epoch} (8-byte accesses are single-copy atomic, so a word whose tag equals
// this half sweep's epoch carries this half sweep's value: no flag, no fence and
// no second round trip between "the producer is done" and "its value is
// here").  A row waits only on the neighbours that precede it in the sweep
// (original index smaller in a forward sweep, larger in a backward sweep: the
// reference's in-place loop, amg.cpp:311-322); later neighbours are read from
// the plain z, which their owners overwrite only after consuming this row's
// tagged value (structurally symmetric pattern, BsrStruct::sym_pattern).
__device__ __forceinline__ void st_tagged(ulonglong2* p, double v, unsigned int tag)
{
    const unsigned long long b = static_cast<unsigned long long>(__double_as_longlong(v));
    const unsigned long long t = static_cast<unsigned long long>(tag) << 32;
    const unsigned long long w0 = (b & 0xffffffffull) | t, w1 = (b >> 32) | t;
    asm volatile("st.relaxed.gpu.global.v2.u64 [%0], {%1, %2};" ::"l"(p), "l"(w0), "l"(w1) : "memory");
}

__device__ __forceinline__ bool ld_tagged(const ulonglong2* p, unsigned int tag, double& v)
{
    unsigned long long w0, w1;
    asm volatile("ld.relaxed.gpu.global.v2.u64 {%0, %1}, [%2];" : "=l"(w0), "=l"(w1) : "l"(p) : "memory");
    v = __longlong_as_double(static_cast<long long>((w0 & 0xffffffffull) | (w1 << 32)));
    return static_cast<unsigned int>(w0 >> 32) == tag && static_cast<unsigned int>(w1 >> 32) == tag;
}

// NQ blocks per lane: columns c[q] (-1: none), row `row`.  Entries of the
// neighbours that precede the row in the sweep are polled until their tags
// carry this epoch (all lanes of the warp iterate together); the others come
// from the plain z.  (Measured alternatives, profiles/r02/sweeps.md: polling
// one sentinel word per row first, re-polling only the missing values, and a
// frontier hint for far-ahead warps were all slower.)
template <int B, int NQ, bool FWD>
__device__ __forceinline__ void gather_tagged(const int (&c)[NQ], int row, const double* z, const ulonglong2* zt,
                                              unsigned int epoch, double (&zv)[NQ][B])
{
    bool fresh[NQ];
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
        fresh[q] = c[q] >= 0 && (FWD ? c[q] < row : c[q] > row);
        const int64_t cc = c[q] >= 0 ? c[q] : 0;
#pragma unroll
        for (int d = 0; d < B; ++d) zv[q][d] = fresh[q] ? 0.0 : __ldcg(z + cc * B + d);
    }
    for (;;) {
        bool ok = true;
#pragma unroll
        for (int q = 0; q < NQ; ++q) {
            if (!fresh[q]) continue;
#pragma unroll
            for (int d = 0; d < B; ++d) ok = ld_tagged(zt + static_cast<int64_t>(c[q]) * B + d, epoch, zv[q][d]) && ok;
        }
        if (__all_sync(0xffffffffu, ok)) break;
        __nanosleep(40);
    }
}

template <int B, int L, int PF, bool FWD>
__device__ __forceinline__ void finish_row_tagged(const BsrArgs& m, double* z, ulonglong2* zt, unsigned int epoch,
                                                  bool valid, int lane, const RowPref<B, PF>& P)
{
    double acc[B];
#pragma unroll
    for (int r = 0; r < B; ++r) acc[r] = 0.0;
    {
        double zv[PF][B];
        gather_tagged<B, PF, FWD>(P.c, P.row, z, zt, epoch, zv);
#pragma unroll
        for (int q = 0; q < PF; ++q) {
            const bool use = P.c[q] >= 0 && P.c[q] != P.row;
#pragma unroll
            for (int d = 0; d < B; ++d)
#pragma unroll
                for (int r = 0; r < B; ++r) acc[r] = use ? fma(P.v[q][r * B + d], zv[q][d], acc[r]) : acc[r];
        }
    }
    // long rows: the rest in batches of NB blocks per lane (warp-uniform trip count)
    constexpr int NB = B == 3 ? 2 : 8;
    int more = 0;
    for (int k0 = P.kb + PF * L; k0 < P.ke; k0 += NB * L) ++more;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) more = max(more, __shfl_xor_sync(0xffffffffu, more, o));
    for (int it = 0; it < more; ++it) {
        const int k0 = P.kb + (PF + it * NB) * L;
        int cb[NB];
        double vb[NB][B * B], zb[NB][B];
#pragma unroll
        for (int p = 0; p < NB; ++p) {
            const int k = k0 + p * L;
            const bool in = k < P.ke;
            cb[p] = in ? __ldg(m.col + k) : -1;
#pragma unroll
            for (int e = 0; e < B * B; ++e) vb[p][e] = in ? __ldg(m.val + static_cast<int64_t>(k) * (B * B) + e) : 0.0;
        }
        gather_tagged<B, NB, FWD>(cb, P.row, z, zt, epoch, zb);
#pragma unroll
        for (int p = 0; p < NB; ++p) {
            const bool use = cb[p] >= 0 && cb[p] != P.row;
#pragma unroll
            for (int d = 0; d < B; ++d)
#pragma unroll
                for (int r = 0; r < B; ++r) acc[r] = use ? fma(vb[p][r * B + d], zb[p][d], acc[r]) : acc[r];
        }
    }
#pragma unroll
    for (int r = 0; r < B; ++r) acc[r] = group_sum<L>(acc[r]);
    if (valid && lane == 0) {
        double zs[B];
#pragma unroll
        for (int d = 0; d < B; ++d) zs[d] = P.zs[d];
#pragma unroll
        for (int ci = 0; ci < B; ++ci) {
            const int c = FWD ? ci : B - 1 - ci;
            double a = P.b[c] - acc[c];
#pragma unroll
            for (int d = 0; d < B; ++d)
                if (d != c) a -= P.D[c * B + d] * zs[d];
            zs[c] = a * P.id[c];
        }
#pragma unroll
        for (int d = 0; d < B; ++d) st_tagged(zt + static_cast<int64_t>(P.row) * B + d, zs[d], epoch);
#pragma unroll
        for (int d = 0; d < B; ++d) z[static_cast<int64_t>(P.row) * B + d] = zs[d];
    }
}

// One Gauss-Seidel half sweep, tagged dataflow.  Work items are 32/L rows of
// one level; every WARP takes items in level order from a ticket counter (the
// next ticket is taken before the current item is processed, so the atomic's
// latency is hidden): no CTA barrier and no level counter.  Deadlock-free under
// any residency: a row only waits on rows of earlier tickets, tickets are only
// held by running warps, and a warp works through its tickets in order.
template <int B, int L, bool FWD>
__global__ void __launch_bounds__(kThreads, 2) k_sgs_tag(BsrArgs m, const double* __restrict__ bvec, double* z,
                                                      ulonglong2* zt, unsigned int epoch,
                                                      const double* __restrict__ invd, int nitems,
                                                      const int* __restrict__ item_row, unsigned int* ticket)
{
    constexpr int PF = (B == 3) ? 3 : 4;
    constexpr int WPI = kThreads / 32; // warp items per table item (items hold <= kThreads / L rows)
    constexpr int RPW = 32 / L;        // rows per warp item
    const int lane32 = threadIdx.x & 31;
    const int g = lane32 / L;
    const int lane = lane32 % L;
    const int nw = nitems * WPI;
    auto take = [&]() {
        unsigned int t = 0;
        if (lane32 == 0) t = atomicAdd(ticket, 1u);
        return static_cast<int>(__shfl_sync(0xffffffffu, t, 0));
    };
    int t = take();
    while (t < nw) {
        const int tn = take();
        const int tt = FWD ? t : nw - 1 - t;
        const int item = tt / WPI;
        const int s = item_row[item] + (tt % WPI) * RPW + g;
        const bool valid = s < item_row[item + 1];
        if (__any_sync(0xffffffffu, valid)) {
            RowPref<B, PF> P;
            prefetch_row<B, L, PF>(m, bvec, invd, z, s, valid, lane, P);
            if (!valid) {
#pragma unroll
                for (int q = 0; q < PF; ++q) P.c[q] = -1;
            }
            finish_row_tagged<B, L, PF, FWD>(m, z, zt, epoch, valid, lane, P);
        }
        t = tn;
    }
}

template <int B, int L, bool FWD>
__global__ void __launch_bounds__(512) k_sgs_chain(BsrArgs m, const double* __restrict__ bvec, double* z,
                                                    const double* __restrict__ invd, const int* __restrict__ lev_ptr,
                                                    int nlev)
{
    constexpr int PF = (B == 3) ? 2 : 4;
    constexpr int G = 512 / L;
    const int g = threadIdx.x / L;
    const int lane = threadIdx.x % L;
    for (int li = 0; li < nlev; ++li) {
        const int lev = FWD ? li : nlev - 1 - li;
        const int r0 = lev_ptr[lev], r1 = lev_ptr[lev + 1];
        for (int base = r0; base < r1; base += G) {
            const int s = base + g;
            const bool valid = s < r1;
            RowPref<B, PF> P;
            prefetch_row<B, L, PF>(m, bvec, invd, z, s, valid, lane, P);
            finish_row<B, L, PF, FWD, false>(m, z, valid, lane, P);
        }
        __syncthreads();
    }
}

template <int RB, int CB, int L>
__global__ void __launch_bounds__(kThreads) k_scale(BsrArgs m, double* val, const double* __restrict__ wr,
                                                    const double* __restrict__ wc)
{
    const int64_t gid = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const int s = static_cast<int>(gid / L);
    const int lane = static_cast<int>(gid % L);
    if (s >= m.nbr) return;
    const int row = m.perm ? m.perm[s] : s;
    for (int k = m.rowptr[s] + lane; k < m.rowptr[s + 1]; k += L) {
        const int c = m.col[k];
        double* vp = val + static_cast<int64_t>(k) * (RB * CB);
#pragma unroll
        for (int r = 0; r < RB; ++r)
#pragma unroll
            for (int d = 0; d < CB; ++d)
                // blocksystem.cpp:85: val *= wrow[r] * wcol[c]
                vp[r * CB + d] = vp[r * CB + d] * (wr[static_cast<int64_t>(row) * RB + r] * wc[static_cast<int64_t>(c) * CB + d]);
    }
}

template <int B>
__global__ void k_diag(BsrArgs m, double* d)
{
    const int s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= m.nbr) return;
    const int row = m.perm ? m.perm[s] : s;
    const int dp = m.dpos[s];
#pragma unroll
    for (int r = 0; r < B; ++r)
        d[static_cast<int64_t>(row) * B + r] = dp >= 0 ? m.val[static_cast<int64_t>(dp) * (B * B) + r * B + r] : 0.0;
}

__global__ void k_inv_diag(const double* __restrict__ d, double* invd, int64_t n)
{
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < n) invd[i] = d[i] != 0.0 ? 1.0 / d[i] : 1.0;
}

__global__ void k_recip(const double* __restrict__ d, double* out, int64_t n)
{
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < n) out[i] = 1.0 / d[i];
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
    for (int j = lane; j < n; j += 32) s = fma(P[static_cast<int64_t>(row) * n + j], r[j], s);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) z[row] = s;
}

inline int grid_groups(int64_t rows, int L) { return static_cast<int>((rows * L + kThreads - 1) / kThreads); }

#define ED_LANES(L, ...)                   \
    switch (L) {                           \
    case 2: { constexpr int LL = 2; __VA_ARGS__; break; }  \
    case 4: { constexpr int LL = 4; __VA_ARGS__; break; }  \
    case 8: { constexpr int LL = 8; __VA_ARGS__; break; }  \
    case 16: { constexpr int LL = 16; __VA_ARGS__; break; } \
    default: { constexpr int LL = 32; __VA_ARGS__; break; } \
    }

template <int RB, int CB>
void launch_spmv(const Bsr& M, const double* x, double* y, const double* b, int mode, cudaStream_t s)
{
    const BsrStruct& S = *M.st;
    if (S.nbr == 0) return;
    const BsrArgs a = args_of(M);
    const int g = grid_groups(S.nbr, S.L);
    ED_LANES(S.L, {
        if (mode == 0) k_spmv<RB, CB, LL, 0><<<g, kThreads, 0, s>>>(a, x, y, b);
        else if (mode == 1) k_spmv<RB, CB, LL, 1><<<g, kThreads, 0, s>>>(a, x, y, b);
        else k_spmv<RB, CB, LL, 2><<<g, kThreads, 0, s>>>(a, x, y, b);
    })
    after_launch("k_spmv");
}

template <int RB, int C1, int C2>
void launch_spmv2(const Bsr& M1, const double* x1, const Bsr& M2, const double* x2, double* y, double sgn,
                  cudaStream_t s)
{
    const BsrStruct& S = *M1.st;
    if (S.nbr == 0) return;
    const int g = grid_groups(S.nbr, S.L);
    ED_LANES(S.L, { k_spmv2<RB, C1, C2, LL><<<g, kThreads, 0, s>>>(args_of(M1), args_of(M2), x1, x2, y, sgn); })
    after_launch("k_spmv2");
}

template <int B>
void launch_sgs(const Bsr& A, const double* b, double* z, const double* invd, bool fwd, cudaStream_t s,
                const double* dense)
{
    const BsrStruct& S = *A.st;
    if (S.nitems == 0) return;
    const int nlev = S.nlev();
    const BsrArgs a = args_of(A);
    if (group_sweep_on(S)) {
        sgs_group(A, b, z, invd, fwd, s, dense);
        return;
    }
    if (S.chain) {
        ED_LANES(S.Ls, {
            if (fwd)
                k_sgs_chain<B, LL, true><<<1, 512, 0, s>>>(a, b, z, invd, S.d_lev_ptr.p, nlev);
            else
                k_sgs_chain<B, LL, false><<<1, 512, 0, s>>>(a, b, z, invd, S.d_lev_ptr.p, nlev);
        })
        after_launch("k_sgs_chain");
        return;
    }
    // the tagged dataflow sweep (every leveled operator is structurally symmetric: pattern_symmetric
    // is checked where the level schedule is built)
    {
        if (S.ztag.n != static_cast<size_t>(S.nbr) * B) {
            S.ztag.alloc(static_cast<size_t>(S.nbr) * B);
            S.ztag.zero(s);
            S.tag_epoch = 0;
        }
        if (++S.tag_epoch == 0) { // epoch wrap: start over from clean tags
            S.ztag.zero(s);
            S.tag_epoch = 1;
        }
        ED_CUDA(cudaMemsetAsync(S.sync.p, 0, sizeof(unsigned int), s)); // the ticket
        // eight levels' worth of warps (measured best of 1..16 at 40^3, profiles/r02/sweeps.md): fewer
        // cannot hide an item's ticket + matrix-prefetch latency, more only add polling traffic
        const int64_t per_level = (static_cast<int64_t>(S.nitems) * (kThreads / 32) + nlev - 1) / std::max(nlev, 1);
        static const int lv_ahead = std::getenv("ED_TAG_AHEAD") ? std::atoi(std::getenv("ED_TAG_AHEAD")) : 8;
        const int tgrid =
            static_cast<int>(std::min<int64_t>(148 * 2, std::max<int64_t>(1, (lv_ahead * per_level + 7) / 8)));
        ED_LANES(S.Ls, {
            if (fwd)
                k_sgs_tag<B, LL, true><<<tgrid, kThreads, 0, s>>>(a, b, z, S.ztag.p, S.tag_epoch, invd, S.nitems,
                                                                 S.item_row.p, S.sync.p);
            else
                k_sgs_tag<B, LL, false><<<tgrid, kThreads, 0, s>>>(a, b, z, S.ztag.p, S.tag_epoch, invd, S.nitems,
                                                                  S.item_row.p, S.sync.p);
        })
        after_launch("k_sgs_tag");
    }
}

} // namespace

void spmv(const Bsr& M, const double* x, double* y, const double* b, int mode, cudaStream_t s)
{
    const int RB = M.st->Rb, CB = M.st->Cb;
    AcctScope acct(s, "k_spmv", M.bytes_per_spmv());
    if (RB == 1 && CB == 1) return launch_spmv<1, 1>(M, x, y, b, mode, s);
    if (RB == 3 && CB == 3) return launch_spmv<3, 3>(M, x, y, b, mode, s);
    if (RB == 3 && CB == 1) return launch_spmv<3, 1>(M, x, y, b, mode, s);
    if (RB == 1 && CB == 3) return launch_spmv<1, 3>(M, x, y, b, mode, s);
    throw Error(ED_UNSUPPORTED, "spmv: unsupported block shape");
}

void spmv2(const Bsr& M1, const double* x1, const Bsr& M2, const double* x2, double* y, double sgn, cudaStream_t s)
{
    const int RB = M1.st->Rb, C1 = M1.st->Cb, C2 = M2.st->Cb;
    if (M2.st->Rb != RB || M2.st->nbr != M1.st->nbr || M2.st->h_perm != M1.st->h_perm)
        throw Error(ED_INVALID_ARGUMENT, "spmv2: row layouts differ");
    AcctScope acct(s, "k_spmv2", M1.bytes_per_spmv() + M2.bytes_per_spmv() - 8.0 * M1.st->nbr * RB);
    if (RB == 3 && C1 == 3 && C2 == 1) return launch_spmv2<3, 3, 1>(M1, x1, M2, x2, y, sgn, s);
    if (RB == 1 && C1 == 3 && C2 == 1) return launch_spmv2<1, 3, 1>(M1, x1, M2, x2, y, sgn, s);
    if (RB == 1 && C1 == 1 && C2 == 3) return launch_spmv2<1, 1, 3>(M1, x1, M2, x2, y, sgn, s);
    if (RB == 1 && C1 == 1 && C2 == 1) return launch_spmv2<1, 1, 1>(M1, x1, M2, x2, y, sgn, s);
    throw Error(ED_UNSUPPORTED, "spmv2: unsupported block shape");
}

void sgs_sweep(const Bsr& A, const double* b, double* z, const double* invd, bool forward, cudaStream_t s,
               const double* dense)
{
    const int B = A.st->Rb;
    if (A.st->Cb != B) throw Error(ED_INVALID_ARGUMENT, "sgs: non-square blocks");
    if (!A.st->leveled && A.st->nbr > 1) throw Error(ED_INVALID_ARGUMENT, "sgs: operator has no level schedule");
    const BsrStruct& S = *A.st;
    // algorithmic bytes of one half sweep: blocks + column indices once, row
    // pointers, b and inv_diag read, z read and written
    const double bytes = static_cast<double>(S.nnzb) * (8.0 * B * B + 4.0) + 4.0 * (S.nbr + 1) +
                         4.0 * 8.0 * S.nbr * B;
    const char* kname = group_sweep_on(S) ? "k_group_sweep" : S.chain ? "k_sgs_chain" : "k_sgs_tag";
    AcctScope acct(s, kname, bytes);
    if (B == 1) return launch_sgs<1>(A, b, z, invd, forward, s, dense);
    if (B == 3) return launch_sgs<3>(A, b, z, invd, forward, s, dense);
    throw Error(ED_UNSUPPORTED, "sgs: unsupported block size");
}

int sweep_mode()
{
    // ED_SWEEP=legacy: never the group sweep; ED_SWEEP=group: always (where a schedule exists)
    static const int mode = !std::getenv("ED_SWEEP")                              ? 0
                            : std::string(std::getenv("ED_SWEEP")) == "legacy" ? 1
                            : std::string(std::getenv("ED_SWEEP")) == "group"  ? 2
                                                                               : 0;
    return mode;
}

bool group_sweep_on(const BsrStruct& S)
{
    const int mode = sweep_mode();
    return S.ngrp > 0 && mode != 1 && (mode == 2 || S.grp_use);
}

void sweep_prepare(const Bsr& A, const double* invd, DevArray<double>& aux, cudaStream_t s)
{
    if (group_sweep_on(*A.st)) return group_prepare(A, invd, aux, s);
    aux.release();
}

void jacobi_update(double* z, const double* b, const double* t, const double* invd, double w, int64_t n,
                   cudaStream_t s)
{
    if (n == 0) return;
    k_jacobi<<<static_cast<int>((n + kThreads - 1) / kThreads), kThreads, 0, s>>>(z, b, t, invd, w, n);
    after_launch("k_jacobi");
}

void bsr_scale(Bsr& M, const double* wr, const double* wc, cudaStream_t s)
{
    const BsrStruct& S = *M.st;
    if (S.nbr == 0) return;
    const BsrArgs a = args_of(M);
    const int g = grid_groups(S.nbr, S.L);
#define ED_SCALE(R, C)                                                                    \
    if (S.Rb == R && S.Cb == C) {                                                         \
        ED_LANES(S.L, { k_scale<R, C, LL><<<g, kThreads, 0, s>>>(a, M.val.p, wr, wc); }) \
        after_launch("k_scale");                                                          \
        return;                                                                           \
    }
    ED_SCALE(1, 1)
    ED_SCALE(3, 3)
    ED_SCALE(3, 1)
    ED_SCALE(1, 3)
#undef ED_SCALE
    throw Error(ED_UNSUPPORTED, "scale: unsupported block shape");
}

void bsr_diag(const Bsr& M, double* d, cudaStream_t s)
{
    const BsrStruct& S = *M.st;
    if (S.Rb != S.Cb || S.nbr != S.nbc) throw Error(ED_INVALID_ARGUMENT, "diag: non-square operator");
    if (S.nbr == 0) return;
    const int g = (S.nbr + kThreads - 1) / kThreads;
    if (S.Rb == 1)
        k_diag<1><<<g, kThreads, 0, s>>>(args_of(M), d);
    else
        k_diag<3><<<g, kThreads, 0, s>>>(args_of(M), d);
    after_launch("k_diag");
}

void inv_diag_from(const double* d, double* invd, int64_t n, cudaStream_t s)
{
    if (n == 0) return;
    k_inv_diag<<<static_cast<int>((n + kThreads - 1) / kThreads), kThreads, 0, s>>>(d, invd, n);
    after_launch("k_inv_diag");
}

void recip(const double* d, double* out, int64_t n, cudaStream_t s)
{
    if (n == 0) return;
    k_recip<<<static_cast<int>((n + kThreads - 1) / kThreads), kThreads, 0, s>>>(d, out, n);
    after_launch("k_recip");
}

void dense_gemv(const double* P, const double* r, double* z, int n, cudaStream_t s)
{
    if (n == 0) return;
    const int rows_per_block = kThreads / 32;
    acct_vec("k_dense_gemv", 8.0 * n * n + 16.0 * n);
    k_dense_gemv<<<(n + rows_per_block - 1) / rows_per_block, kThreads, 0, s>>>(P, r, z, n);
    after_launch("k_dense_gemv");
}

} // namespace edb
