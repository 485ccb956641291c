// Blocked Gauss-Seidel half sweep for narrow, deep level schedules -- the
// dense coarse operators of the reference's smoothed aggregation, which have
// ~1 row per dependency level (amg.cpp:311-322 in-place sweep semantics).
//
// Stored rows (a topological order of the sweep) are cut into groups of
// GR = 32/B consecutive block rows, i.e. <= 32 scalar rows.  Sweeping group h:
//   * warp 0 (solver) runs the scalar recurrence of the group in sweep order,
//     one lane per scalar row: z_t = (b_t - acc_t) * invd_t, broadcast by
//     shuffle, then every later row of the group adds its coupling to z_t
//     (the group's own dense block) -- and in the same pass the rows of the
//     NEXT group add theirs (the "fold" block), so the next group never waits
//     for a re-read of z_h;
//   * warps 1..15 (producers) meanwhile stage the next group: its own and fold
//     blocks (one TMA bulk copy each into shared memory), b and inv_diag, and
//     its row sums over every column that is neither in the group being
//     solved nor an earlier row of its own group.  Each producer warp keeps
//     its first two (row, chunk) units of the next group's blocks in registers
//     across the CTA barrier, so their loads overlap the solve.
// One CTA barrier per group instead of one barrier per level; z lives in
// shared memory in stored order.  Row sums are the reference's split into
// partial sums in a fixed order (deterministic, roundoff-level differences).
#include <cuda_runtime.h>

#include <cstdint>

#include "ed_internal.hpp"

namespace edb {
namespace {

constexpr int kT = 512;          // 1 solver warp + 15 producer warps
constexpr int kNPW = 15;         // producer warps
constexpr int kU3 = 2, kU1 = 8;  // blocks per lane per unit (B = 3 / 1)

struct Args {
    const int* perm; // stored -> original block row (null: identity)
    const double* val;
    const int* colp;     // stored position of each block's column
    const double* dense; // [ng*3 + 1][32*32]: own / previous / next group block (col-major), then a zero block
    const int* gunit;    // [ng+1]
    const int4* units;   // (local row, k0, k1, -)
    const int* rowu;     // [ng][33]
    int nbr, ng, nsc;
};

__device__ __forceinline__ void producers_sync() { asm volatile("bar.sync 1, 480;" ::: "memory"); }

__device__ __forceinline__ uint32_t smem_addr(const void* p)
{
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes)
{
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity)
{
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(smem_addr(bar)),
        "r"(parity)
        : "memory");
}

// 1-D bulk copy global -> shared, completing on the mbarrier (TMA engine)
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar)
{
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_addr(dst)),
        "l"(src), "r"(bytes), "r"(smem_addr(bar))
        : "memory");
}

template <int B, int U>
struct Unit {
    int lr, kbeg, kend;
    int sc[U];
    double v[U][B * B];
};

template <int B, int U>
__device__ __forceinline__ void unit_fetch(const Args& q, int kb, int kend, int lane, Unit<B, U>& R)
{
    R.kbeg = kb;
    R.kend = kend;
#pragma unroll
    for (int j = 0; j < U; ++j) {
        const int k = kb + j * 32 + lane;
        const bool ok = k < kend;
        R.sc[j] = ok ? q.colp[k] : -1;
#pragma unroll
        for (int e = 0; e < B * B; ++e) R.v[j][e] = ok ? q.val[static_cast<int64_t>(k) * (B * B) + e] : 0.0;
    }
}

template <int B, int U>
__device__ __forceinline__ void unit_load(const Args& q, int unit, int lane, Unit<B, U>& R)
{
    const int4 rec = q.units[unit];
    R.lr = rec.x;
    unit_fetch<B, U>(q, rec.y, rec.z, lane, R);
}

// Partial row sum of one unit over the columns outside `solving` and outside
// the earlier rows of its own group X (those are the solver's).
template <int B, int U, bool FWD>
__device__ __forceinline__ void unit_sum(const Unit<B, U>& R, const double* zs, int X, int solving, double* acc)
{
    constexpr int GR = 32 / B;
#pragma unroll
    for (int j = 0; j < U; ++j) {
        const int c = R.sc[j];
        if (c < 0) continue;
        const int gc = c / GR;
        if (gc == solving) continue;
        if (gc == X) {
            const int lc = c - X * GR;
#pragma unroll
            for (int d = 0; d < B; ++d) {
                const double zv = zs[c * B + d];
                const int cl = lc * B + d;
#pragma unroll
                for (int r = 0; r < B; ++r) {
                    const int tl = R.lr * B + r;
                    if (FWD ? cl > tl : cl < tl) acc[r] = fma(R.v[j][r * B + d], zv, acc[r]);
                }
            }
        } else {
#pragma unroll
            for (int d = 0; d < B; ++d) {
                const double zv = zs[c * B + d];
#pragma unroll
                for (int r = 0; r < B; ++r) acc[r] = fma(R.v[j][r * B + d], zv, acc[r]);
            }
        }
    }
}

// the whole unit (first U*32 blocks in R, the rest streamed through R)
template <int B, int U, bool FWD>
__device__ __forceinline__ void unit_total(const Args& q, Unit<B, U>& R, const double* zs, int X, int solving,
                                           int lane, double* acc)
{
    unit_sum<B, U, FWD>(R, zs, X, solving, acc);
    for (int kb = R.kbeg + 32 * U; kb < R.kend; kb += 32 * U) {
        unit_fetch<B, U>(q, kb, R.kend, lane, R);
        unit_sum<B, U, FWD>(R, zs, X, solving, acc);
    }
}

template <int B, bool FWD>
__global__ void __launch_bounds__(kT) k_sgs_blocked(Args q, const double* __restrict__ bvec, double* z,
                                                     const double* __restrict__ invd)
{
    constexpr int GR = 32 / B;
    constexpr int U = B == 3 ? kU3 : kU1;
    extern __shared__ __align__(128) double smem[];
    __shared__ __align__(8) uint64_t mbar[2];
    const int nsc = q.nsc, ng = q.ng, nbr = q.nbr;
    double* Gs = smem;       // [2][32*32] own block, col-major (c, t)   (TMA destination, 16-B aligned)
    double* Fs = Gs + 2048;  // [2][32*32] fold block                     (TMA destination)
    double* far = Fs + 2048; // [2][32]
    double* bs = far + 64;   // [2][32]
    double* is = bs + 64;    // [2][32]
    double* part = is + 64;  // [kBlockedMaxUnits][B]
    double* zs = part + BsrStruct::kBlockedMaxUnits * B; // [nsc] stored order
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    if (tid == 0) {
        mbar_init(&mbar[0], 1);
        mbar_init(&mbar[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    for (int i = tid; i < nsc; i += kT) {
        const int s = i / B, d = i - s * B;
        zs[i] = z[static_cast<int64_t>(q.perm ? q.perm[s] : s) * B + d];
    }
    // this producer warp's first two units of the next group, in flight across the barrier
    Unit<B, U> P0, P1;
    auto prefetch = [&](int X) {
        if (X < 0 || X >= ng) return;
        const int u0 = q.gunit[X], nu = q.gunit[X + 1] - u0;
        if (warp - 1 < nu) unit_load<B, U>(q, u0 + warp - 1, lane, P0);
        if (warp - 1 + kNPW < nu) unit_load<B, U>(q, u0 + warp - 1 + kNPW, lane, P1);
    };
    if (warp > 0) prefetch(FWD ? 0 : ng - 1);
    __syncthreads();

    // producers: stage group X into buffer `buf` while the solver works on `solving`
    auto stage = [&](int X, int buf, int solving) {
        const int ptid = tid - 32;
        const int s0 = X * GR;
        const int R = min(GR, nbr - s0);
        const int Ts = R * B;
        if (ptid == 0) {
            const int hf = FWD ? X + 1 : X - 1;
            const double* dg = q.dense + static_cast<int64_t>(X) * 3 * 1024;
            const double* df = (hf >= 0 && hf < ng) ? q.dense + (static_cast<int64_t>(hf) * 3 + (FWD ? 1 : 2)) * 1024
                                                    : q.dense + static_cast<int64_t>(ng) * 3 * 1024; // zero block
            // generic-proxy reads of this buffer (two iterations ago) precede the async-proxy writes
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            mbar_expect_tx(&mbar[buf], 2 * 1024 * sizeof(double));
            bulk_g2s(Gs + buf * 1024, dg, 1024 * sizeof(double), &mbar[buf]);
            bulk_g2s(Fs + buf * 1024, df, 1024 * sizeof(double), &mbar[buf]);
        }
        double bb = 0.0, ii = 1.0;
        int ru0 = 0, ru1 = 0;
        if (ptid < Ts) {
            const int s = s0 + ptid / B;
            const int64_t gi = static_cast<int64_t>(q.perm ? q.perm[s] : s) * B + (ptid - (ptid / B) * B);
            bb = bvec[gi];
            ii = invd[gi];
            ru0 = q.rowu[X * 33 + ptid / B];
            ru1 = q.rowu[X * 33 + ptid / B + 1];
        }
        const int u0 = q.gunit[X], nu = q.gunit[X + 1] - u0;
        int j = 0;
        for (int ul = warp - 1; ul < nu; ul += kNPW, ++j) {
            double acc[B];
#pragma unroll
            for (int r = 0; r < B; ++r) acc[r] = 0.0;
            if (j == 0) {
                unit_total<B, U, FWD>(q, P0, zs, X, solving, lane, acc);
            } else {
                if (j > 1) unit_load<B, U>(q, u0 + ul, lane, P1); // beyond the first two: on demand
                unit_total<B, U, FWD>(q, P1, zs, X, solving, lane, acc);
            }
#pragma unroll
            for (int r = 0; r < B; ++r) {
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) acc[r] += __shfl_xor_sync(0xffffffffu, acc[r], o);
            }
            if (lane == 0)
#pragma unroll
                for (int r = 0; r < B; ++r) part[ul * B + r] = acc[r];
        }
        // the group staged next time: its first units go in flight now
        prefetch(FWD ? X + 1 : X - 1);
        if (ptid < 32) {
            bs[buf * 32 + ptid] = bb;
            is[buf * 32 + ptid] = ii;
        }
        producers_sync();
        if (ptid < Ts) {
            const int r = ptid - (ptid / B) * B;
            double a = 0.0;
            for (int u = ru0; u < ru1; ++u) a += part[u * B + r];
            far[buf * 32 + ptid] = a;
        }
    };

    if (warp > 0) stage(FWD ? 0 : ng - 1, 0, -1);
    __syncthreads();
    double carry = 0.0;
    for (int it = 0; it < ng; ++it) {
        const int h = FWD ? it : ng - 1 - it;
        const int cb = it & 1;
        if (warp == 0) {
            const int R = min(GR, nbr - h * GR);
            const int Ts = R * B;
            const int t = lane;
            double acc = t < Ts ? far[cb * 32 + t] + carry : 0.0;
            const double bq = bs[cb * 32 + t], iq = is[cb * 32 + t];
            mbar_wait(&mbar[cb], static_cast<uint32_t>((it >> 1) & 1));
            const double* G = Gs + cb * 1024;
            const double* F = Fs + cb * 1024;
            double fold = 0.0, zval = 0.0;
#pragma unroll 4
            for (int jj = 0; jj < Ts; ++jj) {
                const int cur = FWD ? jj : Ts - 1 - jj;
                const double g = G[cur * 32 + t], f = F[cur * 32 + t];
                const double u = (bq - acc) * iq;
                const double zj = __shfl_sync(0xffffffffu, u, cur);
                if (t == cur) zval = u;
                if (FWD ? t > cur : t < cur) acc = fma(g, zj, acc);
                fold = fma(f, zj, fold);
            }
            if (t < Ts) zs[h * GR * B + t] = zval;
            carry = fold;
        } else if (it + 1 < ng) {
            stage(FWD ? h + 1 : h - 1, cb ^ 1, h);
        }
        __syncthreads();
    }
    for (int i = tid; i < nsc; i += kT) {
        const int s = i / B, d = i - s * B;
        z[static_cast<int64_t>(q.perm ? q.perm[s] : s) * B + d] = zs[i];
    }
}

size_t smem_bytes(int nsc, int B)
{
    return (static_cast<size_t>(2048) + 2048 + 64 * 3 + static_cast<size_t>(BsrStruct::kBlockedMaxUnits) * B + nsc) *
           sizeof(double);
}

__global__ void k_blocked_dense(const int* __restrict__ imap, const double* __restrict__ val, double* dense, int64_t n,
                                int64_t ntot)
{
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < n) dense[i] = imap[i] >= 0 ? val[imap[i]] : 0.0;
    else if (i < ntot) dense[i] = 0.0; // trailing zero block (fold of the last group)
}

template <int B>
void launch(const Bsr& A, const double* b, double* z, const double* invd, bool fwd, cudaStream_t s,
            const double* dense)
{
    const BsrStruct& S = *A.st;
    const int nsc = S.nbr * B;
    auto kern = fwd ? k_sgs_blocked<B, true> : k_sgs_blocked<B, false>;
    static bool attr_done[2] = {};
    if (!attr_done[fwd ? 1 : 0]) {
        ED_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     static_cast<int>(smem_bytes(BsrStruct::kBlockedMaxScalars, B))));
        attr_done[fwd ? 1 : 0] = true;
    }
    const Args q{S.perm.p, A.val.p, S.colp.p, dense, S.gunit.p, S.units.p, S.rowu.p, S.nbr, S.ngroups, nsc};
    kern<<<1, kT, smem_bytes(nsc, B), s>>>(q, b, z, invd);
    after_launch("k_sgs_blocked");
}

} // namespace

void blocked_dense(const Bsr& A, DevArray<double>& dense, cudaStream_t s)
{
    const BsrStruct& S = *A.st;
    if (S.ring_cs > 0) return ring_pack(A, dense, s); // push sweep: packed blocks (kernels_ring.cu)
    if (!S.blocked) return;
    const int64_t n = static_cast<int64_t>(S.ngroups) * 3 * 1024;
    const int64_t ntot = n + 1024;
    dense.alloc(ntot);
    k_blocked_dense<<<static_cast<unsigned>((ntot + 255) / 256), 256, 0, s>>>(S.imap.p, A.val.p, dense.p, n, ntot);
    after_launch("k_blocked_dense");
}

void sgs_blocked(const Bsr& A, const double* b, double* z, const double* invd, bool fwd, cudaStream_t s,
                 const double* dense)
{
    if (!dense) throw Error(ED_INVALID_ARGUMENT, "blocked Gauss-Seidel needs the operator's dense group blocks");
    if (A.st->Rb == 1) return launch<1>(A, b, z, invd, fwd, s, dense);
    if (A.st->Rb == 3) return launch<3>(A, b, z, invd, fwd, s, dense);
    throw Error(ED_UNSUPPORTED, "blocked sweep: unsupported block size");
}

} // namespace edb
