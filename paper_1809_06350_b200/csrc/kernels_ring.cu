// Cluster push Gauss-Seidel half sweep (amg.cpp:311-322 semantics) for deep,
// moderately wide level schedules -- the first coarse levels of the
// reference's smoothed aggregation (hundreds of dependency levels of tens of
// long rows) and the S_hat operator.
//
// One thread-block cluster (16 CTAs, one per SM) runs the whole half sweep
// with no cluster-wide barrier per level:
//   * every stored row is owned by one CTA (rows of each level are dealt
//     round-robin, bsr_host.cpp:ring_order); the owner keeps the row's z, b
//     and inv_diag in its shared memory;
//   * for level l, CTA c computes for EVERY row of the level the partial row
//     sum over the columns c owns -- local shared-memory z reads only -- and
//     pushes it to the row's owner with st.async, which completes on the
//     owner's mbarrier for that level (kSlots slots, by level; a CTA that
//     owns no row for kSlots-1 levels could overrun a slot, so setup inserts
//     a cluster barrier there, bsr_host.cpp:push_barriers);
//   * the owner waits for its mbarrier (all cs partials of all its rows of
//     the level), adds the partials in CTA order (deterministic), solves the
//     row's diagonal block in sweep order and writes z locally; a CTA barrier
//     publishes the new z to its own warps for the next level;
//   * the matrix streams through a per-CTA byte ring in shared memory: one
//     elected thread keeps up to 32 (level, CTA) chunks in flight (partial
//     segments, packed column indices and blocks, the own rows' diagonal
//     blocks: four cp.async.bulk copies completing on one mbarrier).
// A level costs one local gather + FMA + lane reduction, one DSMEM push, one
// mbarrier hand-off and the diagonal solve.
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>

#include "ed_internal.hpp"

namespace edb {
namespace {

namespace cg = cooperative_groups;

constexpr int kT = 512;             // 16 warps: 15 workers (partials), 1 owner warp (solves, producer)
constexpr int kW = kT - 32;
constexpr int kNMB = 32;            // chunks in flight (mbarrier ring)
constexpr int kDynMax = 225 * 1024; // dynamic shared memory per CTA
constexpr int kSlots = 4;           // partial-sum slots (bsr_host.cpp: kRingSlots, push_barriers)

struct PushArgs {
    const int4* chunk; // [nlev*cs][2]
    const int4* seg;
    const int* pcol;
    const double* pval;  // packed off-diagonal blocks
    const double* pdiag; // diagonal blocks, stored row order
    const int* own;
    const int* own_ptr;
    int nlev, cap, slice, part, maxm;
    long long* prof;
    int exp; // ED_PUSH_EXP (profiling builds only): 1 skip early sums, 2 skip late blocks
    int lgmax; // log2 of the widest lane group per segment in the early sums
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_tx(uint64_t* bar, uint32_t bytes)
{
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
// acquire at cluster scope: the partials come from other CTAs
__device__ __forceinline__ void mbar_wait_cluster(uint64_t* bar, uint32_t parity)
{
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "PW_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra PW_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
    // one cluster-scope acquire after the spin (restricted to shared memory:
    // the partials land in this CTA's shared memory), not one per poll
    asm volatile("fence.acquire.sync_restrict::shared::cluster.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity)
{
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "RW_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra RW_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar)
{
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ uint32_t mapa(uint32_t a, int rank)
{
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
    return r;
}
__device__ __forceinline__ void st_async_f64(uint32_t a, double v, uint32_t bar)
{
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.f64 [%0], %1, [%2];" ::"r"(a), "d"(v), "r"(bar)
                 : "memory");
}
__device__ __forceinline__ void st_async_v2f64(uint32_t a, double v0, double v1, uint32_t bar)
{
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f64 [%0], {%1, %2}, [%3];" ::"r"(a),
                 "d"(v0), "d"(v1), "r"(bar)
                 : "memory");
}
// cluster barrier ordering this thread's own shared-memory accesses (no MEMBAR.GPU)
__device__ __forceinline__ void cl_sync()
{
    asm volatile("fence.release.sync_restrict::shared::cta.cluster;" ::: "memory");
    asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");
    asm volatile("barrier.cluster.wait.aligned;" ::: "memory");
}

template <int B, bool FWD, bool PROF>
__global__ void __launch_bounds__(kT, 1) k_sgs_push(PushArgs q, const double* __restrict__ bvec, double* z,
                                                      const double* __restrict__ invd)
{
    constexpr int BB = B * B;
    constexpr int PB = B == 3 ? 4 : 1; // doubles per partial entry (16-B aligned v2 pushes for B = 3)
    // late partials by threads [0, kL), early sums by [kE0, kW).  Measured
    // (ED_RING_PROF, A1 at 40^3): giving the two disjoint warp groups
    // (kL = kE0 = 128) leaves the per-level time unchanged (~2,900 cycles
    // profiled), so every worker does both in turn.
    constexpr int kL = kW;
    constexpr int kE0 = 0;
    extern __shared__ __align__(128) unsigned char dsm[];
    __shared__ __align__(8) uint64_t mbar[kNMB];
    __shared__ __align__(8) uint64_t pbar[kSlots];
    __shared__ int pst[kNMB];
    __shared__ int4 meta[kNMB];  // {ring offset, first segment, rows of the level, first packed block}
    __shared__ int4 meta2[kNMB]; // {own rows start, own rows, z offset, barrier flags}
    __shared__ int4 meta3[kNMB]; // {column-word bytes, value bytes, packed blocks, 0}
    unsigned char* ring = dsm;
    double* zs = reinterpret_cast<double*>(dsm + q.cap);
    double* bs = zs + q.slice;
    double* is = bs + q.slice;
    double* part = is + q.slice; // [kSlots][part bytes]
    double* esum = part + kSlots * (q.part / 8); // [2][maxm][B] early sums of the next level's segments
    const int tid = threadIdx.x;
    cg::cluster_group cl = cg::this_cluster();
    const int rank = static_cast<int>(cl.block_rank());
    const int cs = static_cast<int>(cl.num_blocks());
    const int nlev = q.nlev, cap = q.cap;
    const bool producer = tid == kW - 32; // lane 0 of the last worker warp (off the owner warp's path)

    if (tid == 0) {
        for (int i = 0; i < kNMB; ++i) mbar_init(&mbar[i], 1);
        for (int i = 0; i < kSlots; ++i) mbar_init(&pbar[i], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    const int o0 = q.own_ptr[rank], o1 = q.own_ptr[rank + 1];
    for (int i = tid; i < (o1 - o0) * B; i += kT) {
        const int r = i / B, d = i - r * B;
        const int64_t gi = static_cast<int64_t>(q.own[o0 + r]) * B + d;
        zs[i] = z[gi];
        bs[i] = bvec[gi];
        is[i] = invd[gi];
    }
    __syncthreads();

    // ---- producer: chunk (level i of the sweep) -> ring, table entry loaded one issue ahead
    int issued = 0, head = 0;
    int4 n1 = make_int4(0, 0, 0, 0), n2 = n1;
    auto load_next = [&]() {
        if (issued < nlev) {
            const int lev = FWD ? issued : nlev - 1 - issued;
            n1 = q.chunk[(lev * cs + rank) * 2];
            n2 = q.chunk[(lev * cs + rank) * 2 + 1];
        }
    };
    // at most max_issue chunks per call: in steady state one chunk is freed per
    // level, and the table entry of the next chunk (loaded one issue ahead)
    // then has a whole level to arrive instead of stalling the producer
    auto issue_more = [&](int consumed, int max_issue) {
        for (int it = 0; it < max_issue && issued < nlev && issued - consumed < kNMB; ++it) {
            const int m = n1.y, pk0 = n1.z, pk1 = n1.w, s0 = n2.x, nown = n2.y;
            const int ca = pk0 & ~3, ce = (pk1 + 3) & ~3, va = pk0 & ~1, ve = (pk1 + 1) & ~1;
            const int da = s0 & ~1, de = (s0 + nown + 1) & ~1;
            const int hb = 16 * m, cb = 4 * (ce - ca), vb = 8 * BB * (ve - va), db = 8 * BB * (de - da);
            const int sz = hb + cb + vb + db;
            int p = head;
            const int off = p % cap;
            if (off + sz > cap) p += cap - off;
            const int tail = consumed < issued ? pst[consumed % kNMB] : p;
            if (p + sz - tail > cap) break;
            const int slot = issued % kNMB;
            pst[slot] = p;
            meta[slot] = make_int4(p % cap, n1.x, m, pk0);
            meta2[slot] = make_int4(s0, nown, n2.z, n2.w);
            meta3[slot] = make_int4(cb, vb, pk1 - pk0, 0);
            head = p + sz;
            uint64_t* bar = &mbar[slot];
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            mbar_arrive_tx(bar, static_cast<uint32_t>(sz));
            unsigned char* dst = ring + (p % cap);
            if (hb) bulk_g2s(dst, q.seg + n1.x, hb, bar);
            if (cb) bulk_g2s(dst + hb, q.pcol + ca, cb, bar);
            if (vb) bulk_g2s(dst + hb + cb, q.pval + static_cast<int64_t>(va) * BB, vb, bar);
            if (db) bulk_g2s(dst + hb + cb + vb, q.pdiag + static_cast<int64_t>(da) * BB, db, bar);
            ++issued;
            load_next();
        }
    };
    if (producer) {
        load_next();
        issue_more(0, kNMB);
    }
    // every CTA's barriers initialised before anyone pushes
    cl_sync();

    const uint32_t part_u32 = smem_u32(part);
    const uint32_t pbar_u32 = smem_u32(&pbar[0]);
    const bool prof = PROF && tid == 0;
    const bool prof7 = PROF && tid == kW; // owner warp: wait for partials / solve
    long long w7[3] = {0, 0, 0};
    long long pt[6] = {0, 0, 0, 0, 0, 0};
    const long long t_start = prof ? clock64() : 0;

    // chunk view (everything from shared memory; slot metadata written by the
    // producer before its arrive on the chunk's mbarrier)
    struct View {
        const int4* segs;
        const int* pc;
        const double* pv;
        const double* pd;
        int m, s0, nown, zoff, flags, pk0, nblk;
    };
    auto open_chunk = [&](int i) {
        const int slot = i % kNMB;
        mbar_wait(&mbar[slot], static_cast<uint32_t>((i / kNMB) & 1));
        const int4 mt = meta[slot], m2 = meta2[slot];
        const int4 m3 = meta3[slot];
        View v;
        const unsigned char* base = ring + mt.x;
        v.m = mt.z;
        v.s0 = m2.x;
        v.nown = m2.y;
        v.zoff = m2.z;
        v.flags = m2.w;
        v.pk0 = mt.w;
        v.nblk = m3.z;
        v.segs = reinterpret_cast<const int4*>(base);
        v.pc = reinterpret_cast<const int*>(base + 16 * v.m) - (mt.w & ~3);
        v.pv = reinterpret_cast<const double*>(base + 16 * v.m + m3.x) - static_cast<int64_t>(mt.w & ~1) * BB;
        v.pd = reinterpret_cast<const double*>(base + 16 * v.m + m3.x + m3.y) - static_cast<int64_t>(v.s0 & ~1) * BB;
        return v;
    };
    // blocks [k0, k1) of a segment: acc += A_blocks z_cols (local z)
    auto seg_sum = [&](const View& v, int k0, int k1, int step, double* acc) {
        auto fma_blk = [&](const double* bl, const double* zz) {
#pragma unroll
            for (int d = 0; d < B; ++d)
#pragma unroll
                for (int r = 0; r < B; ++r) acc[r] = fma(bl[r * B + d], zz[d], acc[r]);
        };
        int k = k0;
        // two blocks per trip: both blocks' column words, z and values are
        // loaded before the FMAs (shared-memory latency overlapped), the FMAs
        // keep the one-block-at-a-time order (results unchanged)
        for (; k + step < k1; k += 2 * step) {
            const int c0 = v.pc[k], c1 = v.pc[k + step];
            double z0[B], z1[B], b0[BB], b1[BB];
#pragma unroll
            for (int d = 0; d < B; ++d) {
                z0[d] = zs[c0 + d];
                z1[d] = zs[c1 + d];
            }
            const double* p0 = v.pv + static_cast<int64_t>(k) * BB;
            const double* p1 = v.pv + static_cast<int64_t>(k + step) * BB;
#pragma unroll
            for (int e = 0; e < BB; ++e) {
                b0[e] = p0[e];
                b1[e] = p1[e];
            }
            fma_blk(b0, z0);
            fma_blk(b1, z1);
        }
        if (k < k1) {
            const int c0 = v.pc[k];
            double z0[B], b0[BB];
#pragma unroll
            for (int d = 0; d < B; ++d) z0[d] = zs[c0 + d];
            const double* p0 = v.pv + static_cast<int64_t>(k) * BB;
#pragma unroll
            for (int e = 0; e < BB; ++e) b0[e] = p0[e];
            fma_blk(b0, z0);
        }
    };
    // early phase of chunk v (workers only): each segment's early part
    // (columns not on the level solved just before it) by a group of G lanes,
    // reduced by shuffles in a fixed order -> es[j]
    // t: thread index inside the early group of nt threads (whole warps)
    auto early = [&](const View& v, double* es, int t, int nt) {
        // largest lg <= 5 with m << lg <= nt (closed form, no per-thread loop)
        const int lg = min(q.lgmax, v.m > 0 ? min(5, max(0, 31 - __clz(nt / v.m))) : 5);
        const int G = 1 << lg, lane = t & (G - 1);
        for (int j0 = 0; j0 < v.m; j0 += nt >> lg) {
            const int j = j0 + (t >> lg);
            double acc[B];
#pragma unroll
            for (int r = 0; r < B; ++r) acc[r] = 0.0;
            if (j < v.m) {
                const int4 h = v.segs[j];
                const int na = h.w >> 16, nb = h.w & 0xFFFF;
                const int e0 = FWD ? h.x + na : h.x, e1 = FWD ? h.y : h.y - nb;
                seg_sum(v, e0 + lane, e1, G, acc);
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1)
                if (o < G) {
#pragma unroll
                    for (int r = 0; r < B; ++r) acc[r] += __shfl_xor_sync(0xffffffffu, acc[r], o);
                }
            if (j < v.m && lane == 0)
#pragma unroll
                for (int r = 0; r < B; ++r) es[j * B + r] = acc[r];
        }
    };

    View cur = open_chunk(0);
    if (tid >= kE0 && tid < kW) early(cur, esum, tid - kE0, kW - kE0);
    __syncthreads();
    for (int li = 0; li < nlev; ++li) {
        const int par = li % kSlots;
        const long long t0 = prof ? clock64() : 0;
        // slot reuse guard (bsr_host.cpp: push_barriers); identical on every CTA
        if (cur.flags & (FWD ? 1 : 2)) cl_sync();
        // arm this level's partial barrier: every CTA pushes one entry per own row
        if (tid == 0) mbar_arrive_tx(&pbar[par], static_cast<uint32_t>(cur.nown * cs * B * 8));
        const double* es = esum + (li & 1) * q.maxm * B;
        // ---- early sum + late part (columns solved on the previous level,
        // fresh z), pushed to the owners
        if (tid < kL) {
            for (int j = tid; j < cur.m; j += kL) {
                const int4 h = cur.segs[j];
                const int na = h.w >> 16, nb = h.w & 0xFFFF;
                double acc[B];
#pragma unroll
                for (int r = 0; r < B; ++r) acc[r] = es[j * B + r];
                if (!(PROF && (q.exp & 2))) {
                    if (FWD) seg_sum(cur, h.x, h.x + na, 1, acc);
                    else seg_sum(cur, h.y - nb, h.y, 1, acc);
                }
                const int owner = h.z >> 24;
                const uint32_t dst = mapa(part_u32, owner) + static_cast<uint32_t>(par * q.part + (h.z & 0xFFFFFF));
                const uint32_t bar = mapa(pbar_u32 + 8 * par, owner);
                if (B == 3) {
                    st_async_v2f64(dst, acc[0], acc[B > 1 ? 1 : 0], bar);
                    st_async_f64(dst + 16, acc[B - 1], bar);
                } else {
                    st_async_f64(dst, acc[0], bar);
                }
            }
        }
        const long long t1 = prof ? clock64() : 0;
        View nxt = cur;
        if (li + 1 < nlev) {
            // ---- workers: products of the next level while the partials travel
            if (tid < kW) {
                nxt = open_chunk(li + 1);
                if (prof) pt[5] += clock64() - t1;
                if (tid >= kE0 && !(PROF && (q.exp & 1)))
                    early(nxt, esum + ((li + 1) & 1) * q.maxm * B, tid - kE0, kW - kE0);
            }
        }
        const long long t2 = prof ? clock64() : 0;
        // ---- last warp: own rows, 8 lanes per row -- the cs partials summed in
        // a fixed tree, the diagonal block solved in sweep order
        if (tid >= kW) {
            const int lane = tid - kW;
            // the next chunk's view while the partials travel (its copies were
            // issued levels ago), not after the solve on the critical path
            if (li + 1 < nlev) nxt = open_chunk(li + 1);
            const long long ta = prof7 ? clock64() : 0;
            long long tb = ta;
            for (int t = lane; t < cur.nown; t += 32) {
                // everything but the partials, before the wait
                const int zl = cur.zoff + t * B;
                const double* Dp = cur.pd + static_cast<int64_t>(cur.s0 + t) * BB;
                double D[BB], zn[B], bb[B], ii[B];
#pragma unroll
                for (int e = 0; e < BB; ++e) D[e] = Dp[e];
#pragma unroll
                for (int d = 0; d < B; ++d) {
                    zn[d] = zs[zl + d];
                    bb[d] = bs[zl + d];
                    ii[d] = is[zl + d];
                }
                mbar_wait_cluster(&pbar[par], static_cast<uint32_t>((li / kSlots) & 1));
                if (prof7) tb = w7[2] = clock64();
                const double* pp = part + par * (q.part / 8) + static_cast<int64_t>(t) * cs * PB;
                // the cs partials in a fixed pairwise tree
                double acc[B];
#pragma unroll
                for (int r = 0; r < B; ++r) {
                    double h[16];
#pragma unroll
                    for (int c = 0; c < 16; ++c) h[c] = c < cs ? pp[c * PB + r] : 0.0;
#pragma unroll
                    for (int w = 8; w > 0; w >>= 1)
#pragma unroll
                        for (int c = 0; c < w; ++c) h[c] += h[c + w];
                    acc[r] = h[0];
                }
#pragma unroll
                for (int ci = 0; ci < B; ++ci) {
                    const int c = FWD ? ci : B - 1 - ci;
                    double a = bb[c] - acc[c];
#pragma unroll
                    for (int d = 0; d < B; ++d)
                        if (d != c) a -= D[c * B + d] * zn[d];
                    zn[c] = a * ii[c];
                }
#pragma unroll
                for (int d = 0; d < B; ++d) zs[zl + d] = zn[d];
            }
            if (prof7) {
                const long long tc = clock64();
                w7[0] += tb - ta;
                w7[1] += tc - tb;
            }
        }
    const long long t3 = prof ? clock64() : 0;
        if (PROF && (rank == 0 || rank == 7) && li >= 200 && li < 264 && (tid & 31) == 0) {
            long long* tr = q.prof + 128 + ((rank ? 1 : 0) * 64 + li - 200) * 16;
            tr[tid >> 5] = clock64();
            if (tid == 0) {
                tr[9] = t0;
                tr[10] = t1;
                tr[11] = cur.flags;
                tr[12] = cur.m;
                tr[13] = cur.nown;
            }
            if (tid == kW) tr[8] = w7[2];
        }
        __syncthreads(); // new z visible to every warp; chunk li consumed
        if (producer) issue_more(li + 1, 1);
        cur = nxt;
        if (prof) {
            const long long t4 = clock64();
            pt[0] += t1 - t0;
            pt[1] += t2 - t1;
            pt[2] += t3 - t2;
            pt[3] += t4 - t3;
        }
    }
    if (prof) {
        pt[4] = clock64() - t_start;
        for (int k = 0; k < 5; ++k) q.prof[rank * 8 + k] = pt[k];
        q.prof[rank * 8 + 7] = pt[5];
    }
    if (prof7) {
        q.prof[rank * 8 + 5] = w7[0];
        q.prof[rank * 8 + 6] = w7[1];
    }
    // no CTA leaves while a peer may still push into it
    cl_sync();
    for (int i = tid; i < (o1 - o0) * B; i += kT) {
        const int r = i / B, d = i - r * B;
        z[static_cast<int64_t>(q.own[o0 + r]) * B + d] = zs[i];
    }
}

// packed = [off-diagonal blocks, padded to an even count (16-B aligned bulk
// copies)][diagonal blocks in stored row order]
__global__ void k_ring_pack(const int* __restrict__ psrc, const int* __restrict__ dpos, const double* __restrict__ val,
                            double* out, int64_t npk, int nbr, int BB)
{
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const int64_t nv = ((npk + 1) & ~1LL) * BB;
    if (i < nv) {
        out[i] = i < npk * BB ? val[static_cast<int64_t>(psrc[i / BB]) * BB + i % BB] : 0.0;
    } else if (i < nv + static_cast<int64_t>(nbr) * BB) {
        const int64_t j = i - nv;
        const int s = static_cast<int>(j / BB);
        out[i] = dpos[s] >= 0 ? val[static_cast<int64_t>(dpos[s]) * BB + j % BB] : 0.0;
    }
}

// widest lane group per segment of the early sums (log2): narrower groups mean
// fewer shuffle rounds and fewer issuing warps per level.  Measured at 40^3
// (ED_PUSH_LG sweep, profiles/r01d_ncu_summary.md): A1 sweep 674 us at 5, 661-665
// at 3 and 2, 706 at 1; S0 430 us at 5, 427 at 2
template <int B>
constexpr int kLgMax()
{
    return B == 3 ? 3 : 2;
}

template <int B>
void launch(const Bsr& A, const double* b, double* z, const double* invd, bool fwd, cudaStream_t s,
            const double* packed)
{
    const BsrStruct& S = *A.st;
    static const bool prof_on = std::getenv("ED_RING_PROF") != nullptr;
    auto kern = prof_on ? (fwd ? k_sgs_push<B, true, true> : k_sgs_push<B, false, true>)
                        : (fwd ? k_sgs_push<B, true, false> : k_sgs_push<B, false, false>);
    static bool attr_done[2] = {};
    if (!attr_done[fwd ? 1 : 0]) {
        ED_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, kDynMax));
        ED_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
        attr_done[fwd ? 1 : 0] = true;
    }
    static long long* prof = nullptr;
    if (prof_on && !prof) ED_CUDA(cudaMallocManaged(&prof, sizeof(long long) * (128 + 2 * 64 * 16)));
    const int slice = (S.ring_slice + 1) & ~1;
    const PushArgs q{S.rchunk.p, S.rseg.p,     S.rpcol.p, packed,     packed + ((S.ring_npk + 1) & ~1LL) * B * B,
                     S.rown.p,   S.rown_ptr.p, S.nlev(),  S.ring_cap, slice,
                     S.ring_part, S.ring_maxm, prof_on ? prof : nullptr,
                     std::getenv("ED_PUSH_EXP") ? std::atoi(std::getenv("ED_PUSH_EXP")) : 0,
                     std::getenv("ED_PUSH_LG") ? std::atoi(std::getenv("ED_PUSH_LG")) : kLgMax<B>()};
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(S.ring_cs, 1, 1);
    cfg.blockDim = dim3(kT, 1, 1);
    cfg.dynamicSmemBytes = static_cast<size_t>(S.ring_cap) + 3 * static_cast<size_t>(slice) * sizeof(double) +
                           kSlots * static_cast<size_t>(S.ring_part) + push_scratch_bytes(S.ring_maxm, B);
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = S.ring_cs;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    ED_CUDA(cudaLaunchKernelEx(&cfg, kern, q, b, z, invd));
    after_launch("k_sgs_push");
    if (prof_on) {
        static int nprint = 0;
        ED_CUDA(cudaStreamSynchronize(s));
        if (nprint++ < 8) {
            std::fprintf(stderr, "[push] B=%d %s nlev=%d rows=%d cs=%d cap=%d |", B, fwd ? "fwd" : "bwd", S.nlev(), S.nbr,
                         S.ring_cs, S.ring_cap);
            for (int k = 0; k < 8; ++k) std::fprintf(stderr, " %.0f", prof[k] / static_cast<double>(S.nlev()));
            std::fprintf(stderr, " cyc/level (late+push early-next own-solve sync | total | w7: wait solve | open-next)\n");
            if (nprint == 1)
                for (int r = 0; r < 2; ++r)
                    for (int li = 0; li < 40; ++li) {
                        const long long* tr = prof + 128 + (r * 64 + li) * 16;
                        std::fprintf(stderr, "   trace cta%d lev%2d m=%3lld own=%2lld fl=%lld | push %5lld | w7 ready %5lld | warps at sync:",
                                     r ? 7 : 0, li, tr[12], tr[13], tr[11], tr[10] - tr[9], tr[8] - tr[9]);
                        for (int w = 0; w < 8; ++w) std::fprintf(stderr, " %5lld", tr[w] - tr[9]);
                        std::fprintf(stderr, "\n");
                    }
            for (int c = 1; c < S.ring_cs; c += 5)
                std::fprintf(stderr, "   cta %d: %.0f %.0f %.0f %.0f | %.0f | %.0f %.0f\n", c, prof[c * 8] / double(S.nlev()),
                             prof[c * 8 + 1] / double(S.nlev()), prof[c * 8 + 2] / double(S.nlev()),
                             prof[c * 8 + 3] / double(S.nlev()), prof[c * 8 + 4] / double(S.nlev()),
                             prof[c * 8 + 5] / double(S.nlev()), prof[c * 8 + 6] / double(S.nlev()));
        }
    }
}

} // namespace

static int ring_cluster_size_query()
{
    int cs = 0;
    auto kern = k_sgs_push<3, true, false>;
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, kDynMax) != cudaSuccess ||
        cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) != cudaSuccess) {
        cudaGetLastError();
        return cs;
    }
    for (int c = 16; c >= 8; c /= 2) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(c, 1, 1);
        cfg.blockDim = dim3(kT, 1, 1);
        cfg.dynamicSmemBytes = kDynMax;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = c;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        int n = 0;
        if (cudaOccupancyMaxActiveClusters(&n, kern, &cfg) == cudaSuccess && n > 0) {
            cs = c;
            break;
        }
        cudaGetLastError();
    }
    return cs;
}

int ring_cluster_size()
{
    // largest cluster (16 non-portable, else 8) of full-shared-memory CTAs the device can co-schedule
    static const int cs = ring_cluster_size_query(); // thread-safe once
    return cs;
}

int push_scratch_bytes(int maxm, int B) { return 8 * ((2 * maxm * B + 1) & ~1); }

int ring_capacity(int slice, int parts)
{
    const int zb = 3 * ((slice * 8 + 15) & ~15); // z, b, inv_diag slices
    return (kDynMax - zb - parts) & ~15;
}

void ring_pack(const Bsr& A, DevArray<double>& packed, cudaStream_t s)
{
    const BsrStruct& S = *A.st;
    const int BB = S.Rb * S.Cb;
    const int64_t n = (((S.ring_npk + 1) & ~1LL) + S.nbr) * BB;
    packed.alloc(static_cast<size_t>(n));
    k_ring_pack<<<static_cast<unsigned>((n + 255) / 256), 256, 0, s>>>(S.rpsrc.p, S.dpos.p, A.val.p, packed.p,
                                                                      S.ring_npk, S.nbr, BB);
    after_launch("k_ring_pack");
}

void sgs_ring(const Bsr& A, const double* b, double* z, const double* invd, bool fwd, cudaStream_t s,
              const double* packed)
{
    if (!packed) throw Error(ED_INVALID_ARGUMENT, "push sweep needs the operator's packed blocks (ring_pack)");
    if (A.st->Rb == 1) return launch<1>(A, b, z, invd, fwd, s, packed);
    if (A.st->Rb == 3) return launch<3>(A, b, z, invd, fwd, s, packed);
    throw Error(ED_UNSUPPORTED, "push sweep: unsupported block size");
}

} // namespace edb
