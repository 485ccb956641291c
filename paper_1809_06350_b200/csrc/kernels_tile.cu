// Tiled cluster Gauss-Seidel half sweep (amg.cpp:311-322 semantics) for the
// fine velocity level when its vector fits a 16-CTA cluster's shared memory
// (the 40^3 cube of BASELINE configs[1]: 120 dependency levels of ~560 rows).
//
// The free nodes are partitioned into 16 spatial tiles (equal-count x/y
// bisection of the node coordinates, bsr_host.cpp:tile_order); CTA c owns
// the rows of tile c and keeps their z in its shared memory.  Levels are
// swept in order; a row reads the z of its columns from the owning CTA's
// shared memory -- its own for the interior of the tile, a neighbour's
// (ld.shared::cluster) only on tile boundaries -- solves its diagonal block
// in sweep order and writes z locally.  Writers fence their shared-memory
// stores at cluster scope (sync_restrict: no MEMBAR.GPU) and one cluster
// barrier (relaxed arrive, acquire wait, ~120 cycles) separates levels.
// The tile's rows of every level stream through a per-CTA byte ring of
// sub-chunks (row headers, column z-locations, blocks: three cp.async.bulk
// copies completing on one mbarrier); between the arrive and the wait every
// thread stages its first rows of the next level (blocks, addresses, b and
// inv_diag from global memory, diagonal block, own old z) into registers.
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>

#include "ed_internal.hpp"

namespace edb {
namespace {

namespace cg = cooperative_groups;

constexpr int kT = 512;
constexpr int kNMB = 32;            // sub-chunks in flight
constexpr int kDynMax = 225 * 1024; // dynamic shared memory per CTA

struct TileArgs {
    const int4* ent;     // per-CTA entries {s0, s1, kb, ke}: stored rows / blocks of a sub-chunk
    const int* ent_ptr;  // [cs+1]
    const int* ent_info; // local z index of the entry's first row << 1 | (last entry of its level: a cluster barrier follows)
    const int4* hdr;     // [nbr] {kb, ke, original row, diagonal block}
    const int* colz;     // [nnzb] owner << 24 | byte offset of the column's z in the owner's slice
    const double* val;   // [nnzb*B*B] stored order
    const int* own;      // [nbr] original rows in (CTA, local) order
    const int* own_ptr;  // [cs+1]
    int cap;
    long long* prof; // ED_TILE_PROF: per-CTA cycle split of thread 0
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
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity)
{
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "TW_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra TW_%=;\n"
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
__device__ __forceinline__ double ld_dsm(uint32_t a)
{
    double v;
    asm volatile("ld.shared::cluster.f64 %0, [%1];" : "=d"(v) : "r"(a) : "memory");
    return v;
}
__device__ __forceinline__ void fence_release_smem()
{
    asm volatile("fence.release.sync_restrict::shared::cta.cluster;" ::: "memory");
}
__device__ __forceinline__ void cl_arrive() { asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory"); }
__device__ __forceinline__ void cl_wait() { asm volatile("barrier.cluster.wait.aligned;" ::: "memory"); }

template <int B>
struct TRow {
    bool valid;
    int lane, G, kb, ke, dp, zl;
    uint32_t a[B == 3 ? 2 : 4];
    double v[B == 3 ? 2 : 4][B * B];
    double b[B], id[B], D[B * B], zo[B];
};

template <int B>
struct TView {
    const int4* h;   // indexed by stored row
    const int* cz;   // indexed by stored block
    const double* vs; // indexed by stored block * B*B
    int s0, m, last, zoff;
};

template <int B, bool FWD>
__global__ void __launch_bounds__(kT, 1) k_sgs_tile(TileArgs q, const double* __restrict__ bvec, double* z,
                                                      const double* __restrict__ invd)
{
    constexpr int BB = B * B;
    constexpr int PF = B == 3 ? 2 : 4;
    extern __shared__ __align__(128) unsigned char dsm[];
    __shared__ __align__(8) uint64_t mbar[kNMB];
    __shared__ int pst[kNMB];
    __shared__ int4 meta[kNMB]; // {ring offset, s0, rows, last}
    __shared__ int2 meta2[kNMB]; // {first column word, first value block}
    __shared__ int meta3[kNMB];  // column-word bytes
    __shared__ int meta4[kNMB];  // local z index of the first row
    __shared__ uint32_t zbase[16];
    unsigned char* ring = dsm;
    double* zs = reinterpret_cast<double*>(dsm + q.cap);
    const int tid = threadIdx.x;
    cg::cluster_group cl = cg::this_cluster();
    const int rank = static_cast<int>(cl.block_rank());
    const int cs = static_cast<int>(cl.num_blocks());
    const int cap = q.cap;
    const int e_begin = q.ent_ptr[rank], nent = q.ent_ptr[rank + 1] - e_begin;
    const bool producer = tid == kT - 32;

    if (tid == 0) {
        for (int i = 0; i < kNMB; ++i) mbar_init(&mbar[i], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    const int o0 = q.own_ptr[rank], o1 = q.own_ptr[rank + 1];
    for (int i = tid; i < (o1 - o0) * B; i += kT) {
        const int r = i / B, d = i - r * B;
        zs[i] = z[static_cast<int64_t>(q.own[o0 + r]) * B + d];
    }
    if (tid < cs) zbase[tid] = mapa(smem_u32(zs), tid);
    __syncthreads();

    // ---- producer (one thread): entries -> ring, the next entry's table row loaded one issue ahead
    int issued = 0, head = 0;
    int4 ne = make_int4(0, 0, 0, 0);
    int nl = 0;
    auto load_next = [&]() {
        if (issued < nent) {
            ne = q.ent[e_begin + issued];
            nl = q.ent_info[e_begin + issued];
        }
    };
    auto issue = [&](int consumed, int max_issue) {
        for (int it = 0; it < max_issue && issued < nent && issued - consumed < kNMB; ++it) {
            const int m = ne.y - ne.x;
            const int ca = ne.z & ~3, ce = (ne.w + 3) & ~3, va = ne.z & ~1, ve = (ne.w + 1) & ~1;
            const int hb = 16 * m, cb = 4 * (ce - ca), vb = 8 * BB * (ve - va);
            const int sz = hb + cb + vb;
            int p = head;
            const int off = p % cap;
            if (off + sz > cap) p += cap - off;
            const int tail = consumed < issued ? pst[consumed % kNMB] : p;
            if (p + sz - tail > cap) break;
            const int slot = issued % kNMB;
            pst[slot] = p;
            meta[slot] = make_int4(p % cap, ne.x, m, nl & 1);
            meta4[slot] = nl >> 1;
            meta2[slot] = make_int2(ca, va);
            meta3[slot] = cb;
            head = p + sz;
            uint64_t* bar = &mbar[slot];
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            mbar_arrive_tx(bar, static_cast<uint32_t>(sz));
            unsigned char* dst = ring + (p % cap);
            if (hb) bulk_g2s(dst, q.hdr + ne.x, hb, bar);
            if (cb) bulk_g2s(dst + hb, q.colz + ca, cb, bar);
            if (vb) bulk_g2s(dst + hb + cb, q.val + static_cast<int64_t>(va) * BB, vb, bar);
            ++issued;
            load_next();
        }
    };
    if (producer) {
        load_next();
        issue(0, kNMB);
    }
    // every slice loaded and every mbarrier initialised before anyone reads a peer
    asm volatile("barrier.cluster.arrive.aligned;" ::: "memory");
    cl_wait();

    auto open = [&](int i) {
        const int slot = i % kNMB;
        mbar_wait(&mbar[slot], static_cast<uint32_t>((i / kNMB) & 1));
        const int4 mt = meta[slot];
        const int2 m2 = meta2[slot];
        TView<B> v;
        const unsigned char* base = ring + mt.x;
        v.s0 = mt.y;
        v.m = mt.z;
        v.last = mt.w;
        v.zoff = meta4[slot];
        v.h = reinterpret_cast<const int4*>(base) - mt.y;
        v.cz = reinterpret_cast<const int*>(base + 16 * mt.z) - m2.x;
        v.vs = reinterpret_cast<const double*>(base + 16 * mt.z + meta3[slot]) - static_cast<int64_t>(m2.y) * BB;
        return v;
    };
    auto stage = [&](const TView<B>& v, int q0, TRow<B>& R) {
        int lg = 5;
        while (lg > 0 && (v.m << lg) > kT) --lg;
        R.G = 1 << lg;
        R.lane = tid & (R.G - 1);
        const int qq = q0 + (tid >> lg);
        R.valid = qq < v.m;
        int4 h = make_int4(0, 0, 0, -1);
        if (R.valid) h = v.h[v.s0 + qq];
        R.kb = h.x;
        R.ke = h.y;
        R.dp = h.w;
        R.zl = v.zoff + qq * B;
#pragma unroll
        for (int t = 0; t < PF; ++t) {
            const int k = R.kb + R.lane + t * R.G;
            const bool ok = R.valid && k < R.ke && k != R.dp;
            const int cz = ok ? v.cz[k] : 0;
            R.a[t] = ok ? zbase[cz >> 24] + (cz & 0xFFFFFF) : 0xFFFFFFFFu;
#pragma unroll
            for (int e = 0; e < BB; ++e) R.v[t][e] = ok ? v.vs[static_cast<int64_t>(k) * BB + e] : 0.0;
        }
        if (R.valid && R.lane == 0) {
            const int64_t row = h.z;
#pragma unroll
            for (int d = 0; d < B; ++d) {
                R.b[d] = bvec[row * B + d];
                R.id[d] = invd[row * B + d];
                R.zo[d] = zs[R.zl + d];
            }
#pragma unroll
            for (int e = 0; e < BB; ++e) R.D[e] = R.dp >= 0 ? v.vs[static_cast<int64_t>(R.dp) * BB + e] : 0.0;
        }
    };
    auto solve = [&](const TView<B>& v, const TRow<B>& R) {
        double acc[B];
#pragma unroll
        for (int r = 0; r < B; ++r) acc[r] = 0.0;
        double zv[PF][B];
#pragma unroll
        for (int t = 0; t < PF; ++t)
#pragma unroll
            for (int d = 0; d < B; ++d) zv[t][d] = R.a[t] != 0xFFFFFFFFu ? ld_dsm(R.a[t] + 8 * d) : 0.0;
#pragma unroll
        for (int t = 0; t < PF; ++t)
#pragma unroll
            for (int d = 0; d < B; ++d)
#pragma unroll
                for (int r = 0; r < B; ++r) acc[r] = fma(R.v[t][r * B + d], zv[t][d], acc[r]);
        if (R.valid) {
            for (int k = R.kb + R.lane + PF * R.G; k < R.ke; k += R.G) {
                if (k == R.dp) continue;
                const int cz = v.cz[k];
                const uint32_t a = zbase[cz >> 24] + (cz & 0xFFFFFF);
                double zz[B];
#pragma unroll
                for (int d = 0; d < B; ++d) zz[d] = ld_dsm(a + 8 * d);
#pragma unroll
                for (int d = 0; d < B; ++d)
#pragma unroll
                    for (int r = 0; r < B; ++r) acc[r] = fma(v.vs[static_cast<int64_t>(k) * BB + r * B + d], zz[d], acc[r]);
            }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1)
            if (o < R.G) {
#pragma unroll
                for (int r = 0; r < B; ++r) acc[r] += __shfl_xor_sync(0xffffffffu, acc[r], o);
            }
        if (R.valid && R.lane == 0) {
            double zn[B];
#pragma unroll
            for (int d = 0; d < B; ++d) zn[d] = R.zo[d];
#pragma unroll
            for (int ci = 0; ci < B; ++ci) {
                const int c = FWD ? ci : B - 1 - ci;
                double a = R.b[c] - acc[c];
#pragma unroll
                for (int d = 0; d < B; ++d)
                    if (d != c) a -= R.D[c * B + d] * zn[d];
                zn[c] = a * R.id[c];
            }
#pragma unroll
            for (int d = 0; d < B; ++d) zs[R.zl + d] = zn[d];
        }
    };

    TRow<B> R;
    TView<B> v;
    if (nent > 0) {
        v = open(0);
        stage(v, 0, R);
    }
    bool wrote = false;
    const bool prof = q.prof != nullptr && tid == 0;
    long long pt[6] = {0, 0, 0, 0, 0, 0};
    long long tlast = prof ? clock64() : 0;
    for (int i = 0; i < nent; ++i) {
        const long long t0 = prof ? clock64() : 0;
        solve(v, R);
        wrote = wrote || (R.valid && R.lane == 0);
        const int rpp = kT / R.G;
        for (int q0 = rpp; q0 < v.m; q0 += rpp) {
            stage(v, q0, R);
            solve(v, R);
            wrote = wrote || (R.valid && R.lane == 0);
        }
        if (v.last) {
            const long long t1 = prof ? clock64() : 0;
            if (wrote) fence_release_smem(); // only writers pay the release
            wrote = false;
            cl_arrive();
            const long long t2 = prof ? clock64() : 0;
            if (i + 1 < nent) {
                v = open(i + 1);
                if (prof) pt[4] += clock64() - t2;
                stage(v, 0, R);
            }
            const long long t3 = prof ? clock64() : 0;
            cl_wait(); // every thread of the cluster finished entry i: its ring space is free
            const long long t4 = prof ? clock64() : 0;
            if (producer) issue(i + 1, 1);
            if (prof) {
                pt[0] += t1 - t0;
                pt[1] += t2 - t1;
                pt[2] += t3 - t2;
                pt[3] += t4 - t3;
                pt[5] += 1;
            }
        } else {
            __syncthreads(); // entry i consumed by every warp of this CTA
            if (producer) issue(i + 1, 1);
            v = open(i + 1);
            stage(v, 0, R);
        }
    }
    if (prof) {
        for (int k = 0; k < 6; ++k) q.prof[rank * 8 + k] = pt[k];
        q.prof[rank * 8 + 6] = clock64() - tlast;
    }
    // no CTA leaves while a peer may still read its slice: the last level ended with a
    // cluster barrier; write the slice back
    for (int i = tid; i < (o1 - o0) * B; i += kT) {
        const int r = i / B, d = i - r * B;
        z[static_cast<int64_t>(q.own[o0 + r]) * B + d] = zs[i];
    }
}

template <int B>
void launch(const Bsr& A, const double* b, double* z, const double* invd, bool fwd, cudaStream_t s)
{
    const BsrStruct& S = *A.st;
    auto kern = fwd ? k_sgs_tile<B, true> : k_sgs_tile<B, false>;
    static const bool prof_on = std::getenv("ED_TILE_PROF") != nullptr;
    static long long* prof = nullptr;
    if (prof_on && !prof) ED_CUDA(cudaMallocManaged(&prof, sizeof(long long) * 16 * 8));
    static bool attr_done[2] = {};
    if (!attr_done[fwd ? 1 : 0]) {
        ED_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, kDynMax));
        ED_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
        attr_done[fwd ? 1 : 0] = true;
    }
    const TileArgs q{fwd ? S.tent.p : S.tent_bwd.p, S.tent_ptr.p, fwd ? S.tent_info.p : S.tent_info_bwd.p,
                     S.thdr.p, S.tcolz.p, A.val.p, S.town.p, S.town_ptr.p, S.tile_cap, prof_on ? prof : nullptr};
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(S.tile_cs, 1, 1);
    cfg.blockDim = dim3(kT, 1, 1);
    cfg.dynamicSmemBytes = static_cast<size_t>(S.tile_cap) + static_cast<size_t>((S.tile_slice + 1) & ~1) * sizeof(double);
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = S.tile_cs;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    ED_CUDA(cudaLaunchKernelEx(&cfg, kern, q, b, z, invd));
    after_launch("k_sgs_tile");
    if (prof_on) {
        static int np = 0;
        ED_CUDA(cudaStreamSynchronize(s));
        if (np++ < 4)
            for (int c = 0; c < S.tile_cs; c += 5) {
                const long long* p = prof + c * 8;
                const double L = p[5] > 0 ? static_cast<double>(p[5]) : 1.0;
                std::fprintf(stderr, "[tile] %s cta %d levels %lld | solve %.0f fence+arrive %.0f open+stage %.0f (open %.0f) wait %.0f | total/level %.0f\n",
                             fwd ? "fwd" : "bwd", c, p[5], p[0] / L, p[1] / L, p[2] / L, p[4] / L, p[3] / L, p[6] / L);
            }
    }
}

} // namespace

int tile_capacity(int slice)
{
    const int zb = ((slice + 1) & ~1) * 8;
    return (kDynMax - zb) & ~15;
}

void sgs_tile(const Bsr& A, const double* b, double* z, const double* invd, bool fwd, cudaStream_t s)
{
    if (A.st->Rb == 1) return launch<1>(A, b, z, invd, fwd, s);
    if (A.st->Rb == 3) return launch<3>(A, b, z, invd, fwd, s);
    throw Error(ED_UNSUPPORTED, "tile sweep: unsupported block size");
}

} // namespace edb
