// Micro-benchmarks of the cluster hand-off primitives the push sweep is built
// on (B200, sm_100a): round-trip latency between two CTAs of a cluster via
//   (a) st.async + remote mbarrier (complete_tx), waiter try_wait.acquire.cluster
//   (b) st.shared::cluster + fence.release + flag polling (ld.acquire.cluster)
//   (c) barrier.cluster arrive/wait (full cluster of 16)
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/dsl scripts/dsmem_latency.cu && /tmp/dsl
#include <cooperative_groups.h>
#include <cstdint>
#include <cstdio>

namespace cg = cooperative_groups;

__device__ __forceinline__ uint32_t su32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ uint32_t mapa(uint32_t a, int r)
{
    uint32_t o;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(o) : "r"(a), "r"(r));
    return o;
}

template <int MODE>
__global__ void k_pingpong(long long* out, int iters)
{
    __shared__ __align__(8) uint64_t bar[2];
    __shared__ __align__(16) double buf[2];
    __shared__ volatile int flag;
    cg::cluster_group cl = cg::this_cluster();
    const int rank = cl.block_rank();
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar[0])));
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar[1])));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        flag = -1;
    }
    cl.sync();
    if (MODE == 2) {
        long long t0 = clock64();
        for (int i = 0; i < iters; ++i) {
            asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");
            asm volatile("barrier.cluster.wait.aligned;" ::: "memory");
        }
        if (rank == 0 && threadIdx.x == 0) out[2] = (clock64() - t0) / iters;
        return;
    }
    if (threadIdx.x == 0 && rank < 2) {
    const int peer = 1 - rank;
    const uint32_t rbuf = mapa(su32(&buf[0]), peer), rbar = mapa(su32(&bar[0]), peer);
    const uint32_t rflag = mapa(su32((const void*)&flag), peer);
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
        const bool mine = (i & 1) == rank; // rank 0 sends on even i
        if (MODE == 0) {
            if (mine) {
                asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.f64 [%0], %1, [%2];" ::"r"(rbuf),
                             "d"(double(i)), "r"(rbar)
                             : "memory");
            } else {
                const int use = i >> 1; // my barrier's use count
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], 8;" ::"r"(su32(&bar[0])) : "memory");
                asm volatile(
                    "{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n"
                    "@!p bra W_%=;\n}\n" ::"r"(su32(&bar[0])),
                    "r"(use & 1)
                    : "memory");
            }
        } else {
            if (mine) {
                asm volatile("st.shared::cluster.f64 [%0], %1;" ::"r"(rbuf), "d"(double(i)) : "memory");
                asm volatile("fence.release.sync_restrict::shared::cta.cluster;" ::: "memory");
                asm volatile("st.relaxed.cluster.shared::cluster.s32 [%0], %1;" ::"r"(rflag), "r"(i) : "memory");
            } else {
                int v;
                do {
                    asm volatile("ld.acquire.cluster.shared::cta.s32 %0, [%1];" : "=r"(v) : "r"(su32((const void*)&flag)) : "memory");
                } while (v != i);
            }
        }
    }
    if (rank == 0) out[MODE] = (clock64() - t0) / iters;
    (void)rbuf;
    }
    __syncwarp();
    cl.sync();
}

int main()
{
    long long* d;
    cudaMalloc(&d, 64);
    cudaMemset(d, 0, 64);
    long long h[3] = {0, 0, 0};
    for (int mode = 0; mode < 3; ++mode) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(16);
        cfg.blockDim = dim3(mode == 2 ? 256 : 32);
        cudaLaunchAttribute a[1];
        a[0].id = cudaLaunchAttributeClusterDimension;
        a[0].val.clusterDim.x = 16;
        a[0].val.clusterDim.y = 1;
        a[0].val.clusterDim.z = 1;
        cfg.attrs = a;
        cfg.numAttrs = 1;
        auto k = mode == 0 ? k_pingpong<0> : mode == 1 ? k_pingpong<1> : k_pingpong<2>;
        cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        cudaError_t e = cudaLaunchKernelEx(&cfg, k, d, 2000);
        cudaError_t e2 = cudaDeviceSynchronize();
        printf("mode %d launch %s sync %s\n", mode, cudaGetErrorString(e), cudaGetErrorString(e2));
    }
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    printf("one-way hand-off (cycles/iter): st.async+mbarrier %lld | st+fence+flag %lld | cluster barrier(16 CTAs x 256) %lld\n",
           h[0], h[1], h[2]);
    return 0;
}
