// Grid-barrier latency on the B200: a persistent kernel (one or two CTAs per
// SM) crosses N barriers; each barrier is a release add on one counter plus
// an acquire spin until every CTA of this round has arrived.  Also the same
// with a little dependent work (an L2 read of a value another CTA wrote).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/gridbar_latency.bin scripts/gridbar_latency.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned ld_acq(const unsigned* p)
{
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void red_rel(unsigned* p, unsigned v)
{
    asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ unsigned atom_add_rel(unsigned* p, unsigned v)
{
    unsigned old;
    asm volatile("atom.add.release.gpu.global.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
    return old;
}
__device__ __forceinline__ unsigned ld_rlx(const unsigned* p)
{
    unsigned v;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_rel(unsigned* p, unsigned v)
{
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// flag barrier: arrivals count on ctr; the last arriver publishes the generation on flag (another line)
__global__ void k_bar2(unsigned* ctr, int nbar, double* buf, int work, int relaxed_poll)
{
    const unsigned G = gridDim.x;
    unsigned* flag = ctr + 32;
    double acc = 0.0;
    for (int b = 0; b < nbar; ++b) {
        if (work && threadIdx.x < 32) {
            const int src = (blockIdx.x + 7 * b + threadIdx.x) % G;
            acc += __ldcg(buf + src * 32 + threadIdx.x);
            buf[blockIdx.x * 32 + threadIdx.x] = acc;
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            const unsigned old = atom_add_rel(ctr, 1u);
            if (old == G * (b + 1) - 1) {
                st_rel(flag, b + 1);
            } else if (relaxed_poll) {
                while (ld_rlx(flag) < static_cast<unsigned>(b + 1)) {
                }
                asm volatile("fence.acq_rel.gpu;" ::: "memory");
            } else {
                while (ld_acq(flag) < static_cast<unsigned>(b + 1)) {
                }
            }
        }
        __syncthreads();
    }
    if (acc == 12345.0) buf[0] = acc;
}

__global__ void k_bar(unsigned* ctr, int nbar, double* buf, int work)
{
    const unsigned G = gridDim.x;
    double acc = 0.0;
    for (int b = 0; b < nbar; ++b) {
        if (work && threadIdx.x < 32) {
            // read a value written by another CTA in the previous round
            const int src = (blockIdx.x + 7 * b + threadIdx.x) % G;
            acc += __ldcg(buf + src * 32 + threadIdx.x);
            buf[blockIdx.x * 32 + threadIdx.x] = acc;
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            red_rel(ctr, 1u);
            const unsigned need = G * (b + 1);
            while (ld_acq(ctr) < need) {
            }
        }
        __syncthreads();
    }
    if (acc == 12345.0) buf[0] = acc;
}

int main()
{
    unsigned* ctr;
    double* buf;
    cudaMalloc(&ctr, 4 * 64);
    cudaMalloc(&buf, 8 * 32 * 4096);
    cudaMemset(buf, 0, 8 * 32 * 4096);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const int nbar = 2000;
    for (int per_sm : {1, 2, 4}) {
        for (int threads : {256, 512}) {
            for (int work : {0, 1}) {
                const int G = 148 * per_sm;
                float best = 1e9;
                for (int rep = 0; rep < 5; ++rep) {
                    cudaMemset(ctr, 0, 4);
                    cudaEventRecord(a);
                    k_bar<<<G, threads>>>(ctr, nbar, buf, work);
                    cudaEventRecord(b);
                    cudaEventSynchronize(b);
                    float ms;
                    cudaEventElapsedTime(&ms, a, b);
                    if (ms < best) best = ms;
                }
                printf("CTAs %4d threads %3d work %d: %.3f us per barrier\n", G, threads, work, best * 1e3 / nbar);
            }
        }
    }
    for (int relaxed : {0, 1}) {
        for (int per_sm : {1, 2}) {
            for (int work : {0, 1}) {
                const int G = 148 * per_sm;
                float best = 1e9;
                for (int rep = 0; rep < 5; ++rep) {
                    cudaMemset(ctr, 0, 4 * 64);
                    cudaEventRecord(a);
                    k_bar2<<<G, 256>>>(ctr, nbar, buf, work, relaxed);
                    cudaEventRecord(b);
                    cudaEventSynchronize(b);
                    float ms;
                    cudaEventElapsedTime(&ms, a, b);
                    if (ms < best) best = ms;
                }
                printf("flag barrier (%s poll) CTAs %4d work %d: %.3f us per barrier\n", relaxed ? "relaxed" : "acquire", G,
                       work, best * 1e3 / nbar);
            }
        }
    }
    cudaError_t e = cudaGetLastError();
    printf("status: %s\n", cudaGetErrorString(e));
    return 0;
}
