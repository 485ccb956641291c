// Cross-SM handoff latency on the B200: two CTAs (on different SMs) bounce a tagged 16-byte word
// {lo | tag, hi | tag} back and forth N times; the time per bounce is one producer -> consumer
// handoff (store becomes visible + the consumer's polling load sees it).  Variants of the load /
// store flavour, idle and with background polling traffic from the other SMs.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/pingpong_latency.bin scripts/pingpong_latency.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int V>
__device__ __forceinline__ void ld2(const unsigned long long* p, unsigned long long& a, unsigned long long& b)
{
    if (V == 0) asm volatile("ld.relaxed.gpu.global.v2.u64 {%0, %1}, [%2];" : "=l"(a), "=l"(b) : "l"(p) : "memory");
    if (V == 1) asm volatile("ld.volatile.global.v2.u64 {%0, %1}, [%2];" : "=l"(a), "=l"(b) : "l"(p) : "memory");
    if (V == 2) asm volatile("ld.global.cg.v2.u64 {%0, %1}, [%2];" : "=l"(a), "=l"(b) : "l"(p) : "memory");
    if (V == 3) asm volatile("ld.global.cv.v2.u64 {%0, %1}, [%2];" : "=l"(a), "=l"(b) : "l"(p) : "memory");
    if (V == 4) { // one 8-byte relaxed load (32-bit payload + tag would fit)
        asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(a) : "l"(p) : "memory");
        b = a;
    }
    if (V == 5) asm volatile("ld.acquire.gpu.global.v2.u64 {%0, %1}, [%2];" : "=l"(a), "=l"(b) : "l"(p) : "memory");
}
template <int V>
__device__ __forceinline__ void st2(unsigned long long* p, unsigned long long a, unsigned long long b)
{
    if (V == 1) asm volatile("st.volatile.global.v2.u64 [%0], {%1, %2};" ::"l"(p), "l"(a), "l"(b) : "memory");
    else if (V == 2 || V == 3) asm volatile("st.global.cg.v2.u64 [%0], {%1, %2};" ::"l"(p), "l"(a), "l"(b) : "memory");
    else if (V == 4) asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(a) : "memory");
    else asm volatile("st.relaxed.gpu.global.v2.u64 [%0], {%1, %2};" ::"l"(p), "l"(a), "l"(b) : "memory");
}

// CTA 0 and CTA `peer` bounce; the other CTAs optionally poll unrelated words (background traffic).
template <int V>
__global__ void k_pingpong(unsigned long long* w, int n, int peer, int background, long long* cycles)
{
    const int me = blockIdx.x;
    if (threadIdx.x != 0 && !(background && me != 0 && me != peer)) return;
    if (me == 0 || me == peer) {
        if (threadIdx.x != 0) return;
        const bool first = me == 0;
        const long long t0 = clock64();
        for (int i = 0; i < n; ++i) {
            const unsigned long long want = 2ull * i + (first ? 2 : 1); // peer waits for odd, CTA 0 for even
            if (first) st2<V>(w, (2ull * i + 1) << 32, (2ull * i + 1) << 32);
            unsigned long long a, b;
            do {
                ld2<V>(w, a, b);
            } while ((a >> 32) != want || (b >> 32) != want);
            if (!first) st2<V>(w, (2ull * i + 2) << 32, (2ull * i + 2) << 32);
        }
        if (first) {
            cycles[0] = clock64() - t0;
            w[2] = 1; // stop the background pollers
        }
        return;
    }
    // background: every thread polls its own words until told to stop
    unsigned long long* mine = w + 64 + 2 * (static_cast<size_t>(me) * blockDim.x + threadIdx.x);
    unsigned long long a, b, stop = 0;
    while (!stop) {
        for (int k = 0; k < 8; ++k) ld2<V>(mine, a, b);
        asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(stop) : "l"(w + 2) : "memory");
    }
}

template <int V>
void run(const char* name, unsigned long long* w, long long* cyc, int n)
{
    for (int background = 0; background < 2; ++background)
        for (int peer : {1, 74, 147}) {
            cudaMemset(w, 0, 64 * 8);
            k_pingpong<V><<<148, background ? 256 : 32>>>(w, n, peer, background, cyc);
            cudaError_t e = cudaDeviceSynchronize();
            if (e != cudaSuccess) {
                std::printf("%s: %s\n", name, cudaGetErrorString(e));
                return;
            }
            std::printf("%-28s peer CTA %3d  background %d  %7.1f ns per handoff\n", name, peer, background,
                        cyc[0] / 1.965 / (2.0 * n));
        }
}

int main()
{
    unsigned long long* w;
    long long* cyc;
    cudaMalloc(&w, (64 + 2 * 148 * 256) * 8);
    cudaMemset(w, 0, (64 + 2 * 148 * 256) * 8);
    cudaMallocManaged(&cyc, 8);
    const int n = 2000;
    run<0>("ld/st.relaxed.gpu v2.u64", w, cyc, n);
    run<1>("ld/st.volatile v2.u64", w, cyc, n);
    run<2>("ld.cg / st.cg v2.u64", w, cyc, n);
    run<3>("ld.cv / st.cg v2.u64", w, cyc, n);
    run<4>("ld/st.relaxed.gpu u64", w, cyc, n);
    run<5>("ld.acquire / st.relaxed v2", w, cyc, n);
    return 0;
}
