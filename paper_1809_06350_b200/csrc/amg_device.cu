// Smoothed-aggregation AMG setup on the GPU; see amg_device.hpp.
#include <cub/cub.cuh>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <numeric>

#include "amg_device.hpp"

namespace edb {

namespace {

// per-thread pinned staging buffer for the power iteration's D2H copies
// (grown, never freed: a cudaFreeHost would synchronise the device under the
// concurrent hierarchy builds)
double* pinned_scratch(int n)
{
    thread_local double* p = nullptr;
    thread_local int cap = 0;
    if (n > cap) {
        if (p) ED_CUDA(cudaFreeHost(p));
        p = nullptr;
        cap = std::max(n, 2 * cap);
        ED_CUDA(cudaMallocHost(reinterpret_cast<void**>(&p), sizeof(double) * cap));
    }
    return p;
}


constexpr int kT = 256;

inline int g1(int64_t n) { return static_cast<int>(std::max<int64_t>(1, (n + kT - 1) / kT)); }

struct Timer {
    bool on = std::getenv("ED_AMG_VERBOSE") != nullptr;
    bool nosync = on && std::atoi(std::getenv("ED_AMG_VERBOSE")) == 2; // host timestamps only
    std::chrono::steady_clock::time_point t = std::chrono::steady_clock::now();
    void lap(cudaStream_t s, const char* what, int lvl, long a, long b)
    {
        if (!on) return;
        if (!nosync) cudaStreamSynchronize(s);
        const auto now = std::chrono::steady_clock::now();
        std::fprintf(stderr, "[amg-dev] L%d %-12s %9.3f s  %ld %ld\n", lvl, what,
                     std::chrono::duration<double>(now - t).count(), a, b);
        t = now;
    }
};

// ---- natural-order copy of a (level-permuted) Bsr -------------------------
__global__ void k_rowlen_nat(const int* __restrict__ rowptr, const int* __restrict__ inv, int n, int* len)
{
    const int I = blockIdx.x * blockDim.x + threadIdx.x;
    if (I >= n) return;
    const int s = inv ? inv[I] : I;
    len[I] = rowptr[s + 1] - rowptr[s];
}

__global__ void k_copy_rows(const int* __restrict__ rp_in, const int* __restrict__ col_in,
                            const double* __restrict__ val_in, const int* __restrict__ inv, int n, int E,
                            const int* __restrict__ rp_out, int* col_out, double* val_out)
{
    const int I = blockIdx.x * blockDim.x + threadIdx.x;
    if (I >= n) return;
    const int s = inv ? inv[I] : I;
    const int k0 = rp_in[s], k1 = rp_in[s + 1], o = rp_out[I];
    for (int k = k0; k < k1; ++k) {
        col_out[o + k - k0] = col_in[k];
        for (int e = 0; e < E; ++e) val_out[static_cast<int64_t>(o + k - k0) * E + e] = val_in[static_cast<int64_t>(k) * E + e];
    }
}

// ---- strength graph (amg.cpp:32-81) ---------------------------------------
template <int B>
__global__ void k_diag_w(const int* __restrict__ rowptr, const int* __restrict__ col, const double* __restrict__ val,
                         int n, double* dw)
{
    const int I = blockIdx.x * blockDim.x + threadIdx.x;
    if (I >= n) return;
    double s = 0.0;
    for (int k = rowptr[I]; k < rowptr[I + 1]; ++k)
        if (col[k] == I) {
            const double* v = val + static_cast<int64_t>(k) * B * B;
#pragma unroll
            for (int e = 0; e < B * B; ++e) s = __dadd_rn(s, __dmul_rn(v[e], v[e]));
        }
    dw[I] = s;
}

// flag: 0 weak, 1 strong, 2 too close to call on the device
template <int B>
__global__ void k_strength(const int* __restrict__ rowptr, const int* __restrict__ col, const double* __restrict__ val,
                           int n, const double* __restrict__ dw, double theta, unsigned char* flag, double* s2out,
                           int* n_amb)
{
    const int I = blockIdx.x * blockDim.x + threadIdx.x;
    if (I >= n) return;
    const double dI = dw[I];
    for (int k = rowptr[I]; k < rowptr[I + 1]; ++k) {
        const int J = col[k];
        unsigned char f = 0;
        if (J != I) {
            const double* v = val + static_cast<int64_t>(k) * B * B;
            double s2 = 0.0;
#pragma unroll
            for (int e = 0; e < B * B; ++e) s2 = __dadd_rn(s2, __dmul_rn(v[e], v[e]));
            s2out[k] = s2;
            const double dJ = dw[J];
            if (dI > 0.0 && dJ > 0.0) {
                const double lhs = sqrt(s2);
                const double rhs = theta * pow(__dmul_rn(dI, dJ), 0.25);
                if (fabs(lhs - rhs) <= 1e-12 * rhs) {
                    f = 2;
                    atomicAdd(n_amb, 1);
                } else {
                    f = lhs > rhs ? 1 : 0;
                }
            }
        }
        flag[k] = f;
    }
}

__global__ void k_symmetrize(const int* __restrict__ rowptr, const int* __restrict__ col,
                             const unsigned char* __restrict__ flag, int n, unsigned char* sym, int* cnt)
{
    const int I = blockIdx.x * blockDim.x + threadIdx.x;
    if (I >= n) return;
    int c = 0;
    for (int k = rowptr[I]; k < rowptr[I + 1]; ++k) {
        const int J = col[k];
        unsigned char s = 0;
        if (J != I) {
            s = flag[k] == 1;
            if (!s) {
                int lo = rowptr[J], hi = rowptr[J + 1];
                while (lo < hi) {
                    const int mid = lo + ((hi - lo) >> 1);
                    if (col[mid] < I) lo = mid + 1;
                    else hi = mid;
                }
                if (lo < rowptr[J + 1] && col[lo] == I) s = flag[lo] == 1;
            }
        }
        sym[k] = s;
        c += s;
    }
    cnt[I] = c;
}

// ---- elementwise helpers --------------------------------------------------
template <int B>
__global__ void k_invdiag(const int* __restrict__ rowptr, const int* __restrict__ col, const double* __restrict__ val,
                          int n, double* invd)
{
    const int I = blockIdx.x * blockDim.x + threadIdx.x;
    if (I >= n) return;
    double d[B];
#pragma unroll
    for (int r = 0; r < B; ++r) d[r] = 0.0;
    for (int k = rowptr[I]; k < rowptr[I + 1]; ++k)
        if (col[k] == I) {
#pragma unroll
            for (int r = 0; r < B; ++r) d[r] = val[static_cast<int64_t>(k) * B * B + r * B + r];
        }
#pragma unroll
    for (int r = 0; r < B; ++r) invd[static_cast<int64_t>(I) * B + r] = d[r] != 0.0 ? 1.0 / d[r] : 1.0;
}

// row-sequential y = A x (csr.cpp:11-18 order, no FMA): one thread per
// scalar row (the scalar CSR row of a block row walks its blocks in column
// order, entries d = 0..CB-1 inside each block)
template <int RB, int CB>
__global__ void k_spmv_seq(const int* __restrict__ rowptr, const int* __restrict__ col, const double* __restrict__ val,
                           int n, const double* __restrict__ x, double* y)
{
    const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const int I = static_cast<int>(t / RB), r = static_cast<int>(t % RB);
    if (I >= n) return;
    double acc = 0.0;
    for (int k = rowptr[I]; k < rowptr[I + 1]; ++k) {
        const int c = col[k];
        const double* v = val + static_cast<int64_t>(k) * RB * CB + r * CB;
#pragma unroll
        for (int d = 0; d < CB; ++d) acc = __dadd_rn(acc, __dmul_rn(v[d], x[static_cast<int64_t>(c) * CB + d]));
    }
    y[t] = acc;
}

__global__ void k_mul_vec(double* w, const double* __restrict__ s, int64_t n)
{
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < n) w[i] = __dmul_rn(w[i], s[i]);
}

__global__ void k_scale_into(double* v, const double* __restrict__ w, double s, int64_t n)
{
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < n) v[i] = __dmul_rn(w[i], s);
}

// csr_scale_rows (csr.cpp:200-205): val *= s[row]
template <int RB, int CB>
__global__ void k_scale_rows(const int* __restrict__ rowptr, double* val, int n, const double* __restrict__ s)
{
    const int I = blockIdx.x * blockDim.x + threadIdx.x;
    if (I >= n) return;
    for (int k = rowptr[I]; k < rowptr[I + 1]; ++k)
#pragma unroll
        for (int r = 0; r < RB; ++r)
#pragma unroll
            for (int d = 0; d < CB; ++d)
                val[static_cast<int64_t>(k) * RB * CB + r * CB + d] =
                    __dmul_rn(val[static_cast<int64_t>(k) * RB * CB + r * CB + d], s[static_cast<int64_t>(I) * RB + r]);
}

// ---- SpGEMM (csr_matmul, csr.cpp:132-166) ----------------------------------
__global__ void k_cand_count(const int* __restrict__ arp, const int* __restrict__ acol, const int* __restrict__ brp,
                             int n, int64_t* cnt)
{
    const int I = blockIdx.x * blockDim.x + threadIdx.x;
    if (I >= n) return;
    int64_t c = 0;
    for (int k = arp[I]; k < arp[I + 1]; ++k) c += brp[acol[k] + 1] - brp[acol[k]];
    cnt[I] = c;
}

__global__ void k_cand_fill(const int* __restrict__ arp, const int* __restrict__ acol, const int* __restrict__ brp,
                            const int* __restrict__ bcol, int r0, int r1, const int* __restrict__ seg, int* keys)
{
    const int I = r0 + blockIdx.x * blockDim.x + threadIdx.x;
    if (I >= r1) return;
    int o = seg[I - r0];
    for (int k = arp[I]; k < arp[I + 1]; ++k) {
        const int K = acol[k];
        for (int kb = brp[K]; kb < brp[K + 1]; ++kb) keys[o++] = bcol[kb];
    }
}

__global__ void k_unique_count(const int* __restrict__ keys, const int* __restrict__ seg, int nseg, int* ucnt)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= nseg) return;
    int c = 0;
    for (int k = seg[i]; k < seg[i + 1]; ++k) c += (k == seg[i] || keys[k] != keys[k - 1]);
    ucnt[i] = c;
}

__global__ void k_unique_write(const int* __restrict__ keys, const int* __restrict__ seg, int nseg,
                               const int* __restrict__ uoff, int* out)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= nseg) return;
    int o = uoff[i];
    for (int k = seg[i]; k < seg[i + 1]; ++k)
        if (k == seg[i] || keys[k] != keys[k - 1]) out[o++] = keys[k];
}

// One thread per scalar row (I, c) of C: every product a*b is added to its
// C entry in (A column, B column) traversal order, mul and add rounded
// separately -- the order and rounding of csr_matmul.
template <int RA, int KA, int CB>
__global__ void k_spgemm_numeric(const int* __restrict__ arp, const int* __restrict__ acol,
                                 const double* __restrict__ aval, const int* __restrict__ brp,
                                 const int* __restrict__ bcol, const double* __restrict__ bval,
                                 const int* __restrict__ crp, const int* __restrict__ ccol, double* cval, int n)
{
    const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const int I = static_cast<int>(t / RA), c = static_cast<int>(t % RA);
    if (I >= n) return;
    const int c0 = crp[I], c1 = crp[I + 1];
    for (int k = arp[I]; k < arp[I + 1]; ++k) {
        const int K = acol[k];
        const int b0 = brp[K], b1 = brp[K + 1];
        if (b0 == b1) continue;
        // position of B row K's first column in C row I, then advance monotonically
        int lo = c0, hi = c1;
        const int j0 = bcol[b0];
        while (lo < hi) {
            const int mid = lo + ((hi - lo) >> 1);
            if (ccol[mid] < j0) lo = mid + 1;
            else hi = mid;
        }
#pragma unroll
        for (int d = 0; d < KA; ++d) {
            const double a = aval[static_cast<int64_t>(k) * RA * KA + c * KA + d];
            int pos = lo;
            for (int kb = b0; kb < b1; ++kb) {
                const int J = bcol[kb];
                while (ccol[pos] < J) ++pos;
                const double* bv = bval + static_cast<int64_t>(kb) * KA * CB + d * CB;
                double* cv = cval + static_cast<int64_t>(pos) * RA * CB + c * CB;
#pragma unroll
                for (int e = 0; e < CB; ++e) cv[e] = __dadd_rn(cv[e], __dmul_rn(a, bv[e]));
            }
        }
    }
}

// ---- warp-per-row variants for long rows (coarse, dense RAP levels) -------
__global__ void k_cand_fill_warp(const int* __restrict__ arp, const int* __restrict__ acol,
                                 const int* __restrict__ brp, const int* __restrict__ bcol, int r0, int r1,
                                 const int* __restrict__ seg, int* keys)
{
    const int64_t w = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    const int I = r0 + static_cast<int>(w);
    if (I >= r1) return;
    int o = seg[I - r0];
    for (int k = arp[I]; k < arp[I + 1]; ++k) {
        const int K = acol[k];
        const int b0 = brp[K], b1 = brp[K + 1];
        for (int kb = b0 + lane; kb < b1; kb += 32) keys[o + kb - b0] = bcol[kb];
        o += b1 - b0;
    }
}

__global__ void k_unique_count_warp(const int* __restrict__ keys, const int* __restrict__ seg, int nseg, int* ucnt)
{
    const int64_t w = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (w >= nseg) return;
    const int a = seg[w], b = seg[w + 1];
    int c = 0;
    for (int k = a + lane; k < b; k += 32) c += (k == a || keys[k] != keys[k - 1]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    if (lane == 0) ucnt[w] = c;
}

__global__ void k_unique_write_warp(const int* __restrict__ keys, const int* __restrict__ seg, int nseg,
                                    const int* __restrict__ uoff, int* out)
{
    const int64_t w = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (w >= nseg) return;
    const int a = seg[w], b = seg[w + 1];
    int o = uoff[w];
    for (int base = a; base < b; base += 32) {
        const int k = base + lane;
        const bool first = k < b && (k == a || keys[k] != keys[k - 1]);
        const unsigned m = __ballot_sync(0xffffffffu, first);
        if (first) out[o + __popc(m & ((1u << lane) - 1u))] = keys[k];
        o += __popc(m);
    }
}

// One warp per scalar row (I, c): the A row is walked in order (K, d); the
// entries of B row K are split across lanes (distinct C columns inside one B
// row), and __syncwarp orders consecutive K steps, so every C entry still
// receives its products in csr_matmul's traversal order.
constexpr int kNumWarpT = 128;   // threads per CTA of the warp-per-row numeric kernel
constexpr int kNumWarps = kNumWarpT / 32;
constexpr int kRowCache = 256;   // C row blocks accumulated in shared memory

template <int RA, int KA, int CB>
__global__ void __launch_bounds__(kNumWarpT) k_spgemm_numeric_warp(
    const int* __restrict__ arp, const int* __restrict__ acol, const double* __restrict__ aval,
    const int* __restrict__ brp, const int* __restrict__ bcol, const double* __restrict__ bval,
    const int* __restrict__ crp, const int* __restrict__ ccol, double* cval, int n)
{
    // rows of up to kRowCache blocks keep their column list and their
    // accumulators (component c) in shared memory: the binary searches and the
    // read-modify-writes stay on chip; the row is written out once at the end
    __shared__ int s_cols[kNumWarps][kRowCache];
    __shared__ double s_acc[kNumWarps][kRowCache * CB];
    const int64_t w = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int I = static_cast<int>(w / RA), c = static_cast<int>(w % RA);
    if (I >= n) return;
    const int c0 = crp[I], c1 = crp[I + 1], nc = c1 - c0;
    const bool cached = nc <= kRowCache;
    const int* cc = cached ? s_cols[wib] : ccol + c0;
    if (cached) {
        for (int t = lane; t < nc; t += 32) s_cols[wib][t] = ccol[c0 + t];
        for (int t = lane; t < nc * CB; t += 32) s_acc[wib][t] = 0.0; // C is zero-initialised
        __syncwarp();
    }
    for (int k = arp[I]; k < arp[I + 1]; ++k) {
        const int K = acol[k];
        const int b0 = brp[K], b1 = brp[K + 1];
        for (int kb = b0 + lane; kb < b1; kb += 32) {
            const int J = bcol[kb];
            int lo = 0, hi = nc;
            while (lo < hi) {
                const int mid = lo + ((hi - lo) >> 1);
                if (cc[mid] < J) lo = mid + 1;
                else hi = mid;
            }
            double* cv = cached ? s_acc[wib] + lo * CB : cval + static_cast<int64_t>(c0 + lo) * RA * CB + c * CB;
#pragma unroll
            for (int d = 0; d < KA; ++d) {
                const double a = aval[static_cast<int64_t>(k) * RA * KA + c * KA + d];
                const double* bv = bval + static_cast<int64_t>(kb) * KA * CB + d * CB;
#pragma unroll
                for (int e = 0; e < CB; ++e) cv[e] = __dadd_rn(cv[e], __dmul_rn(a, bv[e]));
            }
        }
        __syncwarp();
    }
    if (cached)
        for (int t = lane; t < nc * CB; t += 32)
            cval[static_cast<int64_t>(c0 + t / CB) * RA * CB + c * CB + t % CB] = s_acc[wib][t];
}

// ---- csr_add (csr.cpp:168-198) on block rows -------------------------------
__global__ void k_add_count(const int* __restrict__ arp, const int* __restrict__ acol, const int* __restrict__ brp,
                            const int* __restrict__ bcol, int n, int* cnt)
{
    const int I = blockIdx.x * blockDim.x + threadIdx.x;
    if (I >= n) return;
    int ka = arp[I], kb = brp[I], c = 0;
    const int ea = arp[I + 1], eb = brp[I + 1];
    while (ka < ea || kb < eb) {
        if (kb >= eb || (ka < ea && acol[ka] < bcol[kb])) ++ka;
        else if (ka >= ea || bcol[kb] < acol[ka]) ++kb;
        else {
            ++ka;
            ++kb;
        }
        ++c;
    }
    cnt[I] = c;
}

template <int E>
__global__ void k_add_fill(const int* __restrict__ arp, const int* __restrict__ acol, const double* __restrict__ aval,
                           const int* __restrict__ brp, const int* __restrict__ bcol, const double* __restrict__ bval,
                           int n, double alpha, double beta, const int* __restrict__ crp, int* ccol, double* cval)
{
    const int I = blockIdx.x * blockDim.x + threadIdx.x;
    if (I >= n) return;
    int ka = arp[I], kb = brp[I], o = crp[I];
    const int ea = arp[I + 1], eb = brp[I + 1];
    while (ka < ea || kb < eb) {
        double* cv = cval + static_cast<int64_t>(o) * E;
        if (kb >= eb || (ka < ea && acol[ka] < bcol[kb])) {
            ccol[o] = acol[ka];
#pragma unroll
            for (int e = 0; e < E; ++e) cv[e] = __dmul_rn(alpha, aval[static_cast<int64_t>(ka) * E + e]);
            ++ka;
        } else if (ka >= ea || bcol[kb] < acol[ka]) {
            ccol[o] = bcol[kb];
#pragma unroll
            for (int e = 0; e < E; ++e) cv[e] = __dmul_rn(beta, bval[static_cast<int64_t>(kb) * E + e]);
            ++kb;
        } else {
            ccol[o] = acol[ka];
#pragma unroll
            for (int e = 0; e < E; ++e)
                cv[e] = __dadd_rn(__dmul_rn(alpha, aval[static_cast<int64_t>(ka) * E + e]),
                                  __dmul_rn(beta, bval[static_cast<int64_t>(kb) * E + e]));
            ++ka;
            ++kb;
        }
        ++o;
    }
}

// ---- transpose (csr.cpp:39-57) ---------------------------------------------
__global__ void k_row_of_block(const int* __restrict__ rowptr, int n, int* row)
{
    const int I = blockIdx.x * blockDim.x + threadIdx.x;
    if (I >= n) return;
    for (int k = rowptr[I]; k < rowptr[I + 1]; ++k) row[k] = I;
}

__global__ void k_col_hist(const int* __restrict__ col, int64_t nnz, int* cnt)
{
    const int64_t k = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (k < nnz) atomicAdd(cnt + col[k], 1);
}

template <int RB, int CB>
__global__ void k_transpose_fill(const int* __restrict__ perm, const int* __restrict__ row_of,
                                 const double* __restrict__ val, int64_t nnz, int* tcol, double* tval)
{
    const int64_t k = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (k >= nnz) return;
    const int src = perm[k];
    tcol[k] = row_of[src];
#pragma unroll
    for (int r = 0; r < RB; ++r)
#pragma unroll
        for (int c = 0; c < CB; ++c)
            tval[k * RB * CB + c * RB + r] = val[static_cast<int64_t>(src) * RB * CB + r * CB + c];
}

// gather natural rows into level order: stored row s <- natural row perm[s]
__global__ void k_gather_rows(const int* __restrict__ rp_nat, const double* __restrict__ val_nat,
                              const int* __restrict__ perm, int n, int E, const int* __restrict__ rp_out, double* val_out)
{
    const int s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= n) return;
    const int I = perm ? perm[s] : s;
    const int k0 = rp_nat[I], len = rp_nat[I + 1] - k0, o = rp_out[s];
    for (int k = 0; k < len; ++k)
        for (int e = 0; e < E; ++e) val_out[static_cast<int64_t>(o + k) * E + e] = val_nat[static_cast<int64_t>(k0 + k) * E + e];
}

// ---------------------------------------------------------------------------
// host orchestration

void exclusive_scan_host(const std::vector<int>& cnt, std::vector<int>& off)
{
    off.assign(cnt.size() + 1, 0);
    int64_t acc = 0;
    for (size_t i = 0; i < cnt.size(); ++i) {
        acc += cnt[i];
        if (acc >= (1LL << 31)) throw Error(ED_UNSUPPORTED, "block count exceeds int32");
        off[i + 1] = static_cast<int>(acc);
    }
}

DBsr natural_copy(const Bsr& A, cudaStream_t s)
{
    const BsrStruct& S = *A.st;
    DBsr N;
    N.nbr = S.nbr;
    N.nbc = S.nbc;
    N.Rb = S.Rb;
    N.Cb = S.Cb;
    N.nnzb = S.nnzb;
    const int n = S.nbr, E = S.Rb * S.Cb;
    DevArray<int> len(n);
    k_rowlen_nat<<<g1(n), kT, 0, s>>>(S.rowptr.p, S.inv.p, n, len.p);
    after_launch("k_rowlen_nat");
    std::vector<int> off;
    exclusive_scan_host(len.to_host(s), off);
    N.rowptr.upload(off, s);
    N.col.alloc(N.nnzb);
    N.val.alloc(N.nnzb * E);
    k_copy_rows<<<g1(n), kT, 0, s>>>(S.rowptr.p, S.col.p, A.val.p, S.inv.p, n, E, N.rowptr.p, N.col.p, N.val.p);
    after_launch("k_copy_rows");
    ED_CUDA(cudaStreamSynchronize(s));
    return N;
}


// ---- symbolic SpGEMM with a per-warp column bitmap in shared memory --------
// Warp per block row of C: the lanes mark the columns of every B row the A
// row touches (atomicOr into the warp's bitmap), then PASS 0 counts the set
// bits of the touched word range, PASS 1 writes the columns in ascending
// order (popcount prefix over the words).  The touched range is cleared for
// the next row.  Same pattern as csr_matmul's sorted rows (csr.cpp:132-166).
template <int PASS>
__global__ void k_sym_bitmap(const int* __restrict__ arp, const int* __restrict__ acol, const int* __restrict__ brp,
                             const int* __restrict__ bcol, int n, int words, int* cnt, const int* __restrict__ crp,
                             int* ccol)
{
    extern __shared__ unsigned int bm_smem[];
    const int wib = threadIdx.x >> 5, lane = threadIdx.x & 31;
    unsigned int* bm = bm_smem + static_cast<size_t>(wib) * words;
    for (int i = lane; i < words; i += 32) bm[i] = 0u;
    __syncwarp();
    const int nw = (gridDim.x * blockDim.x) >> 5;
    for (int I = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; I < n; I += nw) {
        int lo = words, hi = -1;
        for (int k = arp[I]; k < arp[I + 1]; ++k) {
            const int K = acol[k];
            for (int kb = brp[K] + lane; kb < brp[K + 1]; kb += 32) {
                const int c = bcol[kb];
                atomicOr(&bm[c >> 5], 1u << (c & 31));
                lo = min(lo, c >> 5);
                hi = max(hi, c >> 5);
            }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            lo = min(lo, __shfl_xor_sync(0xffffffffu, lo, o));
            hi = max(hi, __shfl_xor_sync(0xffffffffu, hi, o));
        }
        __syncwarp();
        if (PASS == 0) {
            int c = 0;
            for (int w = lo + lane; w <= hi; w += 32) {
                c += __popc(bm[w]);
                bm[w] = 0u;
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
            if (lane == 0) cnt[I] = c;
        } else {
            int out = crp[I];
            for (int w0 = lo; w0 <= hi; w0 += 32) {
                const int w = w0 + lane;
                unsigned int bits = w <= hi ? bm[w] : 0u;
                const int pc = __popc(bits);
                int incl = pc;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const int v = __shfl_up_sync(0xffffffffu, incl, o);
                    if (lane >= o) incl += v;
                }
                int at = out + incl - pc;
                while (bits) {
                    const int b = __ffs(bits) - 1;
                    ccol[at++] = w * 32 + b;
                    bits &= bits - 1;
                }
                if (w <= hi) bm[w] = 0u;
                out += __shfl_sync(0xffffffffu, incl, 31);
            }
        }
        __syncwarp();
    }
}

// symbolic + numeric C = A B
DBsr spgemm(const DBsr& A, const DBsr& B, cudaStream_t s)
{
    if (A.Cb != B.Rb || A.nbc != B.nbr) throw Error(ED_INVALID_ARGUMENT, "spgemm: shape mismatch");
    DBsr C;
    C.nbr = A.nbr;
    C.nbc = B.nbc;
    C.Rb = A.Rb;
    C.Cb = B.Cb;
    const int n = A.nbr;
    const int words = (B.nbc + 31) / 32;
    int64_t tot_cand = 0; // products a*b (numeric kernel choice)
    static const bool no_bitmap = std::getenv("ED_SPGEMM_SORT") != nullptr;
    if (!no_bitmap && n > 0 && static_cast<int64_t>(words) * 4 <= 96 * 1024) {
        // symbolic via per-warp bitmaps: count, device scan, fill
        const int wpb = std::max(1, std::min(8, static_cast<int>((96 * 1024) / (static_cast<int64_t>(words) * 4))));
        const size_t smem = static_cast<size_t>(wpb) * words * 4;
        static bool attr = false;
        if (!attr) {
            ED_CUDA(cudaFuncSetAttribute(k_sym_bitmap<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024));
            ED_CUDA(cudaFuncSetAttribute(k_sym_bitmap<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024));
            attr = true;
        }
        const int blocks = static_cast<int>(std::min<int64_t>((n + wpb - 1) / wpb, 148LL * 16));
        DevArray<int> cnt(n + 1);
        DevArray<int64_t> ccand(n), ctot(1);
        k_sym_bitmap<0><<<blocks, 32 * wpb, smem, s>>>(A.rowptr.p, A.col.p, B.rowptr.p, B.col.p, n, words, cnt.p,
                                                       nullptr, nullptr);
        after_launch("k_sym_bitmap");
        k_cand_count<<<g1(n), kT, 0, s>>>(A.rowptr.p, A.col.p, B.rowptr.p, n, ccand.p);
        after_launch("k_cand_count");
        C.rowptr.alloc(n + 1);
        size_t tb = 0, tb2 = 0;
        cub::DeviceScan::ExclusiveSum(nullptr, tb, cnt.p, C.rowptr.p, n + 1, s);
        cub::DeviceReduce::Sum(nullptr, tb2, ccand.p, ctot.p, n, s);
        DevArray<unsigned char> tmp(std::max<size_t>(std::max(tb, tb2), 1));
        ED_CUDA(cudaMemsetAsync(cnt.p + n, 0, sizeof(int), s));
        ED_CUDA(cub::DeviceScan::ExclusiveSum(tmp.p, tb, cnt.p, C.rowptr.p, n + 1, s));
        int total = 0;
        ED_CUDA(cudaMemcpyAsync(&total, C.rowptr.p + n, sizeof(int), cudaMemcpyDeviceToHost, s));
        ED_CUDA(cub::DeviceReduce::Sum(tmp.p, tb2, ccand.p, ctot.p, n, s));
        ED_CUDA(cudaMemcpyAsync(&tot_cand, ctot.p, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
        ED_CUDA(cudaStreamSynchronize(s));
        C.nnzb = total;
        C.col.alloc(std::max<int64_t>(C.nnzb, 1));
        k_sym_bitmap<1><<<blocks, 32 * wpb, smem, s>>>(A.rowptr.p, A.col.p, B.rowptr.p, B.col.p, n, words, nullptr,
                                                       C.rowptr.p, C.col.p);
        after_launch("k_sym_bitmap");
    } else {
        DevArray<int64_t> cnt(n);
        k_cand_count<<<g1(n), kT, 0, s>>>(A.rowptr.p, A.col.p, B.rowptr.p, n, cnt.p);
        after_launch("k_cand_count");
        const std::vector<int64_t> hc = cnt.to_host(s);
        cnt.release();
        for (const int64_t v : hc) tot_cand += v;
        std::vector<int> ucnt_all(n, 0);
        std::vector<DevArray<int>> chunk_cols;
        std::vector<int64_t> chunk_tot;
        const int64_t kChunk = 1LL << 28; // candidates per chunk (1 GiB of int keys)
        int r0 = 0;
        while (r0 < n) {
            int r1 = r0;
            int64_t tot = 0;
            while (r1 < n && (r1 == r0 || tot + hc[r1] <= kChunk)) tot += hc[r1++];
            if (tot >= (1LL << 31)) throw Error(ED_UNSUPPORTED, "spgemm: row candidates exceed int32");
            const int nseg = r1 - r0;
            std::vector<int> seg(nseg + 1, 0);
            for (int i = 0; i < nseg; ++i) seg[i + 1] = seg[i] + static_cast<int>(hc[r0 + i]);
            DevArray<int> dseg;
            dseg.upload(seg, s);
            DevArray<int> keys(std::max<int64_t>(tot, 1)), sorted(std::max<int64_t>(tot, 1));
            const bool wide = tot > 256LL * nseg; // long rows: a warp per row
            if (wide)
                k_cand_fill_warp<<<g1(32LL * nseg), kT, 0, s>>>(A.rowptr.p, A.col.p, B.rowptr.p, B.col.p, r0, r1, dseg.p,
                                                               keys.p);
            else
                k_cand_fill<<<g1(nseg), kT, 0, s>>>(A.rowptr.p, A.col.p, B.rowptr.p, B.col.p, r0, r1, dseg.p, keys.p);
            after_launch("k_cand_fill");
            size_t tb = 0;
            cub::DeviceSegmentedSort::SortKeys(nullptr, tb, keys.p, sorted.p, static_cast<int>(tot), nseg, dseg.p,
                                               dseg.p + 1, s);
            DevArray<unsigned char> tmp(std::max<size_t>(tb, 1));
            ED_CUDA(cub::DeviceSegmentedSort::SortKeys(tmp.p, tb, keys.p, sorted.p, static_cast<int>(tot), nseg, dseg.p,
                                                       dseg.p + 1, s));
            after_launch("cub_segmented_sort");
            keys.release();
            DevArray<int> uc(nseg);
            if (wide)
                k_unique_count_warp<<<g1(32LL * nseg), kT, 0, s>>>(sorted.p, dseg.p, nseg, uc.p);
            else
                k_unique_count<<<g1(nseg), kT, 0, s>>>(sorted.p, dseg.p, nseg, uc.p);
            after_launch("k_unique_count");
            const std::vector<int> huc = uc.to_host(s);
            std::vector<int> uoff;
            exclusive_scan_host(huc, uoff);
            DevArray<int> duoff;
            duoff.upload(uoff, s);
            DevArray<int> cols(std::max(uoff[nseg], 1));
            if (wide)
                k_unique_write_warp<<<g1(32LL * nseg), kT, 0, s>>>(sorted.p, dseg.p, nseg, duoff.p, cols.p);
            else
                k_unique_write<<<g1(nseg), kT, 0, s>>>(sorted.p, dseg.p, nseg, duoff.p, cols.p);
            after_launch("k_unique_write");
            for (int i = 0; i < nseg; ++i) ucnt_all[r0 + i] = huc[i];
            chunk_tot.push_back(uoff[nseg]);
            chunk_cols.push_back(std::move(cols));
            ED_CUDA(cudaStreamSynchronize(s));
            r0 = r1;
        }
        std::vector<int> rp;
        exclusive_scan_host(ucnt_all, rp);
        C.nnzb = rp[n];
        C.rowptr.upload(rp, s);
        C.col.alloc(std::max<int64_t>(C.nnzb, 1));
        int64_t o = 0;
        for (size_t i = 0; i < chunk_cols.size(); ++i) {
            if (chunk_tot[i])
                ED_CUDA(cudaMemcpyAsync(C.col.p + o, chunk_cols[i].p, chunk_tot[i] * sizeof(int), cudaMemcpyDeviceToDevice, s));
            o += chunk_tot[i];
        }
    }
    const int E = C.Rb * C.Cb;
    C.val.alloc(std::max<int64_t>(C.nnzb * E, 1));
    C.val.zero(s);
    const int64_t threads = static_cast<int64_t>(n) * A.Rb;
    const bool wide_rows = tot_cand > 256LL * std::max(n, 1);
    if (A.Rb == 3 && A.Cb == 3 && B.Cb == 3) {
        if (wide_rows)
            k_spgemm_numeric_warp<3, 3, 3><<<static_cast<unsigned>((32 * threads + kNumWarpT - 1) / kNumWarpT), kNumWarpT, 0, s>>>(A.rowptr.p, A.col.p, A.val.p, B.rowptr.p,
                                                                          B.col.p, B.val.p, C.rowptr.p, C.col.p,
                                                                          C.val.p, n);
        else
            k_spgemm_numeric<3, 3, 3><<<g1(threads), kT, 0, s>>>(A.rowptr.p, A.col.p, A.val.p, B.rowptr.p, B.col.p,
                                                                 B.val.p, C.rowptr.p, C.col.p, C.val.p, n);
    } else if (A.Rb == 1 && A.Cb == 1 && B.Cb == 1) {
        if (wide_rows)
            k_spgemm_numeric_warp<1, 1, 1><<<static_cast<unsigned>((32 * threads + kNumWarpT - 1) / kNumWarpT), kNumWarpT, 0, s>>>(A.rowptr.p, A.col.p, A.val.p, B.rowptr.p,
                                                                          B.col.p, B.val.p, C.rowptr.p, C.col.p,
                                                                          C.val.p, n);
        else
            k_spgemm_numeric<1, 1, 1><<<g1(threads), kT, 0, s>>>(A.rowptr.p, A.col.p, A.val.p, B.rowptr.p, B.col.p,
                                                                 B.val.p, C.rowptr.p, C.col.p, C.val.p, n);
    } else {
        throw Error(ED_UNSUPPORTED, "spgemm: unsupported block shape");
    }
    after_launch("k_spgemm_numeric");
    ED_CUDA(cudaStreamSynchronize(s));
    return C;
}

DBsr add(const DBsr& A, const DBsr& B, double alpha, double beta, cudaStream_t s)
{
    DBsr C;
    C.nbr = A.nbr;
    C.nbc = A.nbc;
    C.Rb = A.Rb;
    C.Cb = A.Cb;
    const int n = A.nbr;
    DevArray<int> cnt(n);
    k_add_count<<<g1(n), kT, 0, s>>>(A.rowptr.p, A.col.p, B.rowptr.p, B.col.p, n, cnt.p);
    after_launch("k_add_count");
    std::vector<int> rp;
    exclusive_scan_host(cnt.to_host(s), rp);
    C.nnzb = rp[n];
    C.rowptr.upload(rp, s);
    C.col.alloc(std::max<int64_t>(C.nnzb, 1));
    const int E = C.Rb * C.Cb;
    C.val.alloc(std::max<int64_t>(C.nnzb * E, 1));
    if (E == 9)
        k_add_fill<9><<<g1(n), kT, 0, s>>>(A.rowptr.p, A.col.p, A.val.p, B.rowptr.p, B.col.p, B.val.p, n, alpha, beta,
                                           C.rowptr.p, C.col.p, C.val.p);
    else
        k_add_fill<1><<<g1(n), kT, 0, s>>>(A.rowptr.p, A.col.p, A.val.p, B.rowptr.p, B.col.p, B.val.p, n, alpha, beta,
                                           C.rowptr.p, C.col.p, C.val.p);
    after_launch("k_add_fill");
    ED_CUDA(cudaStreamSynchronize(s));
    return C;
}

DBsr transpose(const DBsr& P, cudaStream_t s)
{
    DBsr R;
    R.nbr = P.nbc;
    R.nbc = P.nbr;
    R.Rb = P.Cb;
    R.Cb = P.Rb;
    R.nnzb = P.nnzb;
    const int64_t nnz = P.nnzb;
    DevArray<int> row_of(std::max<int64_t>(nnz, 1)), idx(std::max<int64_t>(nnz, 1)), keys_out(std::max<int64_t>(nnz, 1)),
        perm(std::max<int64_t>(nnz, 1));
    k_row_of_block<<<g1(P.nbr), kT, 0, s>>>(P.rowptr.p, P.nbr, row_of.p);
    after_launch("k_row_of_block");
    std::vector<int> iota(nnz);
    std::iota(iota.begin(), iota.end(), 0);
    idx.upload(iota, s);
    int bits = 1;
    while ((1LL << bits) < R.nbr + 1) ++bits;
    size_t tb = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, tb, P.col.p, keys_out.p, idx.p, perm.p, static_cast<int>(nnz), 0, bits, s);
    DevArray<unsigned char> tmp(std::max<size_t>(tb, 1));
    ED_CUDA(cub::DeviceRadixSort::SortPairs(tmp.p, tb, P.col.p, keys_out.p, idx.p, perm.p, static_cast<int>(nnz), 0, bits,
                                            s)); // stable: equal columns keep ascending source rows
    after_launch("cub_radix_sort");
    DevArray<int> cnt(R.nbr);
    cnt.zero(s);
    k_col_hist<<<g1(nnz), kT, 0, s>>>(P.col.p, nnz, cnt.p);
    after_launch("k_col_hist");
    std::vector<int> rp;
    exclusive_scan_host(cnt.to_host(s), rp);
    R.rowptr.upload(rp, s);
    R.col.alloc(std::max<int64_t>(nnz, 1));
    R.val.alloc(std::max<int64_t>(nnz * P.Rb * P.Cb, 1));
    if (P.Rb == 3 && P.Cb == 3)
        k_transpose_fill<3, 3><<<g1(nnz), kT, 0, s>>>(perm.p, row_of.p, P.val.p, nnz, R.col.p, R.val.p);
    else
        k_transpose_fill<1, 1><<<g1(nnz), kT, 0, s>>>(perm.p, row_of.p, P.val.p, nnz, R.col.p, R.val.p);
    after_launch("k_transpose_fill");
    ED_CUDA(cudaStreamSynchronize(s));
    return R;
}

HostCsr to_host_csr(const DBsr& M, cudaStream_t s)
{
    Bsr tmp;
    auto st = std::make_shared<BsrStruct>();
    st->Rb = M.Rb;
    st->Cb = M.Cb;
    st->nbr = M.nbr;
    st->nbc = M.nbc;
    st->nnzb = M.nnzb;
    st->h_rowptr = M.rowptr.to_host(s);
    std::vector<int> c = M.col.to_host(s);
    c.resize(M.nnzb);
    st->h_col = c;
    tmp.st = st;
    tmp.val.copy_from(M.val, s);
    return bsr_to_csr(tmp, s);
}

DBsr upload_block(const HostCsr& a, int Rb, int Cb, cudaStream_t s)
{
    const BlockPattern pat = block_pattern_of_csr(a, Rb, Cb);
    const std::vector<double> v = block_values_of_csr(a, pat, Rb, Cb);
    DBsr M;
    M.nbr = pat.nbr;
    M.nbc = pat.nbc;
    M.Rb = Rb;
    M.Cb = Cb;
    M.nnzb = pat.nnzb();
    std::vector<int> rp(pat.rowptr.begin(), pat.rowptr.end());
    M.rowptr.upload(rp, s);
    M.col.upload(pat.col, s);
    M.val.upload(v, s);
    ED_CUDA(cudaStreamSynchronize(s));
    return M;
}

} // namespace

Bsr bsr_from_dbsr(DBsr&& m, bool leveled, cudaStream_t s, LevelCache* cache)
{
    Bsr out;
    if (!leveled) {
        auto st = std::make_shared<BsrStruct>();
        st->Rb = m.Rb;
        st->Cb = m.Cb;
        st->nbr = m.nbr;
        st->nbc = m.nbc;
        st->nnzb = m.nnzb;
        st->L = auto_lanes(m.nbr ? static_cast<double>(m.nnzb) / m.nbr : 1.0, m.Rb * m.Cb);
        st->rowptr = std::move(m.rowptr);
        st->col = std::move(m.col);
        st->lev_ptr = {0, m.nbr};
        out.st = st;
        out.val = std::move(m.val);
        return out;
    }
    return bsr_leveled(raw_of(m), s, cache);
}

namespace {
__global__ void k_same_pattern(const int* __restrict__ a, const int* __restrict__ b, int64_t n, int* diff)
{
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < n && a[i] != b[i]) *diff = 1;
}

// Structural symmetry of a square pattern with sorted columns (pattern_symmetric, bsr_host.cpp, on the
// device: the host check took 28 s on an 850 M-entry level at 160^3).  One warp per block row; every
// entry (i, j) looks i up in row j by bisection.
__global__ void k_pattern_symmetric(const int* __restrict__ rowptr, const int* __restrict__ col, int n, int* asym)
{
    const int i = static_cast<int>((static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5);
    const int lane = threadIdx.x & 31;
    if (i >= n) return;
    for (int k = rowptr[i] + lane; k < rowptr[i + 1]; k += 32) {
        const int j = col[k];
        if (j == i) continue;
        int lo = rowptr[j], hi = rowptr[j + 1];
        while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            if (col[mid] < i) lo = mid + 1;
            else hi = mid;
        }
        if (lo >= rowptr[j + 1] || col[lo] != i) *asym = 1;
    }
}
} // namespace

Bsr bsr_leveled(const DBsrRaw& m, cudaStream_t s, LevelCache* cache)
{
    Bsr out;
    const int E = m.Rb * m.Cb;
    if (cache && cache->st && cache->nbr == m.nbr && cache->nbc == m.nbc && cache->nnzb == m.nnzb &&
        cache->Rb == m.Rb && cache->Cb == m.Cb && std::getenv("ED_NO_LEVEL_CACHE") == nullptr) {
        // same pattern as the previous build's level operator? (exact, on the device)
        cache->flag.alloc(1);
        cache->flag.zero(s);
        k_same_pattern<<<g1(m.nbr + 1), kT, 0, s>>>(m.rowptr, cache->rowptr.p, m.nbr + 1, cache->flag.p);
        if (m.nnzb) k_same_pattern<<<g1(m.nnzb), kT, 0, s>>>(m.col, cache->col.p, m.nnzb, cache->flag.p);
        after_launch("k_same_pattern");
        if (cache->flag.to_host(s)[0] == 0) {
            out.st = cache->st;
            out.val.alloc(std::max<int64_t>(m.nnzb * E, 1));
            k_gather_rows<<<g1(m.nbr), kT, 0, s>>>(m.rowptr, m.val, out.st->perm.p ? out.st->perm.p : nullptr, m.nbr, E,
                                                   out.st->rowptr.p, out.val.p);
            after_launch("k_gather_rows");
            ED_CUDA(cudaStreamSynchronize(s));
            return out;
        }
    }
    // level schedule needs the pattern on the host
    const double t_start = now_ms_host();
    BlockPattern pat;
    pat.nbr = m.nbr;
    pat.nbc = m.nbc;
    static const bool verbose = std::getenv("ED_AMG_VERBOSE") != nullptr;
    double tl = now_ms_host();
    auto lap = [&](const char* what) {
        if (!verbose) return;
        const double t = now_ms_host();
        std::fprintf(stderr, "[level-op] %-14s %8.2f ms\n", what, t - tl);
        tl = t;
    };
    std::vector<int> rp(static_cast<size_t>(m.nbr) + 1);
    pat.col.resize(m.nnzb);
    DevArray<int> asym(1);
    asym.zero(s);
    if (m.nbr == m.nbc && m.nbr > 0) {
        k_pattern_symmetric<<<g1(32LL * m.nbr), kT, 0, s>>>(m.rowptr, m.col, m.nbr, asym.p);
        after_launch("k_pattern_symmetric");
    }
    ED_CUDA(cudaMemcpyAsync(rp.data(), m.rowptr, rp.size() * sizeof(int), cudaMemcpyDeviceToHost, s));
    if (m.nnzb) ED_CUDA(cudaMemcpyAsync(pat.col.data(), m.col, m.nnzb * sizeof(int), cudaMemcpyDeviceToHost, s));
    const bool symmetric = m.nbr == m.nbc && asym.to_host(s)[0] == 0; // synchronises the stream
    HostSection hsec;
    pat.rowptr.assign(rp.begin(), rp.end());
    lap("download");
    if (!symmetric) throw Error(ED_UNSUPPORTED, "Gauss-Seidel operator pattern is not symmetric");
    lap("symmetric");
    std::vector<int> order, lvl;
    int nlev = 0;
    gs_level_order(pat, order, lvl, nlev);
    lap("levels");
    BsrLayout lay = make_layout(pat, order, lvl);
    lap("layout");
    out.st = bsr_make_struct(pat, lay, m.Rb, m.Cb, s);
    lap("struct");
    out.st->leveled = true;
    if (std::getenv("ED_AMG_VERBOSE"))
        std::fprintf(stderr,
                     "[amg-dev] level op: block rows %d blocks %lld gs-levels %d lanes %d groups %d (%s) "
                     "(%.1f ms host)\n",
                     m.nbr, static_cast<long long>(m.nnzb), out.st->nlev(), out.st->L, out.st->ngrp,
                     group_sweep_on(*out.st) ? "group sweep" : "tagged dataflow sweep", now_ms_host() - t_start);
    out.val.alloc(std::max<int64_t>(m.nnzb * E, 1));
    k_gather_rows<<<g1(m.nbr), kT, 0, s>>>(m.rowptr, m.val, out.st->perm.p ? out.st->perm.p : nullptr, m.nbr, E,
                                           out.st->rowptr.p, out.val.p);
    after_launch("k_gather_rows");
    if (cache) {
        cache->nbr = m.nbr;
        cache->nbc = m.nbc;
        cache->nnzb = m.nnzb;
        cache->Rb = m.Rb;
        cache->Cb = m.Cb;
        cache->rowptr.alloc(static_cast<size_t>(m.nbr) + 1);
        ED_CUDA(cudaMemcpyAsync(cache->rowptr.p, m.rowptr, sizeof(int) * (m.nbr + 1), cudaMemcpyDeviceToDevice, s));
        cache->col.alloc(std::max<int64_t>(m.nnzb, 1));
        if (m.nnzb) ED_CUDA(cudaMemcpyAsync(cache->col.p, m.col, sizeof(int) * m.nnzb, cudaMemcpyDeviceToDevice, s));
        cache->st = out.st;
    }
    ED_CUDA(cudaStreamSynchronize(s));
    return out;
}

DevSetupResult amg_build_device_impl(const Bsr& A0, const AmgOpts& opts, cudaStream_t s, const LevelHook& on_level);

DevSetupResult amg_build_device(const Bsr& A0, const AmgOpts& opts, cudaStream_t s, const LevelHook& on_level)
{
    try {
        return amg_build_device_impl(A0, opts, s, on_level);
    } catch (...) {
        if (on_level) on_level(-1, DBsrRaw{});
        throw;
    }
}

DevSetupResult amg_build_device_impl(const Bsr& A0, const AmgOpts& opts, cudaStream_t s, const LevelHook& on_level)
{
    const int k = opts.block_size;
    const int Bs = A0.st->Rb;
    if (k != Bs || (Bs != 1 && Bs != 3)) throw Error(ED_UNSUPPORTED, "device AMG setup needs block size == storage block");
    Timer T;
    DevSetupResult res;
    DBsr A = natural_copy(A0, s);
    const int nrows0 = A.nbr * Bs;
    // Row grouping: explicit maps (set_amg_maps) must describe consecutive runs of k
    if (!opts.row_to_node.empty()) {
        for (int r = 0; r < nrows0; ++r)
            if (opts.row_to_node[r] != r / k || opts.row_component[r] != r % k)
                throw Error(ED_UNSUPPORTED, "device AMG setup needs consecutive node rows");
    }
    std::vector<double> Bn(static_cast<size_t>(nrows0) * k, 0.0);
    for (int r = 0; r < nrows0; ++r) Bn[static_cast<size_t>(r) * k + r % k] = 1.0;
    T.lap(s, "start", 0, A.nbr, A.nnzb);

    while (A.nbr * Bs > opts.coarse_max_rows && static_cast<int>(res.levels.size()) + 1 < opts.max_levels) {
        const int lvl = static_cast<int>(res.levels.size());
        const int n = A.nbr;
        // strength graph
        DevArray<double> dw(n), s2(std::max<int64_t>(A.nnzb, 1));
        DevArray<unsigned char> flag(std::max<int64_t>(A.nnzb, 1)), sym(std::max<int64_t>(A.nnzb, 1));
        DevArray<int> namb(1), scnt(n);
        namb.zero(s);
        if (Bs == 3) {
            k_diag_w<3><<<g1(n), kT, 0, s>>>(A.rowptr.p, A.col.p, A.val.p, n, dw.p);
            k_strength<3><<<g1(n), kT, 0, s>>>(A.rowptr.p, A.col.p, A.val.p, n, dw.p, opts.strength_theta, flag.p,
                                               s2.p, namb.p);
        } else {
            k_diag_w<1><<<g1(n), kT, 0, s>>>(A.rowptr.p, A.col.p, A.val.p, n, dw.p);
            k_strength<1><<<g1(n), kT, 0, s>>>(A.rowptr.p, A.col.p, A.val.p, n, dw.p, opts.strength_theta, flag.p,
                                               s2.p, namb.p);
        }
        after_launch("k_strength");
        const int amb = namb.to_host(s)[0];
        if (amb > 0) {
            // re-decide borderline comparisons with the host's libm pow (amg.cpp:65)
            std::vector<unsigned char> hf = flag.to_host(s);
            const std::vector<double> hs2 = s2.to_host(s), hdw = dw.to_host(s);
            const std::vector<int> hrp = A.rowptr.to_host(s), hcol = A.col.to_host(s);
            for (int I = 0; I < n; ++I)
                for (int kk = hrp[I]; kk < hrp[I + 1]; ++kk)
                    if (hf[kk] == 2)
                        hf[kk] = std::sqrt(hs2[kk]) > opts.strength_theta * std::pow(hdw[I] * hdw[hcol[kk]], 0.25);
            flag.upload(hf, s);
        }
        s2.release();
        k_symmetrize<<<g1(n), kT, 0, s>>>(A.rowptr.p, A.col.p, flag.p, n, sym.p, scnt.p);
        after_launch("k_symmetrize");
        T.lap(s, "strength", lvl, n, amb);
        // neighbour lists -> host aggregation
        std::vector<int64_t> nptr(n + 1, 0);
        std::vector<int> agg_of_node;
        int n_agg = 0;
        {
            const std::vector<int> c = scnt.to_host(s);
            for (int I = 0; I < n; ++I) nptr[I + 1] = nptr[I] + c[I];
        }
        {
            std::vector<int> nbr(nptr[n]);
            const std::vector<unsigned char> hs = sym.to_host(s);
            const std::vector<int> hrp = A.rowptr.to_host(s), hcol = A.col.to_host(s);
            HostSection hsec;
            for (int I = 0; I < n; ++I) {
                int64_t o = nptr[I];
                for (int kk = hrp[I]; kk < hrp[I + 1]; ++kk)
                    if (hs[kk]) nbr[o++] = hcol[kk];
            }
            n_agg = amg_aggregate(nptr, nbr, agg_of_node);
        }
        flag.release();
        sym.release();
        T.lap(s, "aggregate", lvl, n_agg, 0);
        if (n_agg <= 0 || n_agg >= n) {
            if (res.levels.empty()) {
                res.fallback = true;
                DevArray<double> inv(nrows0);
                if (Bs == 3) k_invdiag<3><<<g1(n), kT, 0, s>>>(A.rowptr.p, A.col.p, A.val.p, n, inv.p);
                else k_invdiag<1><<<g1(n), kT, 0, s>>>(A.rowptr.p, A.col.p, A.val.p, n, inv.p);
                after_launch("k_invdiag");
                res.fallback_inv_diag = inv.to_host(s);
                return res;
            }
            break;
        }
        // tentative prolongator (host, tiny)
        const int nrows = n * Bs;
        std::vector<double> Bc;
        HostCsr Pt_h;
        {
            HostSection hsec;
            std::vector<int> agg_of_row(nrows);
            for (int r = 0; r < nrows; ++r) agg_of_row[r] = agg_of_node[r / Bs];
            Pt_h = amg_tentative(nrows, k, agg_of_row, n_agg, Bn, Bc);
        }
        DBsr Pt = upload_block(Pt_h, Bs, k, s);
        T.lap(s, "tentative", lvl, Pt.nbr, Pt.nnzb);
        // inverse diagonal + spectral radius of D^-1 A (amg.cpp:170-185)
        DevLevelData L;
        L.invd.alloc(nrows);
        if (Bs == 3) k_invdiag<3><<<g1(n), kT, 0, s>>>(A.rowptr.p, A.col.p, A.val.p, n, L.invd.p);
        else k_invdiag<1><<<g1(n), kT, 0, s>>>(A.rowptr.p, A.col.p, A.val.p, n, L.invd.p);
        after_launch("k_invdiag");
        L.inv_diag = L.invd.to_host(s);
        double omega = 0.0;
        if (opts.smooth_prolongator) {
            // power iteration (amg.cpp:170-185) with the reference's
            // sequential norms on the host.  Only ||w|| gates the next launch;
            // lambda = ||w|| / ||v|| is used after the last iteration only, so
            // ||v|| is formed once, for the v that entered the last iteration
            // (v = w_prev * (1/||w_prev||), bitwise the reference's update).
            DevArray<double> v(nrows), w(nrows);
            vec_fill(v.p, 1.0, nrows, s);
            std::vector<double> hw(nrows), hw_prev;
            double inv_prev = 0.0, lambda = 1.0;
            bool zero = false;
            int it = 0;
            double* hbuf = pinned_scratch(nrows);
            for (it = 0; it < 10; ++it) {
                if (Bs == 3) k_spmv_seq<3, 3><<<g1(3LL * n), kT, 0, s>>>(A.rowptr.p, A.col.p, A.val.p, n, v.p, w.p);
                else k_spmv_seq<1, 1><<<g1(n), kT, 0, s>>>(A.rowptr.p, A.col.p, A.val.p, n, v.p, w.p);
                k_mul_vec<<<g1(nrows), kT, 0, s>>>(w.p, L.invd.p, nrows);
                after_launch("k_spmv_seq");
                ED_CUDA(cudaMemcpyAsync(hbuf, w.p, sizeof(double) * nrows, cudaMemcpyDeviceToHost, s));
                ED_CUDA(cudaStreamSynchronize(s));
                HostSection hsec;
                if (it == 9) hw_prev.swap(hw); // w of iteration 8 (v of iteration 9 = hw_prev * inv_prev)
                hw.assign(hbuf, hbuf + nrows);
                const double nrm = amg_seq_norm(hw);
                if (nrm == 0.0) {
                    lambda = 1.0;
                    zero = true;
                    break;
                }
                const double inv = 1.0 / nrm;
                if (it < 9) {
                    k_scale_into<<<g1(nrows), kT, 0, s>>>(v.p, w.p, inv, nrows);
                    after_launch("k_scale_into");
                    inv_prev = inv;
                } else {
                    // v of this (last) iteration: all ones at it == 0, else w_prev / ||w_prev||
                    std::vector<double> hv(nrows, 1.0);
                    for (int i = 0; i < nrows; ++i) hv[i] = hw_prev[i] * inv_prev;
                    lambda = nrm / amg_seq_norm(hv);
                }
            }
            (void)zero;
            omega = 4.0 / (3.0 * std::max(lambda, 1e-12));
            T.lap(s, "spectral", lvl, nrows, 0);
            DBsr APt = spgemm(A, Pt, s);
            T.lap(s, "AP_tent", lvl, APt.nbr, APt.nnzb);
            if (Bs == 3) k_scale_rows<3, 3><<<g1(n), kT, 0, s>>>(APt.rowptr.p, APt.val.p, n, L.invd.p);
            else k_scale_rows<1, 1><<<g1(n), kT, 0, s>>>(APt.rowptr.p, APt.val.p, n, L.invd.p);
            after_launch("k_scale_rows");
            L.P = add(Pt, APt, 1.0, -omega, s);
            T.lap(s, "smooth_P", lvl, L.P.nbr, L.P.nnzb);
        } else {
            L.P = std::move(Pt);
        }
        L.R = transpose(L.P, s);
        T.lap(s, "transpose", lvl, L.R.nbr, L.R.nnzb);
        DBsr AP = spgemm(A, L.P, s);
        T.lap(s, "AP", lvl, AP.nbr, AP.nnzb);
        DBsr Ac = spgemm(L.R, AP, s);
        T.lap(s, "RAP", lvl, Ac.nbr, Ac.nnzb);
        L.A = std::move(A);
        res.levels.push_back(std::move(L));
        A = std::move(Ac);
        Bn = std::move(Bc);
        if (on_level) on_level(lvl + 1, raw_of(A));
    }
    // coarsest level: dense COD on the host (amg.cpp:278-294)
    DevLevelData L;
    const int n = A.nbr;
    const int nr = n * Bs;
    L.invd.alloc(nr);
    if (Bs == 3) k_invdiag<3><<<g1(n), kT, 0, s>>>(A.rowptr.p, A.col.p, A.val.p, n, L.invd.p);
    else k_invdiag<1><<<g1(n), kT, 0, s>>>(A.rowptr.p, A.col.p, A.val.p, n, L.invd.p);
    after_launch("k_invdiag");
    L.inv_diag = L.invd.to_host(s);
    check_coarse_size(nr, static_cast<int>(res.levels.size()));
    const HostCsr Ah = to_host_csr(A, s);
    HostSection hsec;
    std::vector<double> dense(static_cast<size_t>(nr) * nr, 0.0);
    for (int r = 0; r < nr; ++r)
        for (int64_t kk = Ah.rowptr[r]; kk < Ah.rowptr[r + 1]; ++kk)
            dense[static_cast<size_t>(Ah.col[kk]) * nr + r] = Ah.val[kk];
    res.pinv = cod_pinv(dense, nr, 1e-12);
    if (std::getenv("ED_AMG_VERBOSE")) std::fprintf(stderr, "[amg-dev] alloc/free host ms so far: %.1f\n", alloc_ms());
    res.nc = nr;
    L.A = std::move(A);
    res.levels.push_back(std::move(L));
    T.lap(s, "coarse_cod", static_cast<int>(res.levels.size()) - 1, nr, 0);
    return res;
}

} // namespace edb
