// Internal declarations of the B200-native Newton-step library.
//
// Data model: every operator of the 2x2 block system and of
// both AMG hierarchies is stored in one format, a sliced ELL of small dense
// blocks ("SELL-32, Rb x Cb blocks"): block rows are grouped 32 per slice
// (one warp), each lane owns one block row and walks its blocks in ascending
// block-column order, so a lane's scalar sums happen in exactly the column
// order of the reference CSR row (csr.cpp:11-27).  Values are stored
// entry-major inside a slot, [slot][entry][lane], so a warp's loads of one
// entry are 32 consecutive doubles (256 B, fully coalesced).  Square
// operators used by Gauss-Seidel carry a level schedule: block rows are
// permuted so that each dependency level of the in-place sweep
// (amg.cpp:311-322) is a contiguous run of slices.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/elastodyn_b200.h"

namespace edb {

constexpr int kLanes = 32;

struct Error : std::runtime_error {
    int code;
    int64_t detail;
    Error(int c, const std::string& m, int64_t d = -1) : std::runtime_error(m), code(c), detail(d) {}
};

#define ED_CUDA(call)                                                                       \
    do {                                                                                    \
        cudaError_t e_ = (call);                                                            \
        if (e_ != cudaSuccess)                                                              \
            throw ::edb::Error(ED_CUDA_ERROR, std::string(#call) + ": " + cudaGetErrorString(e_)); \
    } while (0)

// Launch bookkeeping: every kernel launcher calls this after <<<>>>.
void after_launch(const char* what);
int64_t launch_count();

// Owning device array (move-only).
template <class T>
struct DevArray {
    T* p = nullptr;
    size_t n = 0;
    DevArray() = default;
    explicit DevArray(size_t count) { alloc(count); }
    DevArray(const DevArray&) = delete;
    DevArray& operator=(const DevArray&) = delete;
    DevArray(DevArray&& o) noexcept : p(o.p), n(o.n) { o.p = nullptr; o.n = 0; }
    DevArray& operator=(DevArray&& o) noexcept
    {
        if (this != &o) {
            release();
            p = o.p;
            n = o.n;
            o.p = nullptr;
            o.n = 0;
        }
        return *this;
    }
    ~DevArray() { release(); }
    void alloc(size_t count)
    {
        if (count == n && p) return;
        release();
        if (count == 0) return;
        ED_CUDA(cudaMalloc(reinterpret_cast<void**>(&p), count * sizeof(T)));
        n = count;
    }
    void release()
    {
        if (p) cudaFree(p);
        p = nullptr;
        n = 0;
    }
    void upload(const T* h, size_t count, cudaStream_t s)
    {
        alloc(count);
        if (count) ED_CUDA(cudaMemcpyAsync(p, h, count * sizeof(T), cudaMemcpyHostToDevice, s));
    }
    void upload(const std::vector<T>& h, cudaStream_t s) { upload(h.data(), h.size(), s); }
    void download(T* h, cudaStream_t s) const
    {
        if (n) ED_CUDA(cudaMemcpyAsync(h, p, n * sizeof(T), cudaMemcpyDeviceToHost, s));
    }
    std::vector<T> to_host(cudaStream_t s) const
    {
        std::vector<T> h(n);
        download(h.data(), s);
        ED_CUDA(cudaStreamSynchronize(s));
        return h;
    }
    void zero(cudaStream_t s)
    {
        if (n) ED_CUDA(cudaMemsetAsync(p, 0, n * sizeof(T), s));
    }
    void copy_from(const DevArray& o, cudaStream_t s)
    {
        alloc(o.n);
        if (n) ED_CUDA(cudaMemcpyAsync(p, o.p, n * sizeof(T), cudaMemcpyDeviceToDevice, s));
    }
};

// Host-side block-CSR pattern (sorted block columns per block row).
struct BlockPattern {
    int nbr = 0, nbc = 0;
    std::vector<int64_t> rowptr; // nbr + 1
    std::vector<int> col;        // nnzb
    int64_t nnzb() const { return rowptr.empty() ? 0 : rowptr.back(); }
};

// Host-side scalar CSR (mirror of CsrMatrix, csr.hpp:13-46).
struct HostCsr {
    int nrows = 0, ncols = 0;
    std::vector<int> rowptr, col;
    std::vector<double> val;
    int64_t nnz() const { return static_cast<int64_t>(col.size()); }
};

// Structure of a SELL-32 block matrix (shared between copies with
// different values, e.g. the assembled and the scaled working system).
struct SellStruct {
    int Rb = 1, Cb = 1;
    int nbr = 0, nbc = 0; // block rows / block cols
    int nslices = 0;
    int64_t nslots = 0; // total slot rows (sum of slice widths)
    int64_t nnzb = 0;   // structural blocks
    DevArray<int64_t> slice_off; // [nslices+1], in slot rows
    DevArray<int> perm;          // [nslices*32]: block row, or -1 for a padding lane
    DevArray<int> rowlen;        // [nslices*32]
    DevArray<int> inv;           // [nbr]: block row -> slice*32 + lane
    DevArray<int> col;           // [nslots*32]
    std::vector<int> lev_slice;  // [nlev+1] slice ranges of the level schedule
    // host mirrors
    std::vector<int64_t> h_slice_off;
    std::vector<int> h_perm, h_rowlen, h_inv, h_col;
    int nlev() const { return static_cast<int>(lev_slice.size()) - 1; }
    int64_t nval() const { return nslots * kLanes * Rb * Cb; }
};

struct Sell {
    std::shared_ptr<SellStruct> st;
    DevArray<double> val; // [nslots][Rb*Cb][32]
    const SellStruct& s() const { return *st; }
    int nrows() const { return st->nbr * st->Rb; }
    int ncols() const { return st->nbc * st->Cb; }
    double bytes_per_spmv() const; // algorithmic bytes of one y = M x
    void copy_values_from(const Sell& o, cudaStream_t s)
    {
        st = o.st;
        val.copy_from(o.val, s);
    }
};

// Layout of a block pattern in SELL form: per block of the pattern (block-CSR
// order) the address slot*32 + lane.
struct SellLayout {
    std::vector<int64_t> slice_off;
    std::vector<int> perm, rowlen, inv;
    std::vector<int> lev_slice;
    std::vector<int64_t> addr;
    int nslices = 0;
    int64_t nslots = 0;
};

// row_order: block rows in the order they are laid out; level_of_pos: level
// per position (a new slice starts at every level change), or empty.
SellLayout make_sell_layout(const BlockPattern& pat, const std::vector<int>& row_order,
                            const std::vector<int>& level_of_pos);
std::shared_ptr<SellStruct> sell_make_struct(const BlockPattern& pat, const SellLayout& lay, int Rb,
                                             int Cb, cudaStream_t s);
// Block values in pattern order (nnzb blocks, each Rb*Cb row-major) -> SELL value array (host).
std::vector<double> sell_pack_values(const SellStruct& st, const SellLayout& lay,
                                     const std::vector<double>& bvals);
// Level schedule of the in-place Gauss-Seidel sweep on a square block pattern:
// level[i] = 1 + max(level[j] : j < i, (i,j) in pattern).
void gs_level_order(const BlockPattern& pat, std::vector<int>& order, std::vector<int>& level_of_pos,
                    int& nlev);
bool pattern_symmetric(const BlockPattern& pat);
// Build a leveled (square) or natural-order SELL directly from a scalar CSR
// grouped into Rb x Cb blocks (zero-filled).
Sell sell_from_csr(const HostCsr& a, int Rb, int Cb, bool leveled, cudaStream_t s);
// Read a Sell back as scalar CSR (zero-filled blocks included).
HostCsr sell_to_csr(const Sell& m, cudaStream_t s);
BlockPattern block_pattern_of_csr(const HostCsr& a, int Rb, int Cb);
std::vector<double> block_values_of_csr(const HostCsr& a, const BlockPattern& pat, int Rb, int Cb);

// ---------------------------------------------------------------------------
// Kernel launchers (kernels_sparse.cu)

// y = M x (mode 0), y = b - M x (mode 1), y += M x (mode 2)
void spmv(const Sell& M, const double* x, double* y, const double* b, int mode, cudaStream_t s);
// y = (M1 x1) + sgn * (M2 x2); M1, M2 share the row layout (same perm/slices)
void spmv2(const Sell& M1, const double* x1, const Sell& M2, const double* x2, double* y, double sgn,
           cudaStream_t s);
// one in-place Gauss-Seidel half sweep over the level schedule
void sgs_sweep(const Sell& A, const double* b, double* z, const double* inv_diag, bool forward,
               cudaStream_t s);
// Jacobi relaxation z += w * inv_diag * (b - t)
void jacobi_update(double* z, const double* b, const double* t, const double* inv_diag, double w,
                   int64_t n, cudaStream_t s);
// entries *= wr[row] * wc[col]
void sell_scale(Sell& M, const double* wr, const double* wc, cudaStream_t s);
// scalar diagonal of a square Sell (0 when absent)
void sell_diag(const Sell& M, double* d, cudaStream_t s);
// inv_diag[i] = d != 0 ? 1/d : 1
void inv_diag_from(const double* d, double* invd, int64_t n, cudaStream_t s);
// z = Pinv r (dense n x n, row-major)
void dense_gemv(const double* Pinv, const double* r, double* z, int n, cudaStream_t s);

// ---- vectors / reductions (deterministic: fixed grid, fixed order) ----
void vec_fill(double* x, double v, int64_t n, cudaStream_t s);
void vec_copy(double* y, const double* x, int64_t n, cudaStream_t s);
void vec_sub_from(double* r, const double* b, int64_t n, cudaStream_t s); // r = b - r
void vec_mul(double* x, const double* w, int64_t n, cudaStream_t s);      // x *= w
void vec_add(double* x, const double* y, int64_t n, cudaStream_t s);      // x += y
void vec_div_scalar(double* y, const double* x, const double* d_scal, const double* d_guard,
                    int64_t n, cudaStream_t s); // y = x / *d_scal  (skip if guard && *guard <= 1e-300)

// Reduction scratch owned by the context.
struct Reducer {
    DevArray<double> partials; // [max_vals * max_blocks]
    DevArray<unsigned int> ticket;
    int max_blocks = 0;
    int max_vals = 0;
    void ensure(int vals, cudaStream_t s);
};
int reduce_blocks(int64_t n);
// out = x . y   (device scalar)
void dot(Reducer& R, const double* x, const double* y, int64_t n, double* out, cudaStream_t s);
// out = sqrt(x . x)
void norm2(Reducer& R, const double* x, int64_t n, double* out, cudaStream_t s);
// MGS step: if hprev: w -= (*hprev) * vprev; then *hout = vnext . w   (vnext may be null: *hout = w.w)
void mgs_axpy_dot(Reducer& R, double* w, const double* vprev, const double* hprev,
                  const double* vnext, int64_t n, double* hout, cudaStream_t s);
// corr[i] = V_i . w, i < k, V given as device pointer array
void multi_dot(Reducer& R, const double* const* dV, int k, const double* w, int64_t n, double* corr,
               cudaStream_t s);
// GMRES reorthogonalization decision (krylov.cpp:87-105), one thread:
// sc[0] = wnorm^2 in, sc[1] = flag out, sc[2] = wnorm out, h[0..k) += corr when flag.
void reorth_decide(double* sc, double* h, const double* corr, int k, cudaStream_t s);
// if (sc[1] != 0) { w -= sum_i corr[i] V_i (sequential i); sc[0] = w . w; sc[2] = sqrt(sc[0]) }
void reorth_apply(Reducer& R, double* w, const double* const* dV, const double* corr, int k,
                  int64_t n, double* sc, cudaStream_t s);
// x += sum_i y[i] * V_i (sequential in i, exactly vec_axpy order)
void multi_axpy(double* x, const double* const* dV, const double* y, int k, int64_t n, cudaStream_t s);

} // namespace edb
