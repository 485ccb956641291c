// Internal declarations of the B200-native Newton-step library.
//
// Data model: every operator of the 2x2 block system and of
// both AMG hierarchies is a block-sparse (BSR) matrix of small dense blocks
// (3x3, 3x1, 1x3, 1x1) whose block rows are stored in level order: square
// operators used by Gauss-Seidel are permuted so that each dependency level
// of the in-place sweep (amg.cpp:311-322) is a contiguous run of rows, and a
// persistent dataflow kernel walks the levels without a launch per level.
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
std::string& prof_tag(); // ED_PROFILE attribution tag (e.g. hierarchy/level)

// Host milliseconds spent in cudaMalloc/cudaFree (diagnostics, ED_AMG_VERBOSE).
double& alloc_ms();
double now_ms_host();
// Host milliseconds of pure host work on this thread (AMG aggregation, tentative
// prolongator, level schedules, COD): HostSection scopes add to it.
double& host_ms_acc();
struct HostSection {
    double t0 = now_ms_host();
    ~HostSection() { host_ms_acc() += now_ms_host() - t0; }
};

// Stream that device arrays allocated on this thread are ordered on (the
// calling context's stream inside every C-ABI entry point; null outside:
// plain synchronous cudaMalloc/cudaFree).  Stream-ordered allocations come
// from the device's memory pool, which keeps freed memory for reuse, so the
// per-Newton-step AMG rebuild does not pay cudaMalloc/cudaFree (or their
// implicit device synchronisation) for every temporary.
cudaStream_t& alloc_stream();
// stream-ordered caching allocator (api.cpp): size classes with <= 12.5%
// slack, per-stream free lists; a cache miss is a plain cudaMalloc
void* cache_alloc(size_t bytes, cudaStream_t s);
void cache_free(void* p, size_t bytes, cudaStream_t s);
void cache_release_stream(cudaStream_t s);

// Owning device array (move-only).
template <class T>
struct DevArray {
    static constexpr size_t kPad = 256;
    T* p = nullptr;
    size_t n = 0;
    cudaStream_t as = nullptr; // allocation stream (null: synchronous allocation)
    DevArray() = default;
    explicit DevArray(size_t count) { alloc(count); }
    DevArray(const DevArray&) = delete;
    DevArray& operator=(const DevArray&) = delete;
    DevArray(DevArray&& o) noexcept : p(o.p), n(o.n), as(o.as) { o.p = nullptr; o.n = 0; }
    DevArray& operator=(DevArray&& o) noexcept
    {
        if (this != &o) {
            release();
            p = o.p;
            n = o.n;
            as = o.as;
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
        const double t0 = now_ms_host();
        as = alloc_stream();
        // kPad bytes of slack: 16-B vector loads may round a range's end up past the last element
        if (as) p = static_cast<T*>(cache_alloc(count * sizeof(T) + kPad, as));
        else ED_CUDA(cudaMalloc(reinterpret_cast<void**>(&p), count * sizeof(T) + kPad));
        alloc_ms() += now_ms_host() - t0;
        n = count;
    }
    void release()
    {
        if (p) {
            const double t0 = now_ms_host();
            if (as) cache_free(p, n * sizeof(T) + kPad, as);
            else cudaFree(p);
            alloc_ms() += now_ms_host() - t0;
        }
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
    std::vector<int64_t> rowptr;
    std::vector<int> col;
    std::vector<double> val;
    int64_t nnz() const { return static_cast<int64_t>(col.size()); }
};

// Structure of a block-sparse (BSR) operator whose block rows are stored in
// a chosen order (level order for Gauss-Seidel operators).  Columns keep the
// original block numbering; stored row s is original row perm[s].  Kernels
// give each block row a group of L lanes (L sized to the row length) that
// split the row's blocks and combine partial sums with warp shuffles.
struct BsrStruct {
    int Rb = 1, Cb = 1;
    int nbr = 0, nbc = 0; // block rows / block cols
    int64_t nnzb = 0;
    int L = 8;            // lanes per block row (SpMV)
    int Ls = 8;           // lanes per block row of the Gauss-Seidel sweeps (latency-bound)
    DevArray<int> rowptr; // [nbr+1] over stored rows
    DevArray<int> col;    // [nnzb]
    DevArray<int> perm;   // [nbr] stored -> original (empty: identity)
    DevArray<int> inv;    // [nbr] original -> stored (empty: identity)
    DevArray<int> dpos;   // [nbr] block index of the diagonal block per stored row (-1: none)
    std::vector<int> lev_ptr; // [nlev+1] stored-row ranges of the Gauss-Seidel levels
    // dataflow schedule: items of <= rows_per_item rows, never straddling a level
    int rows_per_item = 0, nitems = 0;
    DevArray<int> item_row;   // [nitems+1]
    DevArray<unsigned int> sync; // [0]: the tagged sweep's ticket counter
    // tagged dataflow sweep (k_sgs_tag): z entries published as {lo32, epoch}{hi32, epoch} words
    mutable DevArray<ulonglong2> ztag; // [nbr * Rb], allocated zeroed at the first sweep
    mutable unsigned int tag_epoch = 0; // last epoch used (one per half sweep)
    bool chain = false;          // narrow levels: single-CTA sweep with CTA barriers
    int avg_rows_per_level = 0;
    DevArray<int> d_lev_ptr;     // device copy of lev_ptr
    // level-group sweep (kernels_group.cu): consecutive narrow levels merged
    // into groups whose in-group lower triangle is inverted per value change
    int ngrp = 0;                 // 0: no group schedule
    int grp_maxm = 0;             // scalar rows of the largest multi-level group
    int64_t grp_tinv = 0;         // packed T^-1 doubles per direction (0: all groups single-level)
    int ntchunk = 0;              // (group, 32-column) chunks of the T^-1 build
    bool grp_use = false;         // the group sweep is this operator's sweep (narrow, deep schedules)
    DevArray<int4> grp;           // [ngrp] {r0, r1, m (0: single level), 0} stored rows
    DevArray<long long> grp_toff; // [ngrp] offset of the group's packed T^-1
    DevArray<unsigned char> bcode; // [nnzb] 0 other group, 1 in-group lower, 2 in-group upper, 3 diagonal
    DevArray<int> gptr, gblk;     // in-group blocks per stored row (multi-level groups)
    DevArray<int2> tchunk;        // [ntchunk] {group, j0}
    DevArray<unsigned int> gbar;  // grid-barrier counter
    DevArray<double> gsbuf;       // [grp_maxm] phase-A sums of the current group
    // host mirrors
    std::vector<int> h_rowptr, h_col, h_perm, h_inv;
    int nlev() const { return static_cast<int>(lev_ptr.size()) - 1; }
    int64_t nval() const { return nnzb * Rb * Cb; }
    bool leveled = false;
};

struct Bsr {
    std::shared_ptr<BsrStruct> st;
    DevArray<double> val; // [nnzb][Rb*Cb] row-major blocks, stored-row order
    int nrows() const { return st->nbr * st->Rb; }
    int ncols() const { return st->nbc * st->Cb; }
    double bytes_per_spmv() const; // algorithmic bytes of one y = M x
    void copy_values_from(const Bsr& o, cudaStream_t s)
    {
        st = o.st;
        val.copy_from(o.val, s);
    }
};

// Scaled coupled operator K = [A B; C D] as a 4x4 BSR over the node graph
// (kernels_coupled.cu): natural node order, the D plane's pattern, 16 doubles
// per block; velocity rows/columns of fixed nodes zero.
struct CoupledOp {
    int n_nodes = 0;
    int64_t nnzb = 0;
    const int* rowptr = nullptr; // [n_nodes + 1] (the D plane's)
    const int* col = nullptr;    // [nnzb]
    const int* fidx = nullptr;   // node -> free velocity index (-1: fixed)
    const int2* cf = nullptr;    // [nnzb] {column node, its free velocity index}
    DevArray<double> val;        // [nnzb][16]
    // algorithmic bytes of one y = K x: blocks + one index, row pointers, x and y
    double bytes(int64_t n_unknowns) const
    {
        return static_cast<double>(nnzb) * 132.0 + 4.0 * (n_nodes + 1) + 16.0 * static_cast<double>(n_unknowns);
    }
};
void k44_build(const CoupledOp& K, const double* k4, const double* w, int nv, cudaStream_t s);
void spmv44(const CoupledOp& K, const double* x, double* y, int nv, int np, cudaStream_t s);

// Where each block of a pattern (block-CSR order) lands in the stored order.
struct BsrLayout {
    std::vector<int> perm, inv, lev_ptr;
    std::vector<int64_t> addr; // stored block index per pattern block
};

// row_order: original block rows in stored order; level_of_pos: level per
// stored position (empty: one level).
BsrLayout make_layout(const BlockPattern& pat, const std::vector<int>& row_order,
                      const std::vector<int>& level_of_pos);
std::shared_ptr<BsrStruct> bsr_make_struct(const BlockPattern& pat, const BsrLayout& lay, int Rb, int Cb,
                                           cudaStream_t s, int lanes = 0);
// block values in pattern order -> stored order (host)
std::vector<double> bsr_pack_values(const BsrStruct& st, const BsrLayout& lay, const std::vector<double>& bvals);
// Level schedule of the in-place Gauss-Seidel sweep on a square block pattern:
// level[i] = 1 + max(level[j] : j < i, (i,j) in pattern).
void gs_level_order(const BlockPattern& pat, std::vector<int>& order, std::vector<int>& level_of_pos,
                    int& nlev);
// structural symmetry of a square pattern with sorted columns: required of every Gauss-Seidel
// operator (a row's later neighbours must wait on it: level schedule and tagged sweep)
bool pattern_symmetric(const BlockPattern& pat);
// lanes per block row of the BSR kernels for an average row length (bsr_host.cpp)
int auto_lanes(double avg_blocks, int entries);
Bsr bsr_from_csr(const HostCsr& a, int Rb, int Cb, bool leveled, cudaStream_t s);
HostCsr bsr_to_csr(const Bsr& m, cudaStream_t s);
BlockPattern block_pattern_of_csr(const HostCsr& a, int Rb, int Cb);
std::vector<double> block_values_of_csr(const HostCsr& a, const BlockPattern& pat, int Rb, int Cb);

// ---------------------------------------------------------------------------
// Kernel launchers (kernels_sparse.cu)

// y = M x (mode 0), y = b - M x (mode 1), y += M x (mode 2)
void spmv(const Bsr& M, const double* x, double* y, const double* b, int mode, cudaStream_t s);
// y = (M1 x1) + sgn * (M2 x2); M1, M2 share the row layout (same perm/slices)
void spmv2(const Bsr& M1, const double* x1, const Bsr& M2, const double* x2, double* y, double sgn,
           cudaStream_t s);
// one in-place Gauss-Seidel half sweep over the level schedule (dataflow kernel)
// dense: the operator's sweep auxiliary data (sweep_prepare)
void sgs_sweep(const Bsr& A, const double* b, double* z, const double* inv_diag, bool forward,
               cudaStream_t s, const double* dense = nullptr);
// ED_SWEEP: 0 default (group sweep where BsrStruct::grp_use), 1 legacy, 2 group everywhere
int sweep_mode();
bool group_sweep_on(const BsrStruct& S);
// per-value-change auxiliary data of a Gauss-Seidel operator: the group
// sweep's T^-1, or the push sweep's packed blocks (none for the dataflow / chain sweeps)
void sweep_prepare(const Bsr& A, const double* invd, DevArray<double>& aux, cudaStream_t s);
// level-group half sweep (kernels_group.cu); X = group_prepare output
void sgs_group(const Bsr& A, const double* b, double* z, const double* invd, bool fwd, cudaStream_t s,
               const double* X);
// packed in-group triangular inverses of both sweep directions (values and inv_diag as of the call)
void group_prepare(const Bsr& A, const double* invd, DevArray<double>& X, cudaStream_t s);
// group schedule of a leveled square operator (bsr_host.cpp)
void group_build(BsrStruct& S, cudaStream_t s);
// Jacobi relaxation z += w * inv_diag * (b - t)
void jacobi_update(double* z, const double* b, const double* t, const double* inv_diag, double w,
                   int64_t n, cudaStream_t s);
// entries *= wr[row] * wc[col]
void bsr_scale(Bsr& M, const double* wr, const double* wc, cudaStream_t s);
// scalar diagonal of a square Bsr (0 when absent)
void bsr_diag(const Bsr& M, double* d, cudaStream_t s);
// inv_diag[i] = d != 0 ? 1/d : 1
void inv_diag_from(const double* d, double* invd, int64_t n, cudaStream_t s);
// out[i] = 1 / d[i] (no guard)
void recip(const double* d, double* out, int64_t n, cudaStream_t s);
// z = Pinv r (dense n x n, row-major)
void dense_gemv(const double* Pinv, const double* r, double* z, int n, cudaStream_t s);

// ---- ILU(0) on the monolithic block system (ilu0.cu) ----
struct WorkSysView {
    const Bsr *A, *B, *C, *D;
};
struct DevIlu0 {
    int n = 0, nlf = 0, nlb = 0;
    DevArray<int> rowptr, col, dpos, lf_ptr, rows_f, lb_ptr, rows_b;
    DevArray<double> val; // factors: unit-lower L below the diagonal, U on and above
};
// Ilu0Precond(monolithic_csr(K)) (ilu0.cpp:9-48): throws ED_ZERO_DIAGONAL on a
// missing diagonal or a zero pivot
void ilu0_build(const WorkSysView& W, DevIlu0& f, cudaStream_t s);
// z = U^-1 L^-1 r (ilu0.cpp:50-68)
void ilu0_apply(const DevIlu0& f, const double* r, double* z, cudaStream_t s);

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

namespace edb {
// Live per-kernel accounting (bench.py's roofline): CUDA events around each
// sparse launch on its stream, resolved after the caller synchronises.
bool acct_on();
int acct_begin(cudaStream_t s, const char* name, double bytes);
void acct_end(cudaStream_t s, int idx);
void acct_bytes(const char* name, double bytes);
struct AcctScope {
    cudaStream_t s;
    int idx = -1;
    AcctScope(cudaStream_t st, const char* name, double bytes) : s(st)
    {
        if (acct_on()) idx = acct_begin(s, name, bytes);
    }
    ~AcctScope()
    {
        if (idx >= 0) acct_end(s, idx);
    }
};
// algorithmic bytes of a launch whose time is not recorded (vector kernels)
inline void acct_vec(const char* name, double bytes)
{
    if (acct_on()) acct_bytes(name, bytes);
}
} // namespace edb
