// Dense V-cycle operator of the coarse tail of an AMG hierarchy.
//
// AmgHierarchy::cycle (amg.cpp:326-352) is linear in the residual r (the
// reference's own VcycleIsLinearInTheResidual test): with zero initial
// guess, z = V_l r for a fixed matrix V_l.  Below some level the operators
// of the reference's smoothed aggregation are small and nearly dense
// (hundreds of rows, ~1 row per Gauss-Seidel dependency level), so their
// sweeps are chains of ~n tiny dependent steps on the GPU.  For those levels
// we form V_l explicitly once per hierarchy build and apply it as ONE dense
// GEMV per V-cycle (n^2 doubles streamed at HBM/L2 bandwidth instead of
// ~4n dependent steps).
//
// V_l is built bottom-up with the reference's recursion, on n x n matrix
// right-hand sides (columns = unit residuals):
//   Z  = 0
//   pre sweeps:  Zf = T_f^-1 (I - U Z);  Z = T_b^-1 (I - L Zf)   (amg.cpp:311-322)
//   Res = I - A Z;  Z += P V_{l+1} R Res                         (amg.cpp:341-349)
//   post sweeps: as the pre sweeps                                 (amg.cpp:351)
// where L/U are the strict triangles of A and T_f = D' + L, T_b = D' + U with
// D' = 1/inv_diag (the sweep's z_i = acc * inv_diag_i, inv_diag = 1 for a
// zero diagonal).  The coarsest V is the COD pseudo-inverse (amg.cpp:331-335).
// The products are cuBLAS DGEMM/DTRSM (library GEMMs at setup time); the
// per-cycle apply is dense_gemv (kernels_sparse.cu).  Results equal the
// sequential sweeps up to roundoff.
#include <cublas_v2.h>
#include <cuda_runtime.h>

#include <map>
#include <mutex>
#include <utility>
#include <vector>

#include "amg_device.hpp"
#include "ed_internal.hpp"

namespace edb {
namespace {

#define ED_BLAS(call)                                                                                \
    do {                                                                                             \
        cublasStatus_t st_ = (call);                                                                 \
        if (st_ != CUBLAS_STATUS_SUCCESS)                                                            \
            throw ::edb::Error(ED_CUDA_ERROR, std::string(#call) + ": cublas status " + std::to_string(st_)); \
    } while (0)

// One cuBLAS handle per stream, created once and kept (handles are not
// thread-safe; the concurrent A / S_hat tail builds run on different streams).
cublasHandle_t blas(cudaStream_t s)
{
    static std::mutex mu;
    static std::map<std::pair<int, cudaStream_t>, cublasHandle_t> handles;
    int d = 0;
    ED_CUDA(cudaGetDevice(&d));
    cublasHandle_t h = nullptr;
    {
        std::lock_guard<std::mutex> lk(mu);
        auto it = handles.find({d, s});
        if (it == handles.end()) {
            ED_BLAS(cublasCreate(&h));
            handles[{d, s}] = h;
        } else {
            h = it->second;
        }
    }
    ED_BLAS(cublasSetStream(h, s));
    ED_BLAS(cublasSetPointerMode(h, CUBLAS_POINTER_MODE_HOST));
    return h;
}

// natural-order BSR -> column-major dense (ld = rows); D must be zeroed.
// One warp per block row, lanes over its blocks.
__global__ void k_densify(const int* __restrict__ rowptr, const int* __restrict__ col, const double* __restrict__ val,
                          int nbr, int Rb, int Cb, double* D, int64_t ld)
{
    const int br = static_cast<int>((static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5);
    const int lane = threadIdx.x & 31;
    if (br >= nbr) return;
    for (int k = rowptr[br] + lane; k < rowptr[br + 1]; k += 32) {
        const int c = col[k];
        for (int r = 0; r < Rb; ++r)
            for (int d = 0; d < Cb; ++d)
                D[static_cast<int64_t>(br * Rb + r) + static_cast<int64_t>(c * Cb + d) * ld] =
                    val[static_cast<int64_t>(k) * Rb * Cb + r * Cb + d];
    }
}

// T = A with diagonal D' = 1/inv_diag; Up = strict upper triangle of A (column-major n x n)
__global__ void k_split(const double* __restrict__ A, const double* __restrict__ invd, double* T, double* Up, int n)
{
    const int64_t idx = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (idx >= static_cast<int64_t>(n) * n) return;
    const int i = static_cast<int>(idx % n), j = static_cast<int>(idx / n);
    const double a = A[idx];
    T[idx] = i == j ? 1.0 / invd[i] : a;
    Up[idx] = i < j ? a : 0.0;
}

__global__ void k_recip(const double* __restrict__ invd, double* d, int n)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) d[i] = 1.0 / invd[i];
}

__global__ void k_identity(double* M, int n)
{
    const int64_t idx = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (idx >= static_cast<int64_t>(n) * n) return;
    M[idx] = (idx % n) == (idx / n) ? 1.0 : 0.0;
}

inline unsigned grid_of(int64_t n) { return static_cast<unsigned>((n + 255) / 256); }

void densify(const DBsr& m, DevArray<double>& D, cudaStream_t s)
{
    const int rows = m.nbr * m.Rb, cols = m.nbc * m.Cb;
    D.alloc(static_cast<size_t>(rows) * cols);
    D.zero(s);
    if (m.nbr == 0) return;
    k_densify<<<grid_of(static_cast<int64_t>(m.nbr) * 32), 256, 0, s>>>(m.rowptr.p, m.col.p, m.val.p, m.nbr, m.Rb, m.Cb,
                                                                      D.p, rows);
    after_launch("k_densify");
}

void identity(DevArray<double>& M, int n, cudaStream_t s)
{
    M.alloc(static_cast<size_t>(n) * n);
    k_identity<<<grid_of(static_cast<int64_t>(n) * n), 256, 0, s>>>(M.p, n);
    after_launch("k_identity");
}

} // namespace

void dense_vcycle_operator(const std::vector<DenseTailLevel>& lv, const std::vector<double>& pinv, int nc,
                           int pre_sweeps, int post_sweeps, DevArray<double>& out, cudaStream_t s)
{
    cublasHandle_t h = blas(s);
    const double one = 1.0, mone = -1.0, zero = 0.0;
    // coarsest: pinv is row-major, i.e. the column-major transpose
    DevArray<double> Vc, tmp;
    tmp.upload(pinv, s);
    Vc.alloc(static_cast<size_t>(nc) * nc);
    ED_BLAS(cublasDgeam(h, CUBLAS_OP_T, CUBLAS_OP_N, nc, nc, &one, tmp.p, nc, &zero, tmp.p, nc, Vc.p, nc));
    int ncur = nc;
    for (int l = static_cast<int>(lv.size()) - 1; l >= 0; --l) {
        const DenseTailLevel& L = lv[l];
        const int n = L.A->nbr * L.A->Rb;
        DevArray<double> A, T, Up, Z, M, Pd, Rd, Rc, Ec, UZ, Dp;
        densify(*L.A, A, s);
        T.alloc(static_cast<size_t>(n) * n);
        Up.alloc(T.n);
        k_split<<<grid_of(static_cast<int64_t>(n) * n), 256, 0, s>>>(A.p, L.invd, T.p, Up.p, n);
        after_launch("k_split");
        Dp.alloc(n);
        k_recip<<<grid_of(n), 256, 0, s>>>(L.invd, Dp.p, n);
        after_launch("k_recip");
        Z.alloc(T.n);
        Z.zero(s);
        bool zero_z = true;
        // one symmetric sweep on the matrix iterate Z (right-hand side I).
        // Identities used (T_f = D' + L, T_b = D' + U, T_f Zf = I - U Z):
        //   backward rhs  I - L Zf = U Z + D' Zf  (= D' Zf when Z = 0)
        // so a sweep costs one GEMM (U Z; none from zero) and two TRSMs.
        auto sweep = [&]() {
            // UZ = U Z (zero when Z = 0)
            if (!zero_z) {
                UZ.alloc(T.n);
                ED_BLAS(cublasDgemm(h, CUBLAS_OP_N, CUBLAS_OP_N, n, n, n, &one, Up.p, n, Z.p, n, &zero, UZ.p, n));
            }
            // forward: Zf = T_f^-1 (I - U Z)
            identity(M, n, s);
            if (!zero_z) ED_BLAS(cublasDgeam(h, CUBLAS_OP_N, CUBLAS_OP_N, n, n, &one, M.p, n, &mone, UZ.p, n, M.p, n));
            ED_BLAS(cublasDtrsm(h, CUBLAS_SIDE_LEFT, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_N, CUBLAS_DIAG_NON_UNIT, n, n,
                                &one, T.p, n, M.p, n));
            // backward: Z = T_b^-1 (U Z + D' Zf)
            Z.alloc(T.n);
            ED_BLAS(cublasDdgmm(h, CUBLAS_SIDE_LEFT, n, n, M.p, n, Dp.p, 1, Z.p, n));
            if (!zero_z) ED_BLAS(cublasDgeam(h, CUBLAS_OP_N, CUBLAS_OP_N, n, n, &one, Z.p, n, &one, UZ.p, n, Z.p, n));
            ED_BLAS(cublasDtrsm(h, CUBLAS_SIDE_LEFT, CUBLAS_FILL_MODE_UPPER, CUBLAS_OP_N, CUBLAS_DIAG_NON_UNIT, n, n,
                                &one, T.p, n, Z.p, n));
            zero_z = false;
        };
        for (int k = 0; k < pre_sweeps; ++k) sweep();
        // coarse correction: Z += P Vc R (I - A Z)
        identity(M, n, s);
        if (!zero_z)
            ED_BLAS(cublasDgemm(h, CUBLAS_OP_N, CUBLAS_OP_N, n, n, n, &mone, A.p, n, Z.p, n, &one, M.p, n));
        densify(*L.R, Rd, s); // ncur x n
        densify(*L.P, Pd, s); // n x ncur
        Rc.alloc(static_cast<size_t>(ncur) * n);
        ED_BLAS(cublasDgemm(h, CUBLAS_OP_N, CUBLAS_OP_N, ncur, n, n, &one, Rd.p, ncur, M.p, n, &zero, Rc.p, ncur));
        Ec.alloc(Rc.n);
        ED_BLAS(cublasDgemm(h, CUBLAS_OP_N, CUBLAS_OP_N, ncur, n, ncur, &one, Vc.p, ncur, Rc.p, ncur, &zero, Ec.p,
                            ncur));
        ED_BLAS(cublasDgemm(h, CUBLAS_OP_N, CUBLAS_OP_N, n, n, ncur, &one, Pd.p, n, Ec.p, ncur, zero_z ? &zero : &one,
                            Z.p, n));
        zero_z = false;
        for (int k = 0; k < post_sweeps; ++k) sweep();
        Vc = std::move(Z);
        ncur = n;
    }
    // row-major copy for dense_gemv
    out.alloc(static_cast<size_t>(ncur) * ncur);
    ED_BLAS(cublasDgeam(h, CUBLAS_OP_T, CUBLAS_OP_N, ncur, ncur, &one, Vc.p, ncur, &zero, Vc.p, ncur, out.p, ncur));
}

} // namespace edb
