// ILU(0) preconditioner on the monolithic (scaled) block system
// (Ilu0Precond, ilu0.cpp:9-68; monolithic_csr, blocksystem.cpp:10-56): the
// PrecondKind::Ilu0 baseline of solve_block_system.
//
// Both the factorization and the two triangular solves are sequential over
// rows in the reference.  Here every row is placed on a dependency level
// (factorization and forward solve: the lower pattern; backward solve: the
// upper pattern) and one CTA walks the levels with a barrier between them,
// one thread per row.  Inside a row the operations run in the reference's
// order with multiply and add rounded separately, so the factors and the
// solves are bitwise the reference's.  The monolithic pattern is built on the
// host from the device planes (a copy, no arithmetic).
#include <cuda_runtime.h>

#include <algorithm>
#include <climits>
#include <string>
#include <vector>

#include "ed_internal.hpp"

namespace edb {
namespace {

constexpr int kT = 1024;

__global__ void __launch_bounds__(kT) k_ilu0_factor(const int* __restrict__ rowptr, const int* __restrict__ col,
                                                    const int* __restrict__ dpos, double* val,
                                                    const int* __restrict__ lev_ptr, const int* __restrict__ rows,
                                                    int nlev, int* bad)
{
    for (int l = 0; l < nlev; ++l) {
        for (int t = lev_ptr[l] + threadIdx.x; t < lev_ptr[l + 1]; t += blockDim.x) {
            const int i = rows[t];
            const int ei = rowptr[i + 1];
            for (int kk = rowptr[i]; kk < dpos[i]; ++kk) {
                const int k = col[kk];
                const double piv = val[dpos[k]];
                if (piv == 0.0) {
                    atomicMin(bad, k);
                    break;
                }
                const double lik = __ddiv_rn(val[kk], piv);
                val[kk] = lik;
                // subtract lik * U(k, j) from row i on the pattern intersection
                int pi = kk + 1, pk = dpos[k] + 1;
                const int ek = rowptr[k + 1];
                while (pi < ei && pk < ek) {
                    const int ci = col[pi], ck = col[pk];
                    if (ci < ck) {
                        ++pi;
                    } else if (ci > ck) {
                        ++pk;
                    } else {
                        val[pi] = __dsub_rn(val[pi], __dmul_rn(lik, val[pk]));
                        ++pi;
                        ++pk;
                    }
                }
            }
            if (val[dpos[i]] == 0.0) atomicMin(bad, i);
        }
        __syncthreads();
    }
}

// forward L z = r (unit diagonal), then backward U z = z (ilu0.cpp:54-68)
__global__ void __launch_bounds__(kT) k_ilu0_apply(const int* __restrict__ rowptr, const int* __restrict__ col,
                                                   const int* __restrict__ dpos, const double* __restrict__ val,
                                                   const int* __restrict__ lf_ptr, const int* __restrict__ rows_f,
                                                   int nlf, const int* __restrict__ lb_ptr,
                                                   const int* __restrict__ rows_b, int nlb, const double* r, double* z)
{
    for (int l = 0; l < nlf; ++l) {
        for (int t = lf_ptr[l] + threadIdx.x; t < lf_ptr[l + 1]; t += blockDim.x) {
            const int i = rows_f[t];
            double acc = r[i];
            for (int kk = rowptr[i]; kk < dpos[i]; ++kk) acc = __dsub_rn(acc, __dmul_rn(val[kk], z[col[kk]]));
            z[i] = acc;
        }
        __syncthreads();
    }
    for (int l = 0; l < nlb; ++l) {
        for (int t = lb_ptr[l] + threadIdx.x; t < lb_ptr[l + 1]; t += blockDim.x) {
            const int i = rows_b[t];
            double acc = z[i];
            for (int kk = dpos[i] + 1; kk < rowptr[i + 1]; ++kk) acc = __dsub_rn(acc, __dmul_rn(val[kk], z[col[kk]]));
            z[i] = __ddiv_rn(acc, val[dpos[i]]);
        }
        __syncthreads();
    }
}

// rows grouped by level (counting sort), stable in row order
void group_levels(const std::vector<int>& level, int nlev, std::vector<int>& ptr, std::vector<int>& rows)
{
    ptr.assign(nlev + 1, 0);
    for (const int l : level) ++ptr[l + 1];
    for (int l = 0; l < nlev; ++l) ptr[l + 1] += ptr[l];
    rows.assign(level.size(), 0);
    std::vector<int> at(ptr.begin(), ptr.end() - 1);
    for (int i = 0; i < static_cast<int>(level.size()); ++i) rows[at[level[i]]++] = i;
}

} // namespace

void ilu0_build(const WorkSysView& W, DevIlu0& f, cudaStream_t s)
{
    const HostCsr A = bsr_to_csr(*W.A, s), B = bsr_to_csr(*W.B, s), C = bsr_to_csr(*W.C, s),
                  D = bsr_to_csr(*W.D, s);
    const int nv = A.nrows, np = D.nrows, n = nv + np;
    std::vector<int> rp(n + 1, 0), cl, dp(n, -1);
    std::vector<double> vl;
    cl.reserve(A.nnz() + B.nnz() + C.nnz() + D.nnz());
    vl.reserve(cl.capacity());
    auto append = [&](const HostCsr& M, int r, int off) {
        for (int64_t k = M.rowptr[r]; k < M.rowptr[r + 1]; ++k) {
            cl.push_back(M.col[k] + off);
            vl.push_back(M.val[k]);
        }
    };
    for (int r = 0; r < nv; ++r) {
        append(A, r, 0);
        append(B, r, nv);
        rp[r + 1] = static_cast<int>(cl.size());
    }
    for (int r = 0; r < np; ++r) {
        append(C, r, 0);
        append(D, r, nv);
        rp[nv + r + 1] = static_cast<int>(cl.size());
    }
    for (int r = 0; r < n; ++r) {
        for (int k = rp[r]; k < rp[r + 1]; ++k)
            if (cl[k] == r) dp[r] = k;
        if (dp[r] < 0) throw Error(ED_ZERO_DIAGONAL, "ilu0: missing diagonal entry in row " + std::to_string(r), r);
    }
    // levels: forward (factorization, L solve) over the lower pattern, backward over the upper
    std::vector<int> lf(n, 0), lb(n, 0);
    int nlf = 1, nlb = 1;
    for (int i = 0; i < n; ++i) {
        int l = 0;
        for (int k = rp[i]; k < dp[i]; ++k) l = std::max(l, lf[cl[k]] + 1);
        lf[i] = l;
        nlf = std::max(nlf, l + 1);
    }
    for (int i = n - 1; i >= 0; --i) {
        int l = 0;
        for (int k = dp[i] + 1; k < rp[i + 1]; ++k) l = std::max(l, lb[cl[k]] + 1);
        lb[i] = l;
        nlb = std::max(nlb, l + 1);
    }
    std::vector<int> fptr, frows, bptr, brows;
    group_levels(lf, nlf, fptr, frows);
    group_levels(lb, nlb, bptr, brows);
    f.n = n;
    f.nlf = nlf;
    f.nlb = nlb;
    f.rowptr.upload(rp, s);
    f.col.upload(cl, s);
    f.dpos.upload(dp, s);
    f.val.upload(vl, s);
    f.lf_ptr.upload(fptr, s);
    f.rows_f.upload(frows, s);
    f.lb_ptr.upload(bptr, s);
    f.rows_b.upload(brows, s);
    DevArray<int> bad(1);
    const std::vector<int> big{INT_MAX};
    bad.upload(big, s);
    k_ilu0_factor<<<1, kT, 0, s>>>(f.rowptr.p, f.col.p, f.dpos.p, f.val.p, f.lf_ptr.p, f.rows_f.p, nlf, bad.p);
    after_launch("k_ilu0_factor");
    const int b = bad.to_host(s)[0];
    if (b != INT_MAX) throw Error(ED_ZERO_DIAGONAL, "ilu0: zero pivot at row " + std::to_string(b), b);
}

void ilu0_apply(const DevIlu0& f, const double* r, double* z, cudaStream_t s)
{
    k_ilu0_apply<<<1, kT, 0, s>>>(f.rowptr.p, f.col.p, f.dpos.p, f.val.p, f.lf_ptr.p, f.rows_f.p, f.nlf, f.lb_ptr.p,
                                  f.rows_b.p, f.nlb, r, z);
    after_launch("k_ilu0_apply");
}

} // namespace edb
