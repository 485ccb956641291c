// Coupled 4x4 BSR operator of the block system (BlockMatrix::matvec,
// blocksystem.hpp:27-33) for sm_100a.
//
// For a mesh-assembled system the solver keeps, next to its A/B/C/D planes,
// the scaled coupled operator K = [A B; C D] as a true 4x4 BSR over the node
// graph: one block column index per node-graph edge and 16 doubles (128 B,
// rows v0 v1 v2 p x columns v0 v1 v2 p) per block -- exactly the storage the
// SURVEY's coupled-SpMV byte count assumes (nnzb * (128 + 4) + row pointers +
// vectors).  Velocity rows/columns of fixed nodes are zero.  It is built once
// per solve from the assembled node blocks (K4) with the solver's symmetric
// scaling folded in (the same product w_r * w_c as the planes' k_scale, so
// the entries equal the scaled planes' bitwise), and drives the outer
// FGMRES's K x: the 8 lanes of a node row stream each 128-B block with 16-B loads.
#include <cuda_runtime.h>

#include "ed_internal.hpp"

namespace edb {

namespace {

constexpr int kCT = 256;

// K44[k] = (w_r (x) w_c) o K4[k]; fixed velocity dofs -> 0.  One thread per block.
__global__ void k_k44_build(const int* __restrict__ rowptr, const int* __restrict__ col, int n_nodes,
                            const double* __restrict__ k4, const int* __restrict__ fidx,
                            const double* __restrict__ w, int nv, double* __restrict__ k44)
{
    const int r = blockIdx.x * (kCT / 8) + threadIdx.x / 8;
    const int lane = threadIdx.x % 8;
    if (r >= n_nodes) return;
    const int fr = fidx[r];
    double wr[4];
#pragma unroll
    for (int i = 0; i < 3; ++i) wr[i] = fr >= 0 ? (w ? w[3 * static_cast<int64_t>(fr) + i] : 1.0) : 0.0;
    wr[3] = w ? w[nv + r] : 1.0;
    for (int k = rowptr[r] + lane; k < rowptr[r + 1]; k += 8) {
        const int c = col[k];
        const int fc = fidx[c];
        double wc[4];
#pragma unroll
        for (int j = 0; j < 3; ++j) wc[j] = fc >= 0 ? (w ? w[3 * static_cast<int64_t>(fc) + j] : 1.0) : 0.0;
        wc[3] = w ? w[nv + c] : 1.0;
        const double2* src = reinterpret_cast<const double2*>(k4 + 16 * static_cast<int64_t>(k));
        double2* dst = reinterpret_cast<double2*>(k44 + 16 * static_cast<int64_t>(k));
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            const double2 v = __ldg(src + q);
            const int i = q / 2, j = 2 * (q % 2);
            double2 o;
            o.x = (wr[i] == 0.0 || wc[j] == 0.0) ? 0.0 : v.x * (wr[i] * wc[j]);
            o.y = (wr[i] == 0.0 || wc[j + 1] == 0.0) ? 0.0 : v.y * (wr[i] * wc[j + 1]);
            dst[q] = o;
        }
    }
}

// y = K x, x = [x_v (free velocity dofs); x_p (nodes)].  The 8 lanes of a node
// row share every block: lane q owns the 16-B piece q (block row q/2, columns
// 2(q%2), 2(q%2)+1), so one warp instruction reads four whole 128-B lines
// (LDG.E.128, every sector used once); a block's column comes with its free
// velocity index (int2 {node, free index}, one broadcast load per group), and
// PB blocks of the row are in flight per lane.  Measured at 160^3
// (profiles/r02/spmv_variants_160.txt): 1.49 ms = 87 % of the measured HBM
// peak; one lane per whole block (8 x LDG.128 to 32 different lines per
// instruction) reached 56 %, streaming (evict-first) loads did not help.
template <int PB>
__global__ void __launch_bounds__(kCT) k_spmv44(const int* __restrict__ rowptr, const int2* __restrict__ cf,
                                                 int n_nodes, const double* __restrict__ k44,
                                                 const int* __restrict__ fidx, int nv, const double* __restrict__ x,
                                                 double* __restrict__ y)
{
    const int64_t gid = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const int r = static_cast<int>(gid >> 3);
    const int q = static_cast<int>(gid & 7);
    const int half = q & 1;
    double acc = 0.0;
    if (r < n_nodes) {
        const int k1 = rowptr[r + 1];
        const double2* base = reinterpret_cast<const double2*>(k44) + q;
        for (int k0 = rowptr[r]; k0 < k1; k0 += PB) {
            int2 c[PB];
            double2 v[PB];
#pragma unroll
            for (int p = 0; p < PB; ++p) {
                const int k = k0 + p;
                const bool in = k < k1;
                const int kk = in ? k : k0;
                c[p] = __ldg(cf + kk);
                v[p] = __ldg(base + 8 * static_cast<int64_t>(kk));
                if (!in) v[p] = make_double2(0.0, 0.0);
            }
#pragma unroll
            for (int p = 0; p < PB; ++p) {
                // half 0: x_v[3 fc], x_v[3 fc + 1]; half 1: x_v[3 fc + 2], x_p[c]
                const int fc = c[p].y;
                const double x0 = fc >= 0 ? __ldg(x + 3 * static_cast<int64_t>(fc) + 2 * half) : 0.0;
                const double x1 = half ? __ldg(x + nv + c[p].x)
                                       : (fc >= 0 ? __ldg(x + 3 * static_cast<int64_t>(fc) + 1) : 0.0);
                acc = fma(v[p].x, x0, acc);
                acc = fma(v[p].y, x1, acc);
            }
        }
    }
    acc += __shfl_xor_sync(0xffffffffu, acc, 1);
    if (r < n_nodes && half == 0) {
        const int i = q >> 1;
        if (i == 3) {
            y[nv + r] = acc;
        } else {
            const int fr = fidx[r];
            if (fr >= 0) y[3 * static_cast<int64_t>(fr) + i] = acc;
        }
    }
}

} // namespace

void k44_build(const CoupledOp& K, const double* k4, const double* w, int nv, cudaStream_t s)
{
    if (K.n_nodes == 0) return;
    const int g = (K.n_nodes + kCT / 8 - 1) / (kCT / 8);
    k_k44_build<<<g, kCT, 0, s>>>(K.rowptr, K.col, K.n_nodes, k4, K.fidx, w, nv, K.val.p);
    after_launch("k_k44_build");
}

void spmv44(const CoupledOp& K, const double* x, double* y, int nv, int np, cudaStream_t s)
{
    if (K.n_nodes == 0) return;
    AcctScope acct(s, "k_spmv44", K.bytes(static_cast<int64_t>(nv) + np));
    const int64_t threads = static_cast<int64_t>(K.n_nodes) * 8;
    k_spmv44<4><<<static_cast<unsigned>((threads + kCT - 1) / kCT), kCT, 0, s>>>(K.rowptr, K.cf, K.n_nodes, K.val.p,
                                                                                 K.fidx, nv, x, y);
    after_launch("k_spmv44");
}

} // namespace edb
