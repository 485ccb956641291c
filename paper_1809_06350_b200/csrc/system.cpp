// Block-system construction: node-graph patterns and BSR layouts, element
// colouring and element->K4 maps (mesh-static, built once), planes from K4 or
// from caller CSR, the working copy with symmetric block scaling
// (blocksystem.cpp:53-106) and S_hat (precond.cpp:10-24).
#include <omp.h>

#include <algorithm>
#include <numeric>

#include "ctx.hpp"

namespace edb {

void BlockSys::build_structure(cudaStream_t s)
{
    if (!pattern_symmetric(pA))
        throw Error(ED_UNSUPPORTED, "velocity block pattern is not structurally symmetric");
    std::vector<int> order, lvl;
    int nlev = 0;
    gs_level_order(pA, order, lvl, nlev);
    lA = make_layout(pA, order, lvl);
    lB = make_layout(pB, order, lvl); // same slicing as A
    std::vector<int> porder(pD.nbr);
    std::iota(porder.begin(), porder.end(), 0);
    lC = make_layout(pC, porder, {});
    lD = make_layout(pD, porder, {}); // same slicing as C
    A.st = bsr_make_struct(pA, lA, Bv, Bv, s);
    B.st = bsr_make_struct(pB, lB, Bv, 1, s);
    C.st = bsr_make_struct(pC, lC, 1, Bv, s);
    D.st = bsr_make_struct(pD, lD, 1, 1, s);
    A.val.alloc(A.st->nval());
    B.val.alloc(B.st->nval());
    C.val.alloc(C.st->nval());
    D.val.alloc(D.st->nval());
    A.val.zero(s);
    B.val.zero(s);
    C.val.zero(s);
    D.val.zero(s);
    shat_symbolic = false;
    sS.reset();
}

// Pattern of S_hat = D - C diag(A)^-1 B (csr_matmul + csr_add keep every
// structurally touched entry) and the position maps the numeric kernel uses.
void BlockSys::build_shat_symbolic(cudaStream_t s)
{
    const int np_ = pD.nbr;
    BlockPattern pS;
    pS.nbr = pS.nbc = np_;
    pS.rowptr.assign(np_ + 1, 0);
    std::vector<std::vector<int>> rows(np_);
#pragma omp parallel
    {
        std::vector<int> mark(np_, -1);
#pragma omp for schedule(dynamic, 1024)
        for (int p = 0; p < np_; ++p) {
            std::vector<int>& r = rows[p];
            for (int64_t k = pD.rowptr[p]; k < pD.rowptr[p + 1]; ++k) {
                const int q = pD.col[k];
                if (mark[q] != p) {
                    mark[q] = p;
                    r.push_back(q);
                }
            }
            for (int64_t k = pC.rowptr[p]; k < pC.rowptr[p + 1]; ++k) {
                const int m = pC.col[k];
                for (int64_t kb = pB.rowptr[m]; kb < pB.rowptr[m + 1]; ++kb) {
                    const int q = pB.col[kb];
                    if (mark[q] != p) {
                        mark[q] = p;
                        r.push_back(q);
                    }
                }
            }
            std::sort(r.begin(), r.end());
        }
    }
    for (int p = 0; p < np_; ++p) {
        if (rows[p].size() > 65535) throw Error(ED_UNSUPPORTED, "S_hat row longer than 65535 entries");
        pS.rowptr[p + 1] = pS.rowptr[p] + static_cast<int64_t>(rows[p].size());
    }
    pS.col.resize(pS.rowptr[np_]);
    for (int p = 0; p < np_; ++p) std::copy(rows[p].begin(), rows[p].end(), pS.col.begin() + pS.rowptr[p]);
    rows.clear();
    rows.shrink_to_fit();
    shat_nnz = pS.nnzb();

    std::vector<int64_t> hcb_off(np_ + 1, 0), hd_off(np_ + 1, 0);
    for (int p = 0; p < np_; ++p) {
        int64_t cnt = 0;
        for (int64_t k = pC.rowptr[p]; k < pC.rowptr[p + 1]; ++k) {
            const int m = pC.col[k];
            cnt += pB.rowptr[m + 1] - pB.rowptr[m];
        }
        hcb_off[p + 1] = hcb_off[p] + cnt;
        hd_off[p + 1] = hd_off[p] + (pD.rowptr[p + 1] - pD.rowptr[p]);
    }
    std::vector<uint16_t> hcb(hcb_off[np_]), hd(hd_off[np_]);
#pragma omp parallel for schedule(dynamic, 1024)
    for (int p = 0; p < np_; ++p) {
        const auto b = pS.col.begin() + pS.rowptr[p], e = pS.col.begin() + pS.rowptr[p + 1];
        auto pos = [&](int q) { return static_cast<uint16_t>(std::lower_bound(b, e, q) - b); };
        int64_t o = hcb_off[p];
        for (int64_t k = pC.rowptr[p]; k < pC.rowptr[p + 1]; ++k) {
            const int m = pC.col[k];
            for (int64_t kb = pB.rowptr[m]; kb < pB.rowptr[m + 1]; ++kb) hcb[o++] = pos(pB.col[kb]);
        }
        int64_t od = hd_off[p];
        for (int64_t k = pD.rowptr[p]; k < pD.rowptr[p + 1]; ++k) hd[od++] = pos(pD.col[k]);
    }
    if (!pattern_symmetric(pS)) throw Error(ED_UNSUPPORTED, "S_hat pattern is not structurally symmetric");
    std::vector<int> order, lvl;
    int nlev = 0;
    gs_level_order(pS, order, lvl, nlev);
    BsrLayout lS = make_layout(pS, order, lvl);
    sS = bsr_make_struct(pS, lS, 1, 1, s);
    cb_off.upload(hcb_off, s);
    d_off.upload(hd_off, s);
    cb_pos.upload(hcb, s);
    d_pos.upload(hd, s);
    ED_CUDA(cudaStreamSynchronize(s));
    shat_symbolic = true;
}

void ctx_build_mesh_system(Ctx& c)
{
    cudaStream_t s = c.stream;
    const int N = c.n_nodes, E = c.n_tets;
    const std::vector<int>& T = c.h_tets;
    // node -> elements
    std::vector<int64_t> ne_ptr(N + 1, 0);
    for (int64_t k = 0; k < 4LL * E; ++k) ++ne_ptr[T[k] + 1];
    for (int n = 0; n < N; ++n) ne_ptr[n + 1] += ne_ptr[n];
    std::vector<int> ne(ne_ptr[N]);
    {
        std::vector<int64_t> next(ne_ptr.begin(), ne_ptr.end() - 1);
        for (int e = 0; e < E; ++e)
            for (int a = 0; a < 4; ++a) ne[next[T[4LL * e + a]]++] = e;
    }
    // node graph PN (sorted, includes self)
    std::vector<std::vector<int>> adj(N);
#pragma omp parallel for schedule(dynamic, 1024)
    for (int n = 0; n < N; ++n) {
        auto& l = adj[n];
        for (int64_t k = ne_ptr[n]; k < ne_ptr[n + 1]; ++k)
            for (int a = 0; a < 4; ++a) l.push_back(T[4LL * ne[k] + a]);
        std::sort(l.begin(), l.end());
        l.erase(std::unique(l.begin(), l.end()), l.end());
    }
    BlockPattern& PN = c.PN;
    PN.nbr = PN.nbc = N;
    PN.rowptr.assign(N + 1, 0);
    for (int n = 0; n < N; ++n) PN.rowptr[n + 1] = PN.rowptr[n] + static_cast<int64_t>(adj[n].size());
    PN.col.resize(PN.rowptr[N]);
    for (int n = 0; n < N; ++n) std::copy(adj[n].begin(), adj[n].end(), PN.col.begin() + PN.rowptr[n]);
    adj.clear();
    adj.shrink_to_fit();
    if (PN.nnzb() >= (1LL << 31)) throw Error(ED_UNSUPPORTED, "node graph exceeds int32 block indices");

    // element -> K4 slot of node pair (a, b)
    std::vector<int> k4slot(16LL * E);
#pragma omp parallel for schedule(static)
    for (int e = 0; e < E; ++e)
        for (int a = 0; a < 4; ++a) {
            const int na = T[4LL * e + a];
            const auto b0 = PN.col.begin() + PN.rowptr[na], b1 = PN.col.begin() + PN.rowptr[na + 1];
            for (int b = 0; b < 4; ++b) {
                const int nb = T[4LL * e + b];
                k4slot[16LL * e + 4 * a + b] = static_cast<int>(PN.rowptr[na] + (std::lower_bound(b0, b1, nb) - b0));
            }
        }
    c.k4slot.upload(k4slot, s);

    // greedy element colouring: no two elements of one colour share a node
    std::vector<uint64_t> used(N, 0);
    std::vector<int> color(E);
    int ncol = 0;
    for (int e = 0; e < E; ++e) {
        uint64_t m = 0;
        for (int a = 0; a < 4; ++a) m |= used[T[4LL * e + a]];
        if (m == ~0ULL) throw Error(ED_UNSUPPORTED, "element colouring needs more than 64 colours");
        const int col = __builtin_ctzll(~m);
        color[e] = col;
        ncol = std::max(ncol, col + 1);
        for (int a = 0; a < 4; ++a) used[T[4LL * e + a]] |= (1ULL << col);
    }
    c.color_ptr.assign(ncol + 1, 0);
    for (int e = 0; e < E; ++e) ++c.color_ptr[color[e] + 1];
    for (int k = 0; k < ncol; ++k) c.color_ptr[k + 1] += c.color_ptr[k];
    std::vector<int> order(E);
    {
        std::vector<int> next(c.color_ptr.begin(), c.color_ptr.end() - 1);
        for (int e = 0; e < E; ++e) order[next[color[e]]++] = e;
    }
    c.elem_order.upload(order, s);
    c.k4.alloc(16 * static_cast<size_t>(PN.nnzb()));

    // plane patterns over free nodes (Bv = 3) and their K4 sources
    BlockSys& S = c.sys;
    S.Bv = 3;
    S.nv = 3 * c.nfree;
    S.np = N;
    const int F = c.nfree;
    auto& fidx = c.fidx;
    auto& fnode = c.fnode;
    std::vector<int64_t> srcA, srcB, srcC, srcD;
    S.pA = BlockPattern{};
    S.pA.nbr = S.pA.nbc = F;
    S.pA.rowptr.assign(F + 1, 0);
    S.pB = BlockPattern{};
    S.pB.nbr = F;
    S.pB.nbc = N;
    S.pB.rowptr.assign(F + 1, 0);
    for (int f = 0; f < F; ++f) {
        const int n = fnode[f];
        for (int64_t k = PN.rowptr[n]; k < PN.rowptr[n + 1]; ++k) {
            const int m = PN.col[k];
            if (fidx[m] >= 0) {
                S.pA.col.push_back(fidx[m]);
                srcA.push_back(k);
            }
            S.pB.col.push_back(m);
            srcB.push_back(k);
        }
        S.pA.rowptr[f + 1] = static_cast<int64_t>(S.pA.col.size());
        S.pB.rowptr[f + 1] = static_cast<int64_t>(S.pB.col.size());
    }
    S.pC = BlockPattern{};
    S.pC.nbr = N;
    S.pC.nbc = F;
    S.pC.rowptr.assign(N + 1, 0);
    for (int n = 0; n < N; ++n) {
        for (int64_t k = PN.rowptr[n]; k < PN.rowptr[n + 1]; ++k) {
            const int m = PN.col[k];
            if (fidx[m] >= 0) {
                S.pC.col.push_back(fidx[m]);
                srcC.push_back(k);
            }
        }
        S.pC.rowptr[n + 1] = static_cast<int64_t>(S.pC.col.size());
    }
    S.pD = PN;
    srcD.resize(PN.nnzb());
    std::iota(srcD.begin(), srcD.end(), 0);
    S.build_structure(s);
    auto stored_src = [&](const BsrLayout& L, const std::vector<int64_t>& src, DevArray<int>& out) {
        std::vector<int> v(src.size(), -1);
        for (size_t k = 0; k < src.size(); ++k) v[L.addr[k]] = static_cast<int>(src[k]);
        out.upload(v, s);
        ED_CUDA(cudaStreamSynchronize(s));
    };
    stored_src(S.lA, srcA, c.srcA);
    stored_src(S.lB, srcB, c.srcB);
    stored_src(S.lC, srcC, c.srcC);
    stored_src(S.lD, srcD, c.srcD);
    auto slot_dst = [&](const BsrLayout& L, const std::vector<int64_t>& src, DevArray<int>& out) {
        std::vector<int> v(PN.nnzb(), -1);
        for (size_t k = 0; k < src.size(); ++k) v[src[k]] = static_cast<int>(L.addr[k]);
        out.upload(v, s);
        ED_CUDA(cudaStreamSynchronize(s));
    };
    slot_dst(S.lA, srcA, c.dstA);
    slot_dst(S.lB, srcB, c.dstB);
    slot_dst(S.lC, srcC, c.dstC);
    slot_dst(S.lD, srcD, c.dstD);
    {
        std::vector<int2> cf(PN.nnzb());
        for (int64_t k = 0; k < PN.nnzb(); ++k) cf[k] = make_int2(PN.col[k], fidx[PN.col[k]]);
        c.k44_cf.upload(cf, s);
        ED_CUDA(cudaStreamSynchronize(s));
    }
    c.sys_from_mesh = true;
    c.sys_values = false;
    ED_CUDA(cudaStreamSynchronize(s));
}

void ctx_planes_from_k4(Ctx& c)
{
    BlockSys& S = c.sys;
    cudaStream_t s = c.stream;
    launch_k4_split(c.k4.p, c.dstA.p, c.dstB.p, c.dstC.p, c.dstD.p, S.A.val.p, S.B.val.p, S.C.val.p, S.D.val.p,
                    S.D.st->nnzb, s);
    c.sys_values = true;
}

void ctx_planes_from_csr(Ctx& c, int Bv)
{
    if (c.csr_up.size() != 4) throw Error(ED_NOT_READY, "no block system uploaded");
    if (c.csr_bv == Bv && c.sys.valid()) return;
    cudaStream_t s = c.stream;
    BlockSys& S = c.sys;
    S = BlockSys{};
    S.Bv = Bv;
    S.nv = c.csr_up[0].nrows;
    S.np = c.csr_up[3].nrows;
    S.pA = block_pattern_of_csr(c.csr_up[0], Bv, Bv);
    S.pB = block_pattern_of_csr(c.csr_up[1], Bv, 1);
    S.pC = block_pattern_of_csr(c.csr_up[2], 1, Bv);
    S.pD = block_pattern_of_csr(c.csr_up[3], 1, 1);
    S.build_structure(s);
    S.A.val.upload(bsr_pack_values(*S.A.st, S.lA, block_values_of_csr(c.csr_up[0], S.pA, Bv, Bv)), s);
    ED_CUDA(cudaStreamSynchronize(s));
    S.B.val.upload(bsr_pack_values(*S.B.st, S.lB, block_values_of_csr(c.csr_up[1], S.pB, Bv, 1)), s);
    ED_CUDA(cudaStreamSynchronize(s));
    S.C.val.upload(bsr_pack_values(*S.C.st, S.lC, block_values_of_csr(c.csr_up[2], S.pC, 1, Bv)), s);
    ED_CUDA(cudaStreamSynchronize(s));
    S.D.val.upload(bsr_pack_values(*S.D.st, S.lD, block_values_of_csr(c.csr_up[3], S.pD, 1, 1)), s);
    ED_CUDA(cudaStreamSynchronize(s));
    c.csr_bv = Bv;
    c.sys_values = true;
}

// Working copy K_s = W K W, b = W rhs (precond.cpp:163-177)
void make_work(Ctx& c, WorkSys& W, bool scale, double eps_diag)
{
    cudaStream_t s = c.stream;
    BlockSys& S = c.sys;
    W.Bv = S.Bv;
    W.nv = S.nv;
    W.np = S.np;
    W.A.copy_values_from(S.A, s);
    W.B.copy_values_from(S.B, s);
    W.C.copy_values_from(S.C, s);
    W.D.copy_values_from(S.D, s);
    W.scaled = scale;
    const int nv = S.nv, np = S.np;
    W.w.alloc(static_cast<size_t>(nv) + np);
    // the coupled 4x4 operator from the assembled node blocks (scaling folded in below)
    const bool coupled = c.sys_from_mesh && S.Bv == 3 && c.k4.p && std::getenv("ED_NO_K44") == nullptr;
    W.K.n_nodes = 0;
    if (coupled) {
        W.K.n_nodes = S.D.st->nbr;
        W.K.nnzb = S.D.st->nnzb;
        W.K.rowptr = S.D.st->rowptr.p;
        W.K.col = S.D.st->col.p;
        W.K.fidx = c.d_fidx.p;
        W.K.cf = c.k44_cf.p;
        W.K.val.alloc(16 * static_cast<size_t>(W.K.nnzb));
    }
    if (!scale) {
        if (coupled) k44_build(W.K, c.k4.p, nullptr, nv, s);
        return;
    }
    DevArray<double> da(nv), dd(np), mx(2);
    bsr_diag(W.A, da.p, s);
    bsr_diag(W.D, dd.p, s);
    absmax(c.red, da.p, nv, mx.p + 0, s);
    absmax(c.red, dd.p, np, mx.p + 1, s);
    block_weights(da.p, dd.p, nv, np, mx.p + 0, mx.p + 1, eps_diag, W.w.p, s);
    const double* wv = W.w.p;
    const double* wp = W.w.p + nv;
    bsr_scale(W.A, wv, wv, s);
    bsr_scale(W.B, wv, wp, s);
    bsr_scale(W.C, wp, wv, s);
    bsr_scale(W.D, wp, wp, s);
    if (coupled) k44_build(W.K, c.k4.p, W.w.p, nv, s);
    ED_CUDA(cudaStreamSynchronize(s)); // temporaries die here
}

// build_shat on the working system (precond.cpp:10-24)
void build_shat_work(Ctx& c, WorkSys& W)
{
    cudaStream_t s = c.stream;
    BlockSys& S = c.sys;
    if (!S.shat_symbolic) S.build_shat_symbolic(s);
    DevArray<double> da(W.nv), inv_da(W.nv);
    bsr_diag(W.A, da.p, s);
    const int big = 0x7fffffff;
    ED_CUDA(cudaMemcpyAsync(c.dscratch_i.p + 1, &big, sizeof(int), cudaMemcpyHostToDevice, s));
    shat_inv_diag(da.p, inv_da.p, W.nv, 1e-300, c.dscratch_i.p + 1, s);
    const int bad = c.read_int(c.dscratch_i.p + 1);
    if (bad != big)
        throw Error(ED_ZERO_DIAGONAL, "build_shat: zero diagonal in momentum block at row " + std::to_string(bad), bad);
    W.S.st = S.sS;
    W.S.val.alloc(S.sS->nval());
    ShatArgs a{};
    const BsrStruct& SS = *S.sS;
    a.s_rowptr = SS.rowptr.p;
    a.s_perm = SS.perm.p;
    a.s_val = W.S.val.p;
    a.s_nrows = SS.nbr;
    if (!W.C.st->h_perm.empty() || !W.D.st->h_perm.empty()) throw Error(ED_INVALID_ARGUMENT, "C/D must be in natural order");
    a.c_rowptr = W.C.st->rowptr.p;
    a.c_col = W.C.st->col.p;
    a.c_val = W.C.val.p;
    a.d_rowptr = W.D.st->rowptr.p;
    a.d_val = W.D.val.p;
    a.b_rowptr = W.B.st->rowptr.p;
    a.b_inv = W.B.st->inv.p;
    a.b_val = W.B.val.p;
    a.inv_da = inv_da.p;
    a.cb_off = S.cb_off.p;
    a.cb_pos = S.cb_pos.p;
    a.d_off = S.d_off.p;
    a.d_pos = S.d_pos.p;
    a.Bv = W.Bv;
    launch_shat_numeric(a, s);
    ED_CUDA(cudaStreamSynchronize(s));
}

} // namespace edb
