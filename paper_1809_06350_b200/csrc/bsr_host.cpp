// Host construction of level-ordered BSR operators, Gauss-Seidel level
// schedules and dataflow work items.  Structure is
// mesh-static: built once per mesh (or per AMG level); only values move per
// Newton step.
#include <algorithm>
#include <cstdlib>
#include <numeric>

#include "ed_internal.hpp"

namespace edb {

double Bsr::bytes_per_spmv() const
{
    const BsrStruct& S = *st;
    const double blk = 8.0 * S.Rb * S.Cb + 4.0;
    return static_cast<double>(S.nnzb) * blk + 4.0 * (S.nbr + 1) + 8.0 * S.nbr * S.Rb + 8.0 * S.nbc * S.Cb;
}

void gs_level_order(const BlockPattern& pat, std::vector<int>& order, std::vector<int>& level_of_pos, int& nlev)
{
    const int n = pat.nbr;
    std::vector<int> level(n, 0);
    nlev = n > 0 ? 1 : 0;
    // Row i reads the NEW value of every j < i it couples to (amg.cpp:311-316),
    // so it sits one level above the highest such j.
    for (int i = 0; i < n; ++i) {
        int lv = 0;
        for (int64_t k = pat.rowptr[i]; k < pat.rowptr[i + 1]; ++k) {
            const int j = pat.col[k];
            if (j < i) lv = std::max(lv, level[j] + 1);
        }
        level[i] = lv;
        nlev = std::max(nlev, lv + 1);
    }
    std::vector<int> cnt(nlev + 1, 0);
    for (int i = 0; i < n; ++i) ++cnt[level[i] + 1];
    for (int l = 0; l < nlev; ++l) cnt[l + 1] += cnt[l];
    order.assign(n, 0);
    level_of_pos.assign(n, 0);
    for (int i = 0; i < n; ++i) {
        const int pos = cnt[level[i]]++;
        order[pos] = i;
        level_of_pos[pos] = level[i];
    }
}

bool pattern_symmetric(const BlockPattern& pat)
{
    if (pat.nbr != pat.nbc) return false;
    int bad = 0;
#pragma omp parallel for schedule(dynamic, 256) reduction(| : bad)
    for (int i = 0; i < pat.nbr; ++i)
        for (int64_t k = pat.rowptr[i]; k < pat.rowptr[i + 1] && !bad; ++k) {
            const int j = pat.col[k];
            const auto b = pat.col.begin() + pat.rowptr[j];
            const auto e = pat.col.begin() + pat.rowptr[j + 1];
            if (!std::binary_search(b, e, i)) bad = 1;
        }
    return bad == 0;
}

BsrLayout make_layout(const BlockPattern& pat, const std::vector<int>& row_order, const std::vector<int>& level_of_pos)
{
    BsrLayout L;
    const int n = pat.nbr;
    L.perm = row_order;
    L.inv.assign(n, -1);
    for (int s = 0; s < n; ++s) L.inv[row_order[s]] = s;
    L.lev_ptr.push_back(0);
    for (int s = 1; s < n; ++s)
        if (!level_of_pos.empty() && level_of_pos[s] != level_of_pos[s - 1]) L.lev_ptr.push_back(s);
    L.lev_ptr.push_back(n);
    std::vector<int64_t> srp(n + 1, 0);
    for (int s = 0; s < n; ++s) {
        const int r = row_order[s];
        srp[s + 1] = srp[s] + (pat.rowptr[r + 1] - pat.rowptr[r]);
    }
    L.addr.assign(pat.nnzb(), -1);
#pragma omp parallel for schedule(dynamic, 1024)
    for (int r = 0; r < n; ++r)
        for (int64_t k = pat.rowptr[r]; k < pat.rowptr[r + 1]; ++k) L.addr[k] = srp[L.inv[r]] + (k - pat.rowptr[r]);
    return L;
}

// lanes per block row: about one block per lane for multi-entry blocks; for
// scalar (1x1) operators ~4 entries per lane, so each lane keeps several
// independent loads in flight and the last partial pass wastes fewer lanes
int auto_lanes(double avg_blocks, int entries)
{
    const double per_lane = entries == 1 ? 4.0 : 1.0;
    int L = 2;
    while (L < 32 && L * 2 * per_lane < avg_blocks) L *= 2;
    return L;
}

std::shared_ptr<BsrStruct> bsr_make_struct(const BlockPattern& pat, const BsrLayout& lay, int Rb, int Cb,
                                           cudaStream_t s, int lanes)
{
    if (pat.nnzb() >= (1LL << 31)) throw Error(ED_UNSUPPORTED, "operator exceeds int32 block indices");
    auto st = std::make_shared<BsrStruct>();
    BsrStruct& S = *st;
    S.Rb = Rb;
    S.Cb = Cb;
    S.nbr = pat.nbr;
    S.nbc = pat.nbc;
    S.nnzb = pat.nnzb();
    const int n = pat.nbr;
    S.L = lanes > 0 ? lanes : auto_lanes(n > 0 ? static_cast<double>(S.nnzb) / n : 1.0, Rb * Cb);
    // sweeps are latency-bound: as many lanes as blocks per row (shorter chains)
    static const int ls_env = std::getenv("ED_SGS_LANES") ? std::atoi(std::getenv("ED_SGS_LANES")) : 0;
    S.Ls = lanes > 0 ? lanes : ls_env > 0 ? ls_env : auto_lanes(n > 0 ? static_cast<double>(S.nnzb) / n : 1.0, 9);
    S.h_rowptr.assign(n + 1, 0);
    S.h_col.assign(S.nnzb, 0);
    bool identity = true;
    for (int s2 = 0; s2 < n; ++s2) identity = identity && lay.perm[s2] == s2;
    std::vector<int> dpos(n, -1);
    for (int s2 = 0; s2 < n; ++s2) {
        const int r = lay.perm[s2];
        S.h_rowptr[s2 + 1] = static_cast<int>(S.h_rowptr[s2] + (pat.rowptr[r + 1] - pat.rowptr[r]));
    }
#pragma omp parallel for schedule(dynamic, 1024)
    for (int s2 = 0; s2 < n; ++s2) {
        const int r = lay.perm[s2];
        const int64_t len = pat.rowptr[r + 1] - pat.rowptr[r];
        for (int64_t k = 0; k < len; ++k) {
            const int c = pat.col[pat.rowptr[r] + k];
            S.h_col[S.h_rowptr[s2] + k] = c;
            if (c == r && pat.nbr == pat.nbc) dpos[s2] = static_cast<int>(S.h_rowptr[s2] + k);
        }
    }
    if (!identity) {
        S.h_perm = lay.perm;
        S.h_inv = lay.inv;
        S.perm.upload(S.h_perm, s);
        S.inv.upload(S.h_inv, s);
    }
    S.lev_ptr = lay.lev_ptr;
    S.leveled = !identity || S.lev_ptr.size() > 2;
    S.rowptr.upload(S.h_rowptr, s);
    S.col.upload(S.h_col, s);
    if (pat.nbr == pat.nbc) S.dpos.upload(dpos, s);
    // dataflow items: rows_per_item rows of one level each (256 threads / L lanes)
    const int nlev = S.nlev();
    S.rows_per_item = 256 / S.Ls;
    std::vector<int> irow{0};
    for (int l = 0; l < nlev; ++l)
        for (int r0 = S.lev_ptr[l]; r0 < S.lev_ptr[l + 1]; r0 += S.rows_per_item)
            irow.push_back(std::min(r0 + S.rows_per_item, S.lev_ptr[l + 1]));
    S.nitems = static_cast<int>(irow.size()) - 1;
    S.item_row.upload(irow, s);
    S.sync.alloc(2);
    S.sync.zero(s);
    S.d_lev_ptr.upload(S.lev_ptr, s);
    // narrow level schedules (every level fits one 512-thread CTA in <= 2 passes) run as one CTA
    int widest = 0;
    for (int l = 0; l < nlev; ++l) widest = std::max(widest, S.lev_ptr[l + 1] - S.lev_ptr[l]);
    S.chain = static_cast<int64_t>(widest) * S.Ls <= 1024;
    S.avg_rows_per_level = nlev > 0 ? S.nbr / nlev : 0;
    if (Rb == Cb && (Rb == 1 || Rb == 3) && pat.nbr == pat.nbc && S.leveled && S.nbr > 0) group_build(S, s);
    ED_CUDA(cudaStreamSynchronize(s)); // host vectors die at return
    return st;
}

void group_build(BsrStruct& S, cudaStream_t s)
{
    // narrow consecutive levels are merged while the group has <= grp_rows
    // scalar rows; a level wider than a quarter of that is a group of its own
    static const int grp_rows = std::getenv("ED_GROUP_ROWS") ? std::atoi(std::getenv("ED_GROUP_ROWS")) : 1024;
    const int B = S.Rb, n = S.nbr, nlev = S.nlev();
    std::vector<int4> grp;
    std::vector<int> grp_of(n, -1);
    for (int l = 0; l < nlev;) {
        const int a = S.lev_ptr[l];
        int e = l + 1;
        int m = (S.lev_ptr[e] - a) * B;
        if (grp_rows > 0 && 4 * m <= grp_rows)
            while (e < nlev && m + (S.lev_ptr[e + 1] - S.lev_ptr[e]) * B <= grp_rows &&
                   4 * (S.lev_ptr[e + 1] - S.lev_ptr[e]) * B <= grp_rows) {
                m += (S.lev_ptr[e + 1] - S.lev_ptr[e]) * B;
                ++e;
            }
        const int b = S.lev_ptr[e];
        const bool multi = e - l > 1;
        for (int r = a; r < b; ++r) grp_of[r] = multi ? static_cast<int>(grp.size()) : -1;
        grp.push_back(make_int4(a, b, multi ? m : 0, 0));
        l = e;
    }
    S.ngrp = static_cast<int>(grp.size());
    std::vector<long long> toff(grp.size(), 0);
    std::vector<int2> chunks;
    int64_t tot = 0;
    int maxm = 0;
    for (size_t g = 0; g < grp.size(); ++g) {
        const int m = grp[g].z;
        toff[g] = tot;
        if (m == 0) continue;
        tot += static_cast<int64_t>(m) * (m + 1) / 2;
        maxm = std::max(maxm, m);
        for (int j0 = 0; j0 < m; j0 += 32) chunks.push_back(make_int2(static_cast<int>(g), j0));
    }
    S.grp_tinv = tot;
    S.grp_maxm = maxm;
    // measured at 40^3 (profiles/r02/sweeps.md): one grid barrier costs ~1.3 us,
    // so level groups pay on narrow deep schedules (a coarse level: ~36 block
    // rows per level -> 9 levels per group step); wide levels stay on the
    // tagged dataflow sweep, which needs no grid-wide barrier per level
    static const int max_rpl = std::getenv("ED_GROUP_MAX_RPL") ? std::atoi(std::getenv("ED_GROUP_MAX_RPL")) : 64;
    S.grp_use = nlev > 0 && static_cast<double>(n) / nlev <= max_rpl && tot > 0;
    // dense-row levels (hundreds of blocks per row; the Galerkin products at 160^3): the whole CTA
    // works on one row at a time, so a row's blocks are in flight together (ED_GROUP_WIDE_ROW:
    // average blocks per row from which on, default 192)
    {
        const char* e = std::getenv("ED_GROUP_WIDE_ROW");
        const double wide = e ? std::atof(e) : 192.0;
        if (S.grp_use && n > 0 && static_cast<double>(S.nnzb) / n >= wide) S.Ls = 256;
    }
    S.ntchunk = static_cast<int>(chunks.size());
    const bool identity = S.h_inv.empty();
    std::vector<unsigned char> code(S.nnzb, 0);
    std::vector<int> gptr(n + 1, 0), gblk;
    std::vector<int> gcnt(n, 0);
#pragma omp parallel for schedule(dynamic, 1024)
    for (int sr = 0; sr < n; ++sr) {
        const int row = identity ? sr : S.h_perm[sr];
        int cnt = 0;
        for (int k = S.h_rowptr[sr]; k < S.h_rowptr[sr + 1]; ++k) {
            const int c = S.h_col[k];
            const int sc = identity ? c : S.h_inv[c];
            if (c == row) code[k] = 3;
            else if (grp_of[sr] >= 0 && grp_of[sc] == grp_of[sr]) code[k] = sc < sr ? 1 : 2;
            if (grp_of[sr] >= 0 && code[k] != 0) ++cnt;
        }
        gcnt[sr] = cnt;
    }
    for (int sr = 0; sr < n; ++sr) gptr[sr + 1] = gptr[sr] + gcnt[sr];
    gblk.resize(gptr[n]);
#pragma omp parallel for schedule(dynamic, 1024)
    for (int sr = 0; sr < n; ++sr) {
        if (grp_of[sr] < 0) continue;
        int o = gptr[sr];
        for (int k = S.h_rowptr[sr]; k < S.h_rowptr[sr + 1]; ++k)
            if (code[k] != 0) gblk[o++] = k;
    }
    S.grp.upload(grp, s);
    S.grp_toff.upload(toff, s);
    S.bcode.upload(code, s);
    S.gptr.upload(gptr, s);
    if (gblk.empty()) gblk.push_back(0);
    S.gblk.upload(gblk, s);
    if (chunks.empty()) chunks.push_back(make_int2(0, 0));
    S.tchunk.upload(chunks, s);
    S.gbar.alloc(1);
    S.gsbuf.alloc(std::max(maxm, 1));
}

std::vector<double> bsr_pack_values(const BsrStruct& st, const BsrLayout& lay, const std::vector<double>& bvals)
{
    const int E = st.Rb * st.Cb;
    std::vector<double> v(static_cast<size_t>(st.nval()), 0.0);
#pragma omp parallel for schedule(static)
    for (int64_t k = 0; k < static_cast<int64_t>(lay.addr.size()); ++k)
        for (int e = 0; e < E; ++e) v[lay.addr[k] * E + e] = bvals[k * E + e];
    return v;
}

BlockPattern block_pattern_of_csr(const HostCsr& a, int Rb, int Cb)
{
    if (a.nrows % Rb != 0 || a.ncols % Cb != 0)
        throw Error(ED_INVALID_ARGUMENT, "matrix size is not a multiple of the block size");
    BlockPattern p;
    p.nbr = a.nrows / Rb;
    p.nbc = a.ncols / Cb;
    p.rowptr.assign(p.nbr + 1, 0);
    std::vector<std::vector<int>> rows(p.nbr);
#pragma omp parallel
    {
        std::vector<int> mark(p.nbc, -1);
#pragma omp for schedule(dynamic, 1024)
        for (int I = 0; I < p.nbr; ++I) {
            auto& cols = rows[I];
            for (int r = I * Rb; r < (I + 1) * Rb; ++r)
                for (int64_t k = a.rowptr[r]; k < a.rowptr[r + 1]; ++k) {
                    const int J = a.col[k] / Cb;
                    if (mark[J] != I) {
                        mark[J] = I;
                        cols.push_back(J);
                    }
                }
            std::sort(cols.begin(), cols.end());
        }
    }
    for (int I = 0; I < p.nbr; ++I) p.rowptr[I + 1] = p.rowptr[I] + static_cast<int64_t>(rows[I].size());
    p.col.resize(p.rowptr[p.nbr]);
#pragma omp parallel for schedule(static)
    for (int I = 0; I < p.nbr; ++I) std::copy(rows[I].begin(), rows[I].end(), p.col.begin() + p.rowptr[I]);
    return p;
}

std::vector<double> block_values_of_csr(const HostCsr& a, const BlockPattern& pat, int Rb, int Cb)
{
    const int E = Rb * Cb;
    std::vector<double> v(static_cast<size_t>(pat.nnzb()) * E, 0.0);
#pragma omp parallel for schedule(dynamic, 1024)
    for (int I = 0; I < pat.nbr; ++I) {
        const auto b = pat.col.begin() + pat.rowptr[I];
        const auto e = pat.col.begin() + pat.rowptr[I + 1];
        for (int rr = 0; rr < Rb; ++rr) {
            const int r = I * Rb + rr;
            for (int64_t k = a.rowptr[r]; k < a.rowptr[r + 1]; ++k) {
                const int c = a.col[k];
                const int J = c / Cb, d = c % Cb;
                const int64_t blk = pat.rowptr[I] + (std::lower_bound(b, e, J) - b);
                v[static_cast<size_t>(blk) * E + rr * Cb + d] = a.val[k];
            }
        }
    }
    return v;
}

Bsr bsr_from_csr(const HostCsr& a, int Rb, int Cb, bool leveled, cudaStream_t s)
{
    const BlockPattern pat = block_pattern_of_csr(a, Rb, Cb);
    std::vector<int> order, lvl;
    if (leveled) {
        if (!pattern_symmetric(pat)) throw Error(ED_UNSUPPORTED, "Gauss-Seidel operator pattern is not symmetric");
        int nlev = 0;
        gs_level_order(pat, order, lvl, nlev);
    } else {
        order.resize(pat.nbr);
        std::iota(order.begin(), order.end(), 0);
    }
    BsrLayout lay = make_layout(pat, order, lvl);
    Bsr m;
    m.st = bsr_make_struct(pat, lay, Rb, Cb, s);
    if (leveled) m.st->leveled = true;
    m.val.upload(bsr_pack_values(*m.st, lay, block_values_of_csr(a, pat, Rb, Cb)), s);
    ED_CUDA(cudaStreamSynchronize(s));
    return m;
}

HostCsr bsr_to_csr(const Bsr& m, cudaStream_t s)
{
    const BsrStruct& S = *m.st;
    const std::vector<double> v = m.val.to_host(s);
    const int E = S.Rb * S.Cb;
    HostCsr a;
    a.nrows = S.nbr * S.Rb;
    a.ncols = S.nbc * S.Cb;
    a.rowptr.assign(a.nrows + 1, 0);
    auto srow = [&](int I) { return S.h_inv.empty() ? I : S.h_inv[I]; };
    for (int I = 0; I < S.nbr; ++I) {
        const int s2 = srow(I);
        for (int rr = 0; rr < S.Rb; ++rr)
            a.rowptr[I * S.Rb + rr + 1] = static_cast<int64_t>(S.h_rowptr[s2 + 1] - S.h_rowptr[s2]) * S.Cb;
    }
    for (int r = 0; r < a.nrows; ++r) a.rowptr[r + 1] += a.rowptr[r];
    a.col.resize(a.rowptr[a.nrows]);
    a.val.resize(a.rowptr[a.nrows]);
#pragma omp parallel for schedule(static)
    for (int I = 0; I < S.nbr; ++I) {
        const int s2 = srow(I);
        for (int rr = 0; rr < S.Rb; ++rr) {
            int64_t out = a.rowptr[I * S.Rb + rr];
            for (int k = S.h_rowptr[s2]; k < S.h_rowptr[s2 + 1]; ++k) {
                const int J = S.h_col[k];
                for (int d = 0; d < S.Cb; ++d) {
                    a.col[out] = J * S.Cb + d;
                    a.val[out] = v[static_cast<size_t>(k) * E + rr * S.Cb + d];
                    ++out;
                }
            }
        }
    }
    return a;
}

} // namespace edb
