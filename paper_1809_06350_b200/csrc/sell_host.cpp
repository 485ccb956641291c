// Host construction of SELL-32 block layouts and Gauss-Seidel level
// schedules.  Structure is mesh-static: it is built once per
// mesh (or per AMG level) and only values move per Newton step.
#include <algorithm>
#include <numeric>

#include "ed_internal.hpp"

namespace edb {

double Sell::bytes_per_spmv() const
{
    const SellStruct& S = *st;
    const double blk = 8.0 * S.Rb * S.Cb + 4.0;
    return static_cast<double>(S.nnzb) * blk + 4.0 * (S.nbr + 1) + 8.0 * S.nbr * S.Rb +
           8.0 * S.nbc * S.Cb;
}

void gs_level_order(const BlockPattern& pat, std::vector<int>& order, std::vector<int>& level_of_pos,
                    int& nlev)
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
    // stable counting sort by level (rows ascending inside a level)
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
    for (int i = 0; i < pat.nbr; ++i)
        for (int64_t k = pat.rowptr[i]; k < pat.rowptr[i + 1]; ++k) {
            const int j = pat.col[k];
            const auto b = pat.col.begin() + pat.rowptr[j];
            const auto e = pat.col.begin() + pat.rowptr[j + 1];
            if (!std::binary_search(b, e, i)) return false;
        }
    return true;
}

SellLayout make_sell_layout(const BlockPattern& pat, const std::vector<int>& row_order,
                            const std::vector<int>& level_of_pos)
{
    SellLayout L;
    const int n = pat.nbr;
    std::vector<int> slice_start; // positions where a slice starts
    std::vector<int> lev_first_slice;
    int prev_level = -1;
    int fill = 0;
    for (int pos = 0; pos < n; ++pos) {
        const int lv = level_of_pos.empty() ? 0 : level_of_pos[pos];
        if (lv != prev_level || fill == kLanes) {
            if (lv != prev_level) {
                // levels with no rows are impossible (levels are dense), so one
                // entry per level
                lev_first_slice.push_back(static_cast<int>(slice_start.size()));
                prev_level = lv;
            }
            slice_start.push_back(pos);
            fill = 0;
        }
        ++fill;
    }
    L.nslices = static_cast<int>(slice_start.size());
    lev_first_slice.push_back(L.nslices);
    L.lev_slice = lev_first_slice;
    if (n == 0) L.lev_slice = {0, 0};
    L.perm.assign(static_cast<size_t>(L.nslices) * kLanes, -1);
    L.rowlen.assign(static_cast<size_t>(L.nslices) * kLanes, 0);
    L.inv.assign(n, -1);
    L.slice_off.assign(L.nslices + 1, 0);
    for (int s = 0; s < L.nslices; ++s) {
        const int p0 = slice_start[s];
        const int p1 = (s + 1 < L.nslices) ? slice_start[s + 1] : n;
        int w = 0;
        for (int pos = p0; pos < p1; ++pos) {
            const int r = row_order[pos];
            const int lane = pos - p0;
            const int len = static_cast<int>(pat.rowptr[r + 1] - pat.rowptr[r]);
            L.perm[static_cast<size_t>(s) * kLanes + lane] = r;
            L.rowlen[static_cast<size_t>(s) * kLanes + lane] = len;
            L.inv[r] = s * kLanes + lane;
            w = std::max(w, len);
        }
        L.slice_off[s + 1] = L.slice_off[s] + w;
    }
    L.nslots = L.slice_off[L.nslices];
    L.addr.assign(pat.nnzb(), -1);
    for (int r = 0; r < n; ++r) {
        const int li = L.inv[r];
        const int s = li / kLanes, lane = li % kLanes;
        for (int64_t k = pat.rowptr[r]; k < pat.rowptr[r + 1]; ++k) {
            const int64_t slot = L.slice_off[s] + (k - pat.rowptr[r]);
            L.addr[k] = slot * kLanes + lane;
        }
    }
    return L;
}

std::shared_ptr<SellStruct> sell_make_struct(const BlockPattern& pat, const SellLayout& lay, int Rb,
                                             int Cb, cudaStream_t s)
{
    auto st = std::make_shared<SellStruct>();
    st->Rb = Rb;
    st->Cb = Cb;
    st->nbr = pat.nbr;
    st->nbc = pat.nbc;
    st->nslices = lay.nslices;
    st->nslots = lay.nslots;
    st->nnzb = pat.nnzb();
    st->lev_slice = lay.lev_slice;
    st->h_slice_off = lay.slice_off;
    st->h_perm = lay.perm;
    st->h_rowlen = lay.rowlen;
    st->h_inv = lay.inv;
    st->h_col.assign(static_cast<size_t>(lay.nslots) * kLanes, 0);
    for (int r = 0; r < pat.nbr; ++r)
        for (int64_t k = pat.rowptr[r]; k < pat.rowptr[r + 1]; ++k) st->h_col[lay.addr[k]] = pat.col[k];
    st->slice_off.upload(st->h_slice_off, s);
    st->perm.upload(st->h_perm, s);
    st->rowlen.upload(st->h_rowlen, s);
    st->inv.upload(st->h_inv, s);
    st->col.upload(st->h_col, s);
    return st;
}

std::vector<double> sell_pack_values(const SellStruct& st, const SellLayout& lay,
                                     const std::vector<double>& bvals)
{
    const int E = st.Rb * st.Cb;
    std::vector<double> v(static_cast<size_t>(st.nval()), 0.0);
    for (size_t k = 0; k < lay.addr.size(); ++k) {
        const int64_t a = lay.addr[k];
        const int64_t slot = a / kLanes;
        const int lane = static_cast<int>(a % kLanes);
        for (int e = 0; e < E; ++e) v[(slot * E + e) * kLanes + lane] = bvals[k * E + e];
    }
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
    std::vector<int> mark(p.nbc, -1);
    std::vector<int> cols;
    for (int I = 0; I < p.nbr; ++I) {
        cols.clear();
        for (int r = I * Rb; r < (I + 1) * Rb; ++r)
            for (int k = a.rowptr[r]; k < a.rowptr[r + 1]; ++k) {
                const int J = a.col[k] / Cb;
                if (mark[J] != I) {
                    mark[J] = I;
                    cols.push_back(J);
                }
            }
        std::sort(cols.begin(), cols.end());
        p.col.insert(p.col.end(), cols.begin(), cols.end());
        p.rowptr[I + 1] = static_cast<int64_t>(p.col.size());
    }
    return p;
}

std::vector<double> block_values_of_csr(const HostCsr& a, const BlockPattern& pat, int Rb, int Cb)
{
    const int E = Rb * Cb;
    std::vector<double> v(static_cast<size_t>(pat.nnzb()) * E, 0.0);
    for (int I = 0; I < pat.nbr; ++I) {
        const auto b = pat.col.begin() + pat.rowptr[I];
        const auto e = pat.col.begin() + pat.rowptr[I + 1];
        for (int rr = 0; rr < Rb; ++rr) {
            const int r = I * Rb + rr;
            for (int k = a.rowptr[r]; k < a.rowptr[r + 1]; ++k) {
                const int c = a.col[k];
                const int J = c / Cb, d = c % Cb;
                const int64_t blk = pat.rowptr[I] + (std::lower_bound(b, e, J) - b);
                v[static_cast<size_t>(blk) * E + rr * Cb + d] = a.val[k];
            }
        }
    }
    return v;
}

Sell sell_from_csr(const HostCsr& a, int Rb, int Cb, bool leveled, cudaStream_t s)
{
    const BlockPattern pat = block_pattern_of_csr(a, Rb, Cb);
    std::vector<int> order, lvl;
    if (leveled) {
        int nlev = 0;
        gs_level_order(pat, order, lvl, nlev);
    } else {
        order.resize(pat.nbr);
        std::iota(order.begin(), order.end(), 0);
    }
    const SellLayout lay = make_sell_layout(pat, order, lvl);
    Sell m;
    m.st = sell_make_struct(pat, lay, Rb, Cb, s);
    m.val.upload(sell_pack_values(*m.st, lay, block_values_of_csr(a, pat, Rb, Cb)), s);
    ED_CUDA(cudaStreamSynchronize(s)); // host vectors die at return
    return m;
}

HostCsr sell_to_csr(const Sell& m, cudaStream_t s)
{
    const SellStruct& S = *m.st;
    const std::vector<double> v = m.val.to_host(s);
    const int E = S.Rb * S.Cb;
    HostCsr a;
    a.nrows = S.nbr * S.Rb;
    a.ncols = S.nbc * S.Cb;
    a.rowptr.assign(a.nrows + 1, 0);
    for (int I = 0; I < S.nbr; ++I) {
        const int li = S.h_inv[I];
        for (int rr = 0; rr < S.Rb; ++rr) a.rowptr[I * S.Rb + rr + 1] = S.h_rowlen[li] * S.Cb;
    }
    for (int r = 0; r < a.nrows; ++r) a.rowptr[r + 1] += a.rowptr[r];
    a.col.resize(a.rowptr[a.nrows]);
    a.val.resize(a.rowptr[a.nrows]);
#pragma omp parallel for schedule(static)
    for (int I = 0; I < S.nbr; ++I) {
        const int li = S.h_inv[I];
        const int sl = li / kLanes, lane = li % kLanes;
        const int len = S.h_rowlen[li];
        for (int rr = 0; rr < S.Rb; ++rr) {
            int out = a.rowptr[I * S.Rb + rr];
            for (int t = 0; t < len; ++t) {
                const int64_t slot = S.h_slice_off[sl] + t;
                const int J = S.h_col[slot * kLanes + lane];
                for (int d = 0; d < S.Cb; ++d) {
                    a.col[out] = J * S.Cb + d;
                    a.val[out] = v[(slot * E + rr * S.Cb + d) * kLanes + lane];
                    ++out;
                }
            }
        }
    }
    return a;
}

} // namespace edb
